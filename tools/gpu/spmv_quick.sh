# SpMV timing from standalone iterations (tools/iter_driver.py), three runs
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do timeout 300 python tools/iter_driver.py --reps 20 2>&1 | tail -1; done
