# iter_driver under each in-tree variant .so: VARIANTS="a b" bash tools/gpu/variants.sh
cd $GRAFT_REPO_ROOT
echo "== default"; timeout 300 python tools/iter_driver.py --reps 5 --config ${CFG:-3d_1m} 2>&1 | tail -1
for v in $VARIANTS; do
  echo "== $v"; HFPG_SO_VARIANT=$v timeout 300 python tools/iter_driver.py --reps 5 --config ${CFG:-3d_1m} 2>&1 | tail -1
done
