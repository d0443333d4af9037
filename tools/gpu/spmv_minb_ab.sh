cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for arm in cur minb4_s2 minb4_s3; do
  unset HFPG_SO_VARIANT HFPG_SPMV_STAGES
  case $arm in minb4_s2) export HFPG_SO_VARIANT=minb4 HFPG_SPMV_STAGES=2;; minb4_s3) export HFPG_SO_VARIANT=minb4;; esac
  echo "== $arm"; timeout 300 python tools/iter_driver.py --reps 5 2>&1 | tail -1
done; done
