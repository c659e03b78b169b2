# SM-pass variants (swizzled tile, OUTER pairs; QPINN_HB_G / QPINN_HB_MINB builds in exp/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "large_n or global_memory or hbm or big or whole_state" > gpurun_out/pytest_hbvar.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbvar.log
tail -2 gpurun_out/pytest_hbvar.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbvar.log | head -8
for v in default "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"
  for c in "12 4 16384 strongly" "14 4 4096 strongly" "16 4 1024 strongly" "13 4 8192 cross_mesh" "12 4 16384 no_entanglement"; do
    timeout 120 python scripts/pqc_big_one.py $c 2>&1 | tail -1
    timeout 300 python scripts/pqc_big_bwd.py $c 2>&1 | tail -1
  done
done
