# adjoint tile bits at n = 13 (QPINN_HB_BWD_T = 12 vs 13): parity, then K2 timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QPINN_HB_BWD_T=13 timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "large_n or hbm" > gpurun_out/pytest_hbt2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbt2.log
tail -2 gpurun_out/pytest_hbt2.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbt2.log | head -8
for T in 12 13; do
  echo "== QPINN_HB_BWD_T=$T"
  for c in "13 1 8192 strongly" "13 4 8192 strongly" "13 8 8192 strongly" "13 4 8192 cross_mesh" "13 4 8192 no_entanglement"; do
    QPINN_HB_BWD_T=$T timeout 300 python scripts/pqc_big_bwd.py $c 2>&1 | tail -1
  done
done
