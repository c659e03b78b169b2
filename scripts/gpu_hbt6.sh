# adjoint tile bits at n = 14, 15: 12 vs 13 (with CS passes carrying the checkpoint)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QPINN_HB_BWD_T=13 timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "large_n or hbm" > gpurun_out/pytest_hbt6.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbt6.log
tail -2 gpurun_out/pytest_hbt6.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbt6.log | head -8
for T in 12 13; do
  echo "== QPINN_HB_BWD_T=$T"
  for c in "14 4 4096 strongly" "14 4 4096 cross_mesh" "15 4 2048 strongly" "15 4 2048 no_entanglement"; do
    QPINN_HB_BWD_T=$T timeout 300 python scripts/pqc_big_bwd.py $c 2>&1 | tail -1
  done
done
