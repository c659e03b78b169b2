# forward tile bits at n = 14: 12 vs 13 vs 14 (the whole state per tile)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QPINN_HB_FWD_T=14 timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "large_n or global_memory or hbm" > gpurun_out/pytest_hbt3.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbt3.log
tail -2 gpurun_out/pytest_hbt3.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbt3.log | head -8
for T in 12 13 14; do
  echo "== QPINN_HB_FWD_T=$T"
  for c in "14 4 4096 strongly" "14 8 4096 strongly" "14 4 4096 cross_mesh" "14 4 4096 no_entanglement" "14 4 4096 cross_mesh_cnot"; do
    QPINN_HB_FWD_T=$T timeout 120 python scripts/pqc_big_one.py $c 2>&1 | tail -1
  done
done
