# forward tile bits of the multi-gate HBM passes: parity, then K1 at n = 13..16 with
# QPINN_HB_FWD_T = 12 (32 KB tiles) vs 13 (64 KB tiles, the default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "large_n or global_memory or hbm or big or whole_state" > gpurun_out/pytest_hbt.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbt.log
tail -2 gpurun_out/pytest_hbt.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbt.log | head -8
for T in 12 13; do
  echo "== QPINN_HB_FWD_T=$T"
  for c in "13 4 8192 strongly" "14 4 4096 strongly" "15 4 2048 strongly" "16 4 1024 strongly" "16 8 1024 strongly" "13 4 8192 cross_mesh" "14 4 4096 no_entanglement" "14 4 4096 cross_mesh_cnot"; do
    QPINN_HB_FWD_T=$T QPINN_VERBOSE=1 timeout 120 python scripts/pqc_big_one.py $c 2>&1 | grep -E "TFLOP|passes:" | sed 's/ops in .* passes:.*//' | tr '\n' ' '; echo
  done
done
