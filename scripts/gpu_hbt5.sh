# adjoint with the forward's tile bits in its forward segments: parity + K1/K2 at n = 13..16
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "large_n or global_memory or hbm or big or whole_state" > gpurun_out/pytest_hbt5.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbt5.log
tail -2 gpurun_out/pytest_hbt5.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbt5.log | head -8
for c in "13 4 8192 strongly" "14 4 4096 strongly" "14 8 4096 strongly" "14 4 4096 cross_mesh_cnot" "14 4 4096 no_entanglement" "16 4 1024 strongly"; do
  timeout 120 python scripts/pqc_big_one.py $c 2>&1 | tail -1
  timeout 300 python scripts/pqc_big_bwd.py $c 2>&1 | tail -1
done
