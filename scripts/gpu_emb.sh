# gb_embed4: large-n parity, f64 global paths, K1/K2 timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "large_n or global_memory or hbm or big or whole_state" > gpurun_out/pytest_emb.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_emb.log
tail -2 gpurun_out/pytest_emb.log; grep -E "^FAILED|^E " gpurun_out/pytest_emb.log | head -8
for c in "13 4 8192 strongly" "14 4 4096 strongly" "16 4 1024 strongly" "16 4 1024 no_entanglement"; do
  timeout 120 python scripts/pqc_big_one.py $c 2>&1 | tail -1
  timeout 300 python scripts/pqc_big_bwd.py $c 2>&1 | tail -1
done
