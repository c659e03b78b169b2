cd $GRAFT_REPO_ROOT
for a in "16 4 1024" "13 4 8192" "14 4 4096"; do timeout 120 python scripts/pqc_big_one.py $a strongly; timeout 120 python scripts/pqc_big_one.py $a cross_mesh; done
timeout 300 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "large_n or global_memory" 2>&1 | tail -2
