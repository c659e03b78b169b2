cd $GRAFT_REPO_ROOT
timeout 600 python scripts/race_check.py 60 2>&1 | tail -30
for i in 1 2 3; do timeout 600 python -m pytest tests/test_pqc_gpu.py -q -x -p no:cacheprovider -k "large_batch or mid_sizes or headline" 2>&1 | tail -1; done
for i in 1 2; do timeout 900 python -m pytest tests/test_headline_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
