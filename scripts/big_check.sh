cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pqc_gpu.py -q -p no:cacheprovider -k "cluster" --timeout 600 > gpurun_out/big_tests.log 2>&1; tail -25 gpurun_out/big_tests.log
