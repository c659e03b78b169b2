cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pqc_gpu.py -q -p no:cacheprovider > gpurun_out/pqc_tests.log 2>&1; tail -3 gpurun_out/pqc_tests.log
python scripts/pqc_only.py 65536 strongly 20
python scripts/pqc_only.py 65536 cross_mesh 20
