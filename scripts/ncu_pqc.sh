cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pqc_gpu.py -q -p no:cacheprovider > gpurun_out/pqc_tests.log 2>&1; tail -2 gpurun_out/pqc_tests.log
python scripts/pqc_only.py 65536 strongly 20 > gpurun_out/pqc_only.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:pqc_(forward|backward)_kernel' -s 6 -c 2 \
    -o gpurun_out/pqc_prof python scripts/pqc_only.py 65536 strongly 1 > gpurun_out/ncu_pqc.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_pqc.log
cat gpurun_out/pqc_only.log; tail -2 gpurun_out/ncu_pqc.log
