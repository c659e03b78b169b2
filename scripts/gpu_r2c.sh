cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export QPINN_PARITY_REPORT=gpurun_out/parity
timeout 300 ./scripts/probes/mma_rate > gpurun_out/mma_rate.txt 2>&1
timeout 1500 python -m pytest tests/test_pqc_gpu.py tests/test_train_gpu.py tests/test_headline_gpu.py tests/test_probes_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log; cat gpurun_out/mma_rate.txt
