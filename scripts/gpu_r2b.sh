cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export QPINN_PARITY_REPORT=gpurun_out/parity
timeout 600 python scripts/fp32_error_budget.py > gpurun_out/fp32_error_budget.json 2> gpurun_out/fp32_error_budget.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/fp32_error_budget.json; tail -3 gpurun_out/fp32_error_budget.err
