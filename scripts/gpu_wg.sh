# weight-gradient kernel: GEMM tests, then bench A/B of the in-tree .so vs exp/wold.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_wg.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_wg.log
tail -3 gpurun_out/pytest_wg.log; grep -E "^FAILED|^E " gpurun_out/pytest_wg.log | head -8
QPINN_LIB_OVERRIDE=$PWD/exp/wold.so timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider -k atb 2>&1 | tail -2
KGREP="GPU kernel|wgrad" bash scripts/gpu_var.sh wold
