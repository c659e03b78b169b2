# shared-address-space pointers in the tc kernels: repeatability, GPU suite, bench A/B vs exp/base.so
cd $GRAFT_REPO_ROOT
timeout 900 python scripts/race_gemm.py 300 2>&1 | grep "repeats differ"
timeout 900 python scripts/race_check.py 100 2>&1 | grep "repeats differ"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_smem2.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/pytest_smem2.log; grep -E "^FAILED" gpurun_out/pytest_smem2.log | head -6
KGREP="GPU kernel|gemm3_kernel|wgrad_kernel" bash scripts/gpu_var.sh base
