# shared-address-space fix in the tc kernels: full GPU suite on the in-tree build, bench A/B vs variants
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_smem.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/pytest_smem.log; grep -E "^FAILED|^E " gpurun_out/pytest_smem.log | head -6
KGREP="GPU kernel|gemm3_kernel|wgrad_kernel" bash scripts/gpu_var.sh "$@"
