# GEMM stage-depth variants after the 3-op split: GEMM tests per variant, bench + step kernels A/B
cd $GRAFT_REPO_ROOT
for v in "$@"; do echo "== $v"; QPINN_LIB_OVERRIDE=$PWD/exp/$v.so timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
KGREP="GPU kernel|gemm3_kernel|wgrad_kernel" bash scripts/gpu_var.sh "$@"
