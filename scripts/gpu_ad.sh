# fused-adapter epilogue variants: step-level GPU tests on the in-tree build, then bench A/B
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_headline_gpu.py tests/test_train_gpu.py tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
for v in "$@"; do QPINN_LIB_OVERRIDE=$PWD/exp/$v.so timeout 900 python -m pytest tests/test_headline_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done
KGREP="GPU kernel|gemm3_kernel<128, 1>" bash scripts/gpu_var.sh "$@"
