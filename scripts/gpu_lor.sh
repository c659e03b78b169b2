# split variant: GEMM accuracy under exp/<tag>.so, then bench + per-kernel A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v gemm tests"
  QPINN_LIB_OVERRIDE=$PWD/exp/$v.so timeout 600 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
  QPINN_LIB_OVERRIDE=$PWD/exp/$v.so timeout 300 python scripts/gemm_check.py 2>&1 | tail -12
done
echo "== default"; timeout 300 python scripts/gemm_check.py 2>&1 | tail -12
KGREP="GPU kernel|wgrad|gemm3" bash scripts/gpu_var.sh "$@"
