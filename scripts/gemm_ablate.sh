# GEMM ablation timing (tc_gemm.cu QPINN_ABL_* switches): which role bounds the kernel.
# Build here first: python scripts/build_variant.py <tag> tc_gemm.cu -DQPINN_ABL_...=1
# usage: bash scripts/gemm_ablate.sh default <tag> ...   (exp/<tag>.so must travel)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; python scripts/gemm_check.py 2>&1 | grep -E "262144" | sed 's/torch fp32 [0-9.e-]*;//'
done
