cd $GRAFT_REPO_ROOT
for v in default wp4; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; python scripts/gemm_check.py 2>&1 | grep -E "atb rows=262144"; python scripts/profile_step.py 2>&1 | grep -E "wgrad_kernel|GPU kernel"
done
