cd $GRAFT_REPO_ROOT
for v in default p2 p4; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; python scripts/profile_step.py 2>&1 | grep -E "gemm3|wgrad_kernel|GPU kernel"
done
