cd $GRAFT_REPO_ROOT
for v in default "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; timeout 600 python scripts/race_gemm.py 200 2>&1 | grep "repeats differ"
done
