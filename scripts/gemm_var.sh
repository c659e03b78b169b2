cd $GRAFT_REPO_ROOT
for v in default p2 p4; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; python scripts/gemm_check.py 2>&1 | grep -E "262144|atb rows=262144" | sed 's/torch fp32 [0-9.e-]*;//'
done
