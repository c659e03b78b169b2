# split-mode candidates: full GPU suite under exp/<tag>.so, FP32 error budget per variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  QPINN_LIB_OVERRIDE=$PWD/exp/$v.so timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$v.log 2>&1
  echo "== $v pytest exit $?"; tail -1 gpurun_out/pytest_$v.log; grep -E "^FAILED|^E " gpurun_out/pytest_$v.log | head -6
done
for v in default "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  timeout 600 python scripts/fp32_error_budget.py > gpurun_out/eb_$v.json 2>/dev/null
  echo "== $v"; cat gpurun_out/eb_$v.json | tr -d '\n'; echo
done
