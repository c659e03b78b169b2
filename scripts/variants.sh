cd $GRAFT_REPO_ROOT
for v in default fb2 fb4; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; python scripts/profile_step.py 2>&1 | grep -E "features|GPU kernel"
done
