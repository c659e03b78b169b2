cd $GRAFT_REPO_ROOT
for v in default k1un; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  for k in strongly cross_mesh; do echo "$v $k"; python scripts/pqc_only.py 65536 $k 20 2>&1 | grep -v replay; done
done
