cd $GRAFT_REPO_ROOT
for v in default emb4 emb6; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; KINDS=strongly VARIANTS=auto python scripts/bench_transfer.py 2>&1 | tail -1
done
