cd $GRAFT_REPO_ROOT
for lib in default m3 m4 g2m4; do
  if [ $lib = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$lib.so; fi
  echo "== $lib"
  for a in "16 4 1024" "13 4 8192"; do timeout 120 python scripts/pqc_big_one.py $a strongly; timeout 120 python scripts/pqc_big_one.py $a cross_mesh; done
done
