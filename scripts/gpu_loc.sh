cd $GRAFT_REPO_ROOT
export QPINN_GEMM_PAIR=0
for lib in default snpms; do
  if [ $lib = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$lib.so; fi
  echo "== $lib"
  for s in "262144 128 256" "2097152 128 32" "1048576 128 64" "524288 128 128" "262144 128 128"; do
    timeout 60 python scripts/gemm_one.py $s 20
  done
done
