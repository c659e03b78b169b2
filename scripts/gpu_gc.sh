cd $GRAFT_REPO_ROOT
for lib in snpms snpms_os4 snp_os4; do
  export QPINN_LIB_OVERRIDE=$PWD/exp/$lib.so
  echo "== $lib"
  for s in "262144 128 256" "262144 128 128"; do timeout 60 python scripts/gemm_one.py $s 20; done
done
