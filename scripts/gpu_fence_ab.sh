# proxy fence cost: GEMM timing (gemm_check) and the bench's transfer-GEMM roofline, in-tree vs exp/nofence.so
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in default nofence; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; timeout 300 python scripts/gemm_check.py 2>&1 | grep -E "M=262144"
  timeout 300 python -c "
import bench; r = bench.tensor_gemm_roofline(7, 65536); print('transfer_gemm', r['ms_per_launch'], r['achieved'], r['frac'])"
done; done
