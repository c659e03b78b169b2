cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 180 python scripts/gemm_check.py > gpurun_out/gemm_pair.txt 2>&1; echo "pair exit $?" >> gpurun_out/gemm_pair.txt
QPINN_GEMM_PAIR=0 timeout 180 python scripts/gemm_check.py > gpurun_out/gemm_single.txt 2>&1; echo "single exit $?" >> gpurun_out/gemm_single.txt
cat gpurun_out/gemm_pair.txt; grep 262144 gpurun_out/gemm_single.txt
