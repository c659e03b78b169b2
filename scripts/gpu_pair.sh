cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QPINN_GEMM_PAIR=1 timeout 180 python scripts/gemm_check.py > gpurun_out/gemm_pair.txt 2>&1; echo "pair exit $?" >> gpurun_out/gemm_pair.txt
QPINN_GEMM_PAIR=0 timeout 180 python scripts/gemm_check.py > gpurun_out/gemm_single.txt 2>&1; echo "single exit $?" >> gpurun_out/gemm_single.txt
grep -E "M=|exit" gpurun_out/gemm_pair.txt | cut -c1-130; grep 262144 gpurun_out/gemm_single.txt | cut -c1-130
