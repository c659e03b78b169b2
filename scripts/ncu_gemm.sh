cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/gemm_check.py > gpurun_out/gemm_check.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm3_kernel -s 12 -c 1 \
    -o gpurun_out/gemm_prof python scripts/gemm_check.py > gpurun_out/ncu_gemm.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_gemm.log
tail -4 gpurun_out/gemm_check.log; tail -2 gpurun_out/ncu_gemm.log
