cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out

python scripts/pqc_only.py 65536 strongly 20 > gpurun_out/pqc_only.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:pqc_(forward|backward)_(kernel|layer)' -s 6 -c 2 \
    -o gpurun_out/pqc_prof python scripts/pqc_only.py 65536 strongly 1 > gpurun_out/ncu_pqc.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_pqc.log
cat gpurun_out/pqc_only.log; tail -2 gpurun_out/ncu_pqc.log
