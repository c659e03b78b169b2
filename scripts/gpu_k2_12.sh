# launch list of one n = 12 (and n = 14) adjoint on the multi-gate HBM passes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/pqc_big_bwd.py 12 4 16384 strongly > gpurun_out/k2_12.txt 2>&1
timeout 300 python scripts/pqc_big_one.py 12 4 16384 strongly >> gpurun_out/k2_12.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k2_12_launches.csv python scripts/pqc_big_bwd.py 12 4 16384 strongly > gpurun_out/k2_12_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k2_14_launches.csv python scripts/pqc_big_bwd.py 14 4 4096 strongly > gpurun_out/k2_14_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hb_sm_pass" -s 30 -c 3 -o gpurun_out/k2_12_sm python scripts/pqc_big_bwd.py 12 4 16384 strongly > gpurun_out/k2_12_full.log 2>&1
cat gpurun_out/k2_12.txt
