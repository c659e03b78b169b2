cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python scripts/pqc_only.py 65536 strongly 20 --variant=layer > gpurun_out/k1_layer.txt 2>&1
timeout 120 python scripts/pqc_only.py 65536 cross_mesh 20 --variant=layer >> gpurun_out/k1_layer.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"pqc_forward_layer|pqc_backward_layer" -s 6 -c 2 -o gpurun_out/k1k2_layer python scripts/pqc_only.py 65536 strongly 3 --variant=layer > gpurun_out/ncu_k1.log 2>&1
cat gpurun_out/k1_layer.txt; tail -2 gpurun_out/ncu_k1.log
