# Round-2 measurement pass: bench lines (fp32 headline, fp64 context), ncu launch
# list, per-pass DRAM traffic, full ncu capture of the step's top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 600 python bench.py --dtype f64 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_f64.json 2> $O/bench_f64.err
timeout 300 python scripts/profile_step.py > $O/step_kernels.txt 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_small.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "ncu launches exit $?" >> $O/ncu_launch.log
timeout 600 ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file $O/traffic.csv python scripts/ncu_traffic.py > $O/traffic.log 2>&1 && \
python scripts/traffic_json.py $O/traffic.csv $(awk '/^points/{print $2}' $O/traffic.log) > $O/traffic.json 2>&1
echo "traffic exit $?" >> $O/traffic.log
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'gemm3_kernel|wgrad_kernel|tr_seed|tanh_bwd_bias|features_bwd|adapter_bwd|tr_embed_grad' -s 40 -c 16 \
    -o $O/step_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo "ncu full exit $?" >> $O/ncu_full.log
cut -c1-400 $O/bench.json; tail -1 $O/bench.err; cut -c1-300 $O/bench_f64.json; head -3 $O/step_kernels.txt; tail -1 $O/ncu_launch.log $O/traffic.log $O/ncu_full.log
