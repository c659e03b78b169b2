# Round-2 final measurement pass without the config-4/5 sweeps (after the split-mode change)
# parity reports, FP32 error budget.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
O=gpurun_out/r02
export QPINN_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.json 2> $O/bench_reference.err
timeout 600 python bench.py --dtype f64 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_f64.json 2> $O/bench_f64.err
timeout 900 python bench.py --workload config3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config3_1gpu.json 2> $O/bench_config3.err
QPINN_BENCH_FUNCTIONAL_DP=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_dp2_functional_gloo.log 2>&1
timeout 300 python scripts/profile_step.py > $O/step_kernels.txt 2>&1
timeout 600 python scripts/fp32_error_budget.py > $O/fp32_error_budget.json 2> $O/fp32_error_budget.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_small.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file $O/traffic.csv python scripts/ncu_traffic.py > $O/traffic.log 2>&1 && \
python scripts/traffic_json.py $O/traffic.csv $(awk '/^points/{print $2}' $O/traffic.log) > $O/traffic.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'gemm3_kernel|wgrad_kernel|tr_seed|tanh_bwd_bias|features_bwd|adapter_bwd|tr_embed_grad' -s 40 -c 16 \
    -o $O/step_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
tail -1 $O/pytest_gpu.log; tail -1 $O/smoke.log; cut -c1-200 $O/bench.json
