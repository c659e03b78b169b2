# Full GPU pass: parity suite, smoke, bench, launch list + ncu captures of the top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
python scripts/profile_step.py > gpurun_out/prof_step.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launch.log
# one full capture per hot kernel family, from the bench step itself (after warmup)
ncu --set full --clock-control none --import-source on \
    -k regex:'pqc_backward_layer|pqc_forward_layer|gemm3_kernel|wgrad_kernel|tr_embed|tr_seed|tr_readout' -s 60 -c 14 \
    -o gpurun_out/step_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
# DRAM bytes per pass -> traffic.json (copied to profiles/ after review)
ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file gpurun_out/traffic.csv python scripts/ncu_traffic.py > gpurun_out/traffic.log 2>&1 && \
python scripts/traffic_json.py gpurun_out/traffic.csv $(awk '/^points/{print $2}' gpurun_out/traffic.log) \
    > gpurun_out/traffic.json 2>&1
echo "traffic exit $?" >> gpurun_out/traffic.log
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -1 gpurun_out/bench.err; head -3 gpurun_out/prof_step.txt; tail -1 gpurun_out/ncu_full.log
