# Round-2 full GPU pass: whole GPU suite (with parity reports), smoke, bench,
# per-kernel step profile, launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export QPINN_PARITY_REPORT=gpurun_out/parity
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 python scripts/profile_step.py > gpurun_out/prof_step.txt 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launch.log
tail -2 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head; tail -1 gpurun_out/smoke.log; cut -c1-300 gpurun_out/bench.json; tail -1 gpurun_out/bench.err; head -30 gpurun_out/prof_step.txt
