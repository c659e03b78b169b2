# Round-2 parity pass: headline-size parity, the reference-through-ABI binding,
# the data-parallel domain rule, smoke on the bench path, a short bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export QPINN_PARITY_REPORT=gpurun_out/parity
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -s \
  -k "not config1" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
QPINN_BENCH_FUNCTIONAL_DP=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_dp2.log 2>&1
echo "bench dp2 exit $?" >> gpurun_out/bench_dp2.log
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log | cut -c1-400; tail -2 gpurun_out/bench_dp2.log | cut -c1-300
