# after the proxy-fence fix: GEMM + PQC repeatability, full GPU suite, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/race_gemm.py 400 2>&1 | grep "repeats differ"
timeout 900 python scripts/race_check.py 150 2>&1 | grep "repeats differ"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_fence.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/pytest_fence.log; grep -E "^FAILED" gpurun_out/pytest_fence.log | head -6
for i in 1 2 3; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_f.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_f.json')); print(d['ms_per_step'], d['value'])"; done
timeout 300 python scripts/profile_step.py 2>&1 | grep -E "GPU kernel|gemm3|wgrad"
