# full GPU tests + bench + step kernels (quick check of a step-path change)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_q2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_q2.log
tail -2 gpurun_out/pytest_q2.log; grep -E "^FAILED|^E " gpurun_out/pytest_q2.log | head -8
for i in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_q2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_q2.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
done
timeout 300 python scripts/profile_step.py > gpurun_out/step_kernels_q2.txt 2>&1; grep -E "GPU kernel time|wgrad|colsum" gpurun_out/step_kernels_q2.txt
