# full GPU tests + 3 benches + step kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_q3.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_q3.log
tail -2 gpurun_out/pytest_q3.log; grep -E "^FAILED|^E " gpurun_out/pytest_q3.log | head -8
for v in "" QPINN_SERIAL_BWD=1 "" QPINN_SERIAL_BWD=1; do
  env $v timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b_q3.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_q3.json')); print('$v', d['ms_per_step'], d['value'], d['e2e']['value'], d['gpu_launches'])"
done
timeout 300 python scripts/profile_step.py > gpurun_out/step_kernels_q3.txt 2>&1; grep -E "GPU kernel|tr_" gpurun_out/step_kernels_q3.txt
