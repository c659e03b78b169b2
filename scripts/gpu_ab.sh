# GPU tests, then an A/B of one env switch on the bench: bash scripts/gpu_ab.sh VAR
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_ab.log
tail -2 gpurun_out/pytest_ab.log; grep -E "^FAILED|^E " gpurun_out/pytest_ab.log | head -8
for v in 1 0 1 0; do
  env $1=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_ab.json')); print('$1=$v', d['ms_per_step'], d['value'], d['e2e']['value'])"
done
timeout 300 python scripts/profile_step.py > gpurun_out/step_kernels_ab.txt 2>&1; grep -E "GPU kernel|tanh" gpurun_out/step_kernels_ab.txt
