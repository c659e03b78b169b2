# bench A/B of in-tree .so vs exp/<tag>.so variants: bash scripts/gpu_var.sh tag1 tag2 ...
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_var.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_var.json')); print('$v', d['ms_per_step'], d['value'])"
done
done
for v in default "$@"; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; timeout 300 python scripts/profile_step.py 2>/dev/null | grep -E "$KGREP"
done
