cd $GRAFT_REPO_ROOT
for v in default raw4 bs3 raw4bs3; do
  if [ $v = default ]; then unset QPINN_LIB_OVERRIDE; else export QPINN_LIB_OVERRIDE=$PWD/exp/$v.so; fi
  echo "== $v"; KINDS=strongly VARIANTS=auto python scripts/bench_transfer.py 2>&1 | tail -1
  python bench.py --no-cpu-baseline --steps 30 2>gpurun_out/gv_$v.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', d['ms_per_step'], {k: v['ms_per_launch'] for k,v in d['roofline_kernels'].items()})"
done
