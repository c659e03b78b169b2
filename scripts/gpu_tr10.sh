# transfer-matrix K1/K2 at n = 10 (opt-in): parity, then config 5 n = 9 transfer vs the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 900 -p no:cacheprovider -k "transfer and (10 or 9)" > gpurun_out/pytest_tr10.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_tr10.log
tail -2 gpurun_out/pytest_tr10.log; grep -E "^FAILED|^E " gpurun_out/pytest_tr10.log | head -8
for v in transfer auto; do
  timeout 900 python scripts/sweep_pqc.py --n=10 --variant=$v > gpurun_out/c5_n10_$v.jsonl 2> gpurun_out/c5_n10_$v.err
done
python - <<'PY'
import json
t=[json.loads(l) for l in open('gpurun_out/c5_n10_transfer.jsonl') if l.startswith('{')]
y=[json.loads(l) for l in open('gpurun_out/c5_n10_auto.jsonl') if l.startswith('{')]
for a,b in zip(t,y):
    print(a['L'],a['ansatz'],a['R'],'| K1 transfer',a['k1_ms'],'auto',b['k1_ms'],'| K2 transfer',a.get('k2_ms'),'auto',b.get('k2_ms'))
PY
tail -3 gpurun_out/c5_n10_transfer.err
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_tr10.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b_tr10.json')); print('bench', d['ms_per_step'], d['value'])"
