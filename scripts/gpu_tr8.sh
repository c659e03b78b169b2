# transfer-matrix K1/K2 at n = 8: parity, then config 5 n = 8 transfer vs layer kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pqc_gpu.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "transfer" > gpurun_out/pytest_tr8.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_tr8.log
tail -2 gpurun_out/pytest_tr8.log; grep -E "^FAILED|^E " gpurun_out/pytest_tr8.log | head -8
for v in transfer layer; do
  timeout 900 python scripts/sweep_pqc.py --n=8 --variant=$v > gpurun_out/c5_n8_$v.jsonl 2> gpurun_out/c5_n8_$v.err
done
python - <<'PY'
import json
t=[json.loads(l) for l in open('gpurun_out/c5_n8_transfer.jsonl') if l.startswith('{')]
y=[json.loads(l) for l in open('gpurun_out/c5_n8_layer.jsonl') if l.startswith('{')]
for a,b in zip(t,y):
    print(a['L'],a['ansatz'],a['R'],'| K1 transfer',a['k1_ms'],'layer',b['k1_ms'],'| K2 transfer',a.get('k2_ms'),'layer',b.get('k2_ms'))
PY
tail -3 gpurun_out/c5_n8_transfer.err
