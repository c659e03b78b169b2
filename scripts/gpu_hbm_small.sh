# multi-gate HBM passes at n <= 12 (whole-state tiles): parity, then config-5 n = 9..13 forced on
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "large_n or global_memory or hbm or big or whole_state" > gpurun_out/pytest_hbm_small.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbm_small.log
tail -2 gpurun_out/pytest_hbm_small.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbm_small.log | head -8
QPINN_PQC_HBM_FWD_MIN=9 QPINN_PQC_HBM_BWD_MIN=9 timeout 900 python scripts/sweep_pqc.py --n=9,10,11,12,13 > gpurun_out/c5_hbm_small2.jsonl 2> gpurun_out/c5_hbm_small2.err
python - <<'PY'
import json
for l in open('gpurun_out/c5_hbm_small2.jsonl'):
    if l.startswith('{'):
        a=json.loads(l); print(a['n'],a['L'],a['ansatz'],a['R'],'|',a['k1_ms'],a['k1_tflops'],'|',a['k2_ms'],a['k2_tflops'])
PY
