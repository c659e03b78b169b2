cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "large_n or global_memory or hbm" > gpurun_out/pytest_hbm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbm.log
tail -2 gpurun_out/pytest_hbm.log; grep -E "^FAILED|^E " gpurun_out/pytest_hbm.log | head -8
QPINN_VERBOSE=1 timeout 900 python scripts/sweep_pqc.py --quick --n=13,14,15,16 > gpurun_out/config5_hbm.jsonl 2> gpurun_out/config5_hbm.err
python -c "
import json
for l in open('gpurun_out/config5_hbm.jsonl'):
    d=json.loads(l); print(d['n'], d['L'], d['ansatz'], d['R'], d['k1_ms'], d['k1_tflops'], d.get('k2_ms'), d.get('k2_tflops'))
"
grep -m3 "adjoint" gpurun_out/config5_hbm.err; tail -2 gpurun_out/config5_hbm.err
