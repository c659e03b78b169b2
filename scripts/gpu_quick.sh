# quick GPU pass: the PQC/GEMM/headline parity tests, smoke, a 20-step bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export QPINN_PARITY_REPORT=gpurun_out/parity
timeout 900 python -m pytest tests/test_pqc_gpu.py tests/test_gemm_gpu.py tests/test_headline_gpu.py tests/test_train_gpu.py tests/test_probes_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "not config1" > gpurun_out/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_quick.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
echo "bench exit $?" >> gpurun_out/bench_quick.err
QPINN_FUSE_ADAPTER=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_quick_unfused.json 2>&1
tail -2 gpurun_out/pytest_quick.log; grep -E "^FAILED" gpurun_out/pytest_quick.log | head; tail -1 gpurun_out/smoke.log
python - <<'PY'
import json
for f in ("gpurun_out/bench_quick.json", "gpurun_out/bench_quick_unfused.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        rk = d["roofline_kernels"]
        print(f, d["ms_per_step"], d["value"], {k: rk[k]["ms_per_launch"] for k in rk})
    except Exception as e:
        print(f, "failed", e)
PY
