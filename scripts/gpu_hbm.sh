cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pqc_gpu.py -m gpu -q --timeout 600 -p no:cacheprovider -k "large_n or global_memory or hbm" > gpurun_out/pytest_hbm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_hbm.log
tail -2 gpurun_out/pytest_hbm.log; grep -E "^FAILED|Error" gpurun_out/pytest_hbm.log | head -5
for a in "13 4 8192" "14 4 4096" "15 4 2048" "16 4 1024" "16 1 1024" "16 8 1024"; do timeout 120 python scripts/pqc_big_one.py $a strongly; timeout 120 python scripts/pqc_big_one.py $a cross_mesh; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/hbm_launches.csv python scripts/pqc_big_one.py 16 4 256 > gpurun_out/hbm_one.log 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.DictReader(l for l in open("gpurun_out/hbm_launches.csv") if l.startswith(chr(34)))]
agg=collections.defaultdict(float); cnt=collections.Counter()
for r in rows[len(rows)//2:]:
    k=r["Kernel Name"].split("(")[0][-40:]; v=float(r["Metric Value"].replace(",",""))
    agg[k]+=v; cnt[k]+=1
tot=sum(agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1]): print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}% x{cnt[k]:3d} {k}")
PY
