"""profiles/traffic.json from the ncu CSV of scripts/ncu_traffic.py (one eager config-2
step, dram__bytes_read.sum + dram__bytes_write.sum per kernel): kernels are assigned to
the step's passes by launch order (trunk forward | PQC forward | loss | PQC backward |
trunk backward | Adam)."""
import csv
import json
import sys

src, points = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.DictReader(l for l in open(src) if l.startswith('"'))]
by_id = {}
for r in rows:
    k = by_id.setdefault(r["ID"], {"name": r["Kernel Name"], "bytes": 0.0})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    k["bytes"] += v * scale
seq = [by_id[i] for i in sorted(by_id, key=int)]
PQC_START = ("tr_tables", "pqc_prepare_tables", "pqc_forward", "pqc_backward")
passes = {"trunk_forward": [], "pqc_forward": [], "loss": [], "pqc_backward": [],
          "trunk_backward": [], "adam": []}
state = "trunk_forward"
for k in seq:
    nm = k["name"]
    if state == "trunk_forward" and any(s in nm for s in PQC_START):
        state = "pqc_forward"
    elif state == "pqc_forward" and "loss_" in nm:
        state = "loss"
    elif state == "loss" and "loss_" not in nm:
        state = "pqc_backward"
    elif state == "pqc_backward" and ("features" in nm or "adapter" in nm or "tanh_bwd" in nm):
        state = "trunk_backward"
    elif "adam" in nm:
        state = "adam"
    passes[state].append(k)
out = {}
for name in ("trunk_forward", "pqc_forward", "pqc_backward", "trunk_backward"):
    ks = passes[name]
    out[name] = {"bytes_per_point": round(sum(k["bytes"] for k in ks) / points, 1),
                 "kernels": len(ks),
                 "kernel_names": [k["name"].split("(")[0][-40:] for k in ks],
                 "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                           "(one eager config-2 step, scripts/ncu_traffic.py + traffic_json.py)"}
json.dump(out, sys.stdout, indent=1)
print()
