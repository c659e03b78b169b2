"""Per-kernel table from an ncu --set full report: time, DRAM bytes, issue and
tensor-pipe activity, registers, grid (ncu -i REP --page raw --csv)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
want = [("time_us", "gpu__time_duration.sum", 1),
        ("dram_rd_MB", "dram__bytes_read.sum", None), ("dram_wr_MB", "dram__bytes_write.sum", None),
        ("issue_%", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
        ("tc_pipe_%", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
        ("tmem_%", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
        ("regs", "launch__registers_per_thread", 1), ("grid", "launch__grid_size", 1)]
scale_mb = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
print(f"{'kernel':60s}" + "".join(f"{w[0]:>12s}" for w in want))
for r in data:
    name = r[col["Kernel Name"]][:58]
    out = []
    for label, m, sc in want:
        if m not in col:
            out.append(f"{'-':>12s}")
            continue
        try:
            v = float(r[col[m]].replace(",", "") or 0)
        except ValueError:  # "no data" for this kernel
            out.append(f"{'n/a':>12s}")
            continue
        if sc is None:
            v *= scale_mb.get(units[col[m]], 1e-6)
        elif label == "time_us":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(units[col[m]], 1.0)
        else:
            v *= sc
        out.append(f"{v:12.1f}")
    print(f"{name:60s}" + "".join(out))
