"""Summarise ptxas -v output: registers and spills per kernel (dev tool)."""
import re
import subprocess
import sys

text = open(sys.argv[1] if len(sys.argv) > 1 else "ptxas.log").read().splitlines()
props, regs = {}, {}
cur = None
for i, l in enumerate(text):
    m = re.search(r"Function properties for (\S+)", l)
    if m:
        cur = m.group(1)
        m2 = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", text[i + 1])
        props[cur] = m2.groups() if m2 else None
        continue
    m = re.search(r"Used (\d+) registers", l)
    if m and cur:
        regs[cur] = m.group(1)
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for k in regs:
    dm = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    dm = re.sub(r"\(.*", "", dm)
    if pat in dm:
        print(f"{dm:55s} regs={regs[k]:>4s} stack/spill_st/spill_ld={props.get(k)}")
