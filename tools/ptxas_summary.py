"""Summarise nvcc -Xptxas -v output: kernel, registers, spills, smem (static)."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2103_07706_b200/lib/ptxas.log").read()
cur = None
rows = {}
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        try:
            cur = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        except OSError:
            pass
        cur = re.sub(r"\(pswe::GridDev.*", "", cur).replace("void pswe::", "")
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and "spill" not in rows[cur]:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for k, v in rows.items():
    if pat in k:
        print(f"{k[:60]:60s} regs {v.get('regs', '?'):>4}  spill {v.get('spill', '?')}")
