"""Print the SASS lines with the most stall samples from an `ncu --page source --csv` dump."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
seen = set()
data = []
for r in rows[2:]:
    if len(r) == len(hdr) and r[0] != "Address" and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
S = idx["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[S] or 0) for r in data)
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("total samples", tot)
top = sorted(data, key=lambda r: -float(r[S] or 0))[:n]
for r in top:
    st = sorted(((float(r[idx[c]] or 0), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{r[idx['Address']]:>6} {float(r[S]):6.0f} {100*float(r[S])/tot:5.1f}%  {r[idx['Source']][:60]:60s} " +
          " ".join(f"{c}={int(v)}" for v, c in st if v))
