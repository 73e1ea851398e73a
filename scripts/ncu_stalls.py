"""Per-CUDA-line stall breakdown (excluding barrier waits) from an ncu source CSV."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
acc = defaultdict(lambda: defaultdict(int))
src = {}
cur = fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        cols = {h: i for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
    if r[2].strip() and cur:
        for h, i in cols.items():
            try:
                acc[cur][h] += int(r[i] or 0)
            except ValueError:
                pass
tot = defaultdict(int)
for k, d in acc.items():
    for h, v in d.items():
        tot[h] += v
T = sum(tot.values()) or 1
print("overall:", ", ".join(f"{h[6:]} {100*v/T:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
nb = {k: sum(v for h, v in d.items() if h != "stall_barrier") for k, d in acc.items()}
for k in sorted(nb, key=lambda k: -nb[k])[:top]:
    d = acc[k]
    reasons = ", ".join(f"{h[6:]}={v}" for h, v in sorted(d.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{nb[k]:6d}  {k[0]}:{k[1]:4d}  {src.get(k,'')[:60]:60s} | {reasons}")
