"""Aggregate an `ncu --page source --print-source cuda,sass --csv` dump by CUDA line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
samp = defaultdict(int)
inst = defaultdict(int)
src = {}
cur = None
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:90]
    if r[2].strip() and cur:
        try:
            samp[cur] += int(r[4] or 0)
            inst[cur] += int(r[7] or 0)
        except ValueError:
            pass
tot_s = sum(samp.values()) or 1
tot_i = sum(inst.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{100*samp[k]/tot_s:5.1f}% smp {100*inst[k]/tot_i:5.1f}% ins  {k[0]}:{k[1]:4d}  {src.get(k,'')}")
