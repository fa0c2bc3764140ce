#!/usr/bin/env python
"""Per-CUDA-line instruction counts from `ncu --page source --csv --print-source cuda,sass` output.
usage: ncu_lines.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
per_line = collections.Counter()
stall = collections.Counter()
src = {}
hdr = None
fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if "Instructions Executed" in r:
        hdr = r
        iN = hdr.index("Instructions Executed")
        iSt = hdr.index("# Samples")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if not r[0]:
        continue  # SASS rows under a CUDA line (already summed into that line's row)
    key = (fname, r[0])
    if r[1]:
        src[key] = r[1]
    try:
        per_line[key] += int(r[iN])
        stall[key] += int(r[iSt])
    except ValueError:
        pass
tot = sum(per_line.values()) or 1
stot = sum(stall.values()) or 1
print("total warp instructions", tot, "samples", stot)
for key, n in per_line.most_common(top):
    print(f"{100 * n / tot:5.1f}% inst {100 * stall[key] / stot:5.1f}% smp  {key[0]}:{key[1]}: {src.get(key, '')[:100]}")
