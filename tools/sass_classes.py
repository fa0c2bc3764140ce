#!/usr/bin/env python
"""Per-kernel instruction-class counts of libqadc_b200.so (cuobjdump -sass): which kernels use the 5th-generation
tensor cores (UTC*MMA = tcgen05.mma), tensor memory (LDTM / STTM = tcgen05.ld / st), TMA (UBLKCP = cp.async.bulk,
UTMALDG = cp.async.bulk.tensor), mbarriers (SYNCS) -- and that no legacy HMMA (mma.sync) is left.
usage: python tools/sass_classes.py [out.txt]   (runs on the CPU build box; no GPU needed)"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SO = ROOT / "paper_1812_09162_b200" / "libqadc_b200.so"
CLASSES = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "LDTM", "STTM", "UTCBAR", "UTMALDG", "UBLKCP", "SYNCS", "HMMA", "IMMA",
           "LDS.128", "LDS.64", "LDGSTS", "REDUX", "ATOMG", "RED."]


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True, check=True).stdout
    per = OrderedDict()
    cur = None
    arch = Counter()
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
            per.setdefault(cur, Counter())
            continue
        m = re.match(r"arch = (\S+)", line)
        if m:
            arch[m.group(1)] += 1
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
        if m and cur:
            op = m.group(1)
            per[cur]["_total"] += 1
            for c in CLASSES:
                if op.startswith(c):
                    per[cur][c] += 1
    lines = [f"# SASS instruction classes per kernel of {SO.name} ({', '.join(f'{k} x{v}' for k, v in arch.items())})",
             "# produced by tools/sass_classes.py (cuobjdump -sass); UTC*MMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st,",
             "# UBLKCP = cp.async.bulk (TMA 1-D bulk copy), SYNCS = mbarrier ops, HMMA = legacy mma.sync", ""]
    tot = Counter()
    hdr = f"{'kernel':78s} {'instrs':>7s} " + " ".join(f"{c:>7s}" for c in CLASSES)
    lines.append(hdr)
    for k, c in per.items():
        if not any(c[x] for x in CLASSES) and c["_total"] < 50:
            continue
        lines.append(f"{k[:78]:78s} {c['_total']:7d} " + " ".join(f"{c[x]:7d}" for x in CLASSES))
        tot.update(c)
    lines.append("")
    lines.append(f"{'TOTAL':78s} {tot['_total']:7d} " + " ".join(f"{tot[x]:7d}" for x in CLASSES))
    lines.append("")
    lines.append(f"tensor-core instructions: UTCIMMA {tot['UTCIMMA']} (scan_tc8_kernel: int8 one-hot scan), "
                 f"UTCHMMA {tot['UTCHMMA']} (probe_approx_umma_kernel: bf16 probe prefilter); legacy HMMA {tot['HMMA']}")
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(text)
    print(text)


if __name__ == "__main__":
    main()
