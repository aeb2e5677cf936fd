#!/usr/bin/env python
"""Per-CUDA-source-line summary of an ncu report's source page:
python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
fname = ""
lines = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 4 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] not in ("", "Line No"):
        d = dict(zip(hdr, r))
        def num(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        lines.append((fname, int(r[0]), r[1].strip()[:70], num("Instructions Executed"),
                      num("Warp Stall Sampling (All Samples)"), num("L1 Wavefronts Shared"),
                      num("Avg. Threads Executed")))
ti = sum(x[3] for x in lines) or 1
ts = sum(x[4] for x in lines) or 1
tw = sum(x[5] for x in lines) or 1
print(f"total warp instr {ti:.4g}  stall samples {ts:.4g}  smem wavefronts {tw:.4g}")
for x in sorted(lines, key=lambda x: -(x[3] / ti + x[4] / ts))[:top]:
    print(f"{x[0]}:{x[1]:5d} instr {100*x[3]/ti:5.1f}% stall {100*x[4]/ts:5.1f}% smem {100*x[5]/tw:5.1f}% lanes {x[6]:4.1f} | {x[2]}")
