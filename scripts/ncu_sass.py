#!/usr/bin/env python
"""Top SASS instructions of a kernel in an ncu report by a metric column:
python scripts/ncu_sass.py REPORT KERNEL_REGEX "L1 Wavefronts Shared" [top]"""
import csv, io, subprocess, sys
rep, kern, col = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows:
    if len(r) == len(hdr) and r[0].startswith("0x"):
        try:
            v = float(r[ix[col]] or 0)
        except ValueError:
            continue
        data.append((v, r[ix["Address"]][-5:], r[ix["Source"]].strip(), r[ix["Instructions Executed"]],
                     r[ix.get("Avg. Threads Executed", 0)], r[ix["Warp Stall Sampling (All Samples)"]]))
tot = sum(d[0] for d in data) or 1
print(f"total {col}: {tot:.4g}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100*d[0]/tot:5.1f}%  {d[1]}  {d[2][:60]:60s} inst {d[3]:>10} lanes {d[4]:>5} stall {d[5]}")
