#!/usr/bin/env python
"""Split a kernel's ncu source-page counters into phases by source line:
python scripts/ncu_phases.py REPORT KERNEL_REGEX 'name:file:lo-hi,...'
Lines not covered by any range are reported as 'other' (top few listed)."""
import csv, io, subprocess, sys, collections
rep, kern, spec = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for part in spec.split(","):
    name, f, lh = part.split(":")
    lo, hi = (int(x) for x in lh.split("-"))
    ranges.append((name, f, lo, hi))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname = None, ""
acc = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
other = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
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
        v = (num("Instructions Executed"), num("Warp Stall Sampling (All Samples)"), num("L1 Wavefronts Shared"))
        ln = int(r[0])
        key = None
        for name, f, lo, hi in ranges:
            if fname.startswith(f) and lo <= ln <= hi:
                key = name
                break
        tgt = acc[key] if key else other[(fname, ln, r[1].strip()[:60])]
        for i in range(3):
            tgt[i] += v[i]
        if not key:
            for i in range(3):
                acc["other"][i] += v[i]
tot = [sum(v[i] for v in acc.values()) or 1 for i in range(3)]
print(f"total warp instr {tot[0]:.4g}  stall samples {tot[1]:.4g}  smem wavefronts {tot[2]:.4g}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:12s} instr {100*v[0]/tot[0]:5.1f}%  stall {100*v[1]/tot[1]:5.1f}%  smem {100*v[2]/tot[2]:5.1f}%")
print("top 'other' lines:")
for k, v in sorted(other.items(), key=lambda kv: -kv[1][0])[:12]:
    print(f"  {k[0]}:{k[1]} instr {100*v[0]/tot[0]:4.1f}% stall {100*v[1]/tot[1]:4.1f}% | {k[2]}")
