#!/usr/bin/env python
"""Aggregate scripts/ncu_counters.sh CSVs into profiles/traffic_r02.json:
per config, per bench stage group, counters per launch of the group's
dominant kernel (the unit bench.py's roofline divides by)."""
import collections
import csv
import json
import os
import re
import sys

GROUPS = [("blend_backward", r"blend_backward"), ("blend_forward", r"blend_forward"),
          ("convert_project", r"mesh_to_splats"),
          ("face_vertex_backward", r"face_views_backward|face_convert_backward|vertex_gather"),
          ("binning", r".")]
KEYS = {"gpu__time_duration.sum": "ns", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "smsp__inst_executed.sum": "warp_instructions",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
        "smsp__thread_inst_executed_per_inst_executed.ratio": "lanes_per_instr",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
out = {}
for path in sys.argv[1:]:
    cfg = re.search(r"ncu_counters_(\w+)\.csv", path).group(1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[1:]:
        kid, name, metric = r[ix["ID"]], r[ix["Kernel Name"]], r[ix["Metric Name"]]
        if metric not in KEYS:
            continue
        val = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1)
        per[(int(kid), name)][KEYS[metric]] = val
    # whole calls only: from the first K1 launch to the last vertex gather
    ids = sorted(per)
    first = next(i for i, (k, n) in enumerate(ids) if "mesh_to_splats" in n)
    last = max(i for i, (k, n) in enumerate(ids) if "vertex_gather" in n)
    per = {k: per[k] for k in ids[first:last + 1]}
    steps = sum(1 for (_, n) in per if "blend_forward" in n) or 1
    agg = {}
    for (kid, name), m in per.items():
        grp = next(g for g, rx in GROUPS if re.search(rx, name))
        a = agg.setdefault(grp, collections.defaultdict(float))
        for k in ("ns", "dram_read", "dram_write", "warp_instructions", "smem_wavefronts"):
            a[k] += m.get(k, 0.0) / steps
        a["launches"] += 1 / steps
        if m.get("lanes_per_instr"):
            a["_lanes_w"] += m["lanes_per_instr"] * m.get("warp_instructions", 0.0) / steps
    res = {"source": "profiles/traffic_r02.json from `ncu --metrics ... --clock-control none` of bench.py "
                     f"--config {cfg} (whole steady-state calls; counters per call of the stage group)"}
    for grp, a in agg.items():
        res[grp] = {"dram_bytes": int(a["dram_read"] + a["dram_write"]), "dram_read": int(a["dram_read"]),
                    "dram_write": int(a["dram_write"]), "warp_instructions": int(a["warp_instructions"]),
                    "smem_wavefronts": int(a["smem_wavefronts"]), "ncu_us_per_call": round(a["ns"] / 1e3, 2),
                    "launches_per_call": round(a["launches"], 2),
                    "lanes_per_instr": round(a["_lanes_w"] / a["warp_instructions"], 2) if a["warp_instructions"] else None}
    out[cfg] = res
prev = {}
if os.path.exists("profiles/traffic_r02.json"):
    prev = json.load(open("profiles/traffic_r02.json"))
prev.update(out)
print(json.dumps(prev, indent=1))
