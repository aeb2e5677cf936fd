"""Exact (pixel, splat) pair counts of the config-3 bench step (8 views,
800x800), from the pinned oracle in float32: for every tile entry of the
reference's _RasterPlan lists (render.py:200-229), how many of the tile's
pixels see alpha >= 1/255 (render.py:251-257), and how many of those pairs
are included (transmittance stop not reached, render.py:260-261).
Infrastructure for profiles/pair_sol (it imports the oracle; it is never
run by the product).  Writes pairs_c3.json next to this file."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2602_14493_b200 as gmr  # noqa: E402  (mesh/camera builders only: no GPU)
from oracle import gmr_oracle as orc  # noqa: E402

m = gmr.make_geodesic_sphere(158, seed=0)
cams = gmr.hemisphere_cameras(8, 3.0, (800, 800))
cloud = orc.facet_gaussians(m.vertices, m.facets, np.asarray(m.colors))
yy, xx = np.mgrid[0:16, 0:16]
out = {"views": []}
for vi, cam in enumerate(cams):
    s = orc.project(cloud, cam, np.float32)
    entry, bounds = orc.bin_splats(s.mean2d, s.radius, s.depth, s.source, 800, 800)
    mean = s.mean2d.astype(np.float32)
    conic = s.conic.astype(np.float32)
    vis = inc = 0
    covered_px = 0
    for t in range(2500):
        lo, hi = bounds[t], bounds[t + 1]
        if hi == lo:
            continue
        ty, tx = divmod(t, 50)
        ids = entry[lo:hi]
        px = (tx * 16 + xx).ravel().astype(np.float32)
        py = (ty * 16 + yy).ravel().astype(np.float32)
        dx = px[None, :] - mean[ids, 0:1]
        dy = py[None, :] - mean[ids, 1:2]
        a, b, c = conic[ids, 0:1], conic[ids, 1:2], conic[ids, 2:3]
        power = np.float32(-0.5) * (a * dx * dx + c * dy * dy) - b * dx * dy
        al = np.minimum(np.float32(0.99), np.exp(power))
        v = al >= np.float32(1 / 255)
        vis += int(v.sum())
        covered_px += int(v.any(0).sum())
        # transmittance before each pair; a pair is included while T (1 - alpha) >= 1e-4
        om = np.where(v, 1 - al, 1).astype(np.float32)
        T = np.cumprod(om, axis=0)
        inc += int((v & (T >= np.float32(1e-4))).sum())
    out["views"].append({"entries": int(len(entry)), "visible_pairs": vis, "included_pairs": inc,
                         "covered_pixels": covered_px})
    print(vi, out["views"][-1], flush=True)
out["visible_pairs_per_step"] = sum(v["visible_pairs"] for v in out["views"])
out["included_pairs_per_step"] = sum(v["included_pairs"] for v in out["views"])
out["entries_per_step"] = sum(v["entries"] for v in out["views"])
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "pairs_c3.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "views"}))
