"""Config-5 fit loop: per-iteration time of the eager fast path vs graph
replay, and the device time of the loop (profiling helper, not a test)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import golden_cases as gc  # noqa: E402
import torch  # noqa: E402
import paper_2602_14493_b200 as gmr  # noqa: E402
from paper_2602_14493_b200 import fit as gfit  # noqa: E402

case, g = gc.fit_case(), gc.load("fit_c5_200")
init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
rgbs, masks = list(g["target_rgb"]), list(g["target_mask"])
cfg = gfit.FitConfig(iterations=200, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
for graphs in (False, True, False, True):
    res = gfit.fit(init, case["cameras"], rgbs, masks, cfg, graphs=graphs)
    print(f"graphs={graphs}: wall {1e3 * res.wall_time / 200:.4f} ms/it, loop {1e3 * res.loop_time / 200:.4f} ms/it, "
          f"final {res.history[-1]['total']:.6f}", flush=True)
