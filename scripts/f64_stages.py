"""Config 3 in float64 (render_mesh's default dtype): ms per 8-view step and
the per-stage split (profiling helper)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_14493_b200 as gmr  # noqa: E402
from paper_2602_14493_b200 import engine, lib  # noqa: E402

dt = torch.float64 if (len(sys.argv) < 2 or sys.argv[1] == "f64") else torch.float32
m = gmr.make_geodesic_sphere(158, seed=0)
cams = gmr.hemisphere_cameras(8, 3.0, (800, 800))
dev = torch.device("cuda", 0)
pos = torch.tensor(np.asarray(m.vertices), dtype=dt, device=dev)
col = torch.tensor(np.asarray(m.colors), dtype=dt, device=dev)
faces = torch.tensor(np.asarray(m.facets), dtype=torch.int32, device=dev)
g = torch.randn((8, 800, 800, 3), dtype=dt, device=dev)
ga = torch.randn((8, 800, 800), dtype=dt, device=dev)
L = lib.load()


def step():
    rgb, a, st = engine.render_forward(pos, col, faces, cams, 800, 800, (0.1, 0.1, 0.1), check=False)
    engine.render_backward(st, pos, col, faces, rgb, g, ga)
    return st


for _ in range(4):
    engine.check_status(step())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sts = [step() for _ in range(10)]
e1.record()
torch.cuda.synchronize()
print(f"{dt}: {e0.elapsed_time(e1) / 10:.3f} ms per 8-view step, {8000 / (e0.elapsed_time(e1) / 10):.0f} views/s")
L.gmr_timing_enable(1)
for _ in range(5):
    step()
torch.cuda.synchronize()
ms = (ctypes.c_double * 16)()
launches = (ctypes.c_int64 * 16)()
L.gmr_timing_read(ms, launches, len(lib.STAGES), 1)
print({s: round(ms[i] / 5, 4) for i, s in enumerate(lib.STAGES)})
