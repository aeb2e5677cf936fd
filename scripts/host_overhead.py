"""Host-side cost of one config-1 step through the engine (profiling helper):
cProfile of 200 forward+backward calls, device work tiny."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_14493_b200 as gmr  # noqa: E402
from paper_2602_14493_b200 import engine  # noqa: E402

m = gmr.make_icosphere(1280)
mesh = gmr.TriangleMesh(m.vertices, m.facets, gmr.seeded_colors(m.num_vertices, 0))
cams = gmr.hemisphere_cameras(1, 3.0, (128, 128))
dev = torch.device("cuda", 0)
pos = torch.tensor(np.asarray(mesh.vertices), dtype=torch.float32, device=dev)
col = torch.tensor(np.asarray(mesh.colors), dtype=torch.float32, device=dev)
faces = torch.tensor(np.asarray(mesh.facets), dtype=torch.int32, device=dev)
g = torch.randn((1, 128, 128, 3), device=dev)
ga = torch.randn((1, 128, 128), device=dev)
pending = []


def step():
    rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 128, 128, (0.1, 0.1, 0.1), check=False)
    engine.render_backward(st, pos, col, faces, rgb, g, ga)
    pending.append(st)
    if len(pending) > 2:
        engine.check_status(pending.pop(0))


for _ in range(20):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host {1e6 * (t1 - t0) / 200:.1f} us/step, with drain {1e6 * (t2 - t0) / 200:.1f} us/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
