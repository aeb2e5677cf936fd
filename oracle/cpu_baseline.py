"""CPU baseline timing of the reference algorithm — BENCH INFRASTRUCTURE ONLY.

Times the numpy restatement (oracle/gmr_oracle.py, pinned to the reference)
of fwd+bwd views, for bench.py's `cpu_baseline` field and its
`--impl reference` arm.  Views are independent, so P persistent worker
processes (one per host core, OPENBLAS_NUM_THREADS=1) each own one view and
run concurrently ("view-parallel" CPU number).

Bounded sample per step and view (extrapolated, then reported as such):
* per-face stages (convert, project, projection + conversion backward) run
  on every `face_stride`-th face; their time is scaled by face_stride;
* the binning (`_RasterPlan`, run twice per view by the reference) runs in
  full;
* the per-tile blend loops (forward and backward) run on every
  `tile_stride`-th tile; their time is scaled by T / T_sampled.
"""

from __future__ import annotations

import os
import time

import numpy as np


def _worker(conn, vertices, facets, colors, cam, background, dtype, seed):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import gmr_oracle as orc
    T = time.perf_counter
    rng = np.random.default_rng(seed)
    H, W = cam.height, cam.width
    g_rgb, g_a = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W))
    ntiles = ((W + 15) // 16) * ((H + 15) // 16)
    full = orc.project(orc.facet_gaussians(vertices, facets, colors), cam, dtype)
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        fstride, tstride = msg
        tiles = list(range(0, ntiles, tstride))
        sub = facets[::fstride]
        t0 = T()
        cloud = orc.facet_gaussians(vertices, sub, colors)
        s = orc.project(cloud, cam, dtype)
        m = len(sub)
        gm = rng.normal(size=(len(s), 2)).astype(dtype)
        gc = rng.normal(size=(len(s), 2, 2)).astype(dtype)
        a, b = orc.project_backward(s, cloud, cam, gm, gc + gc.transpose(0, 2, 1))
        G3, C3, CC = np.zeros((m, 3)), np.zeros((m, 3, 3)), np.zeros((m, 3))
        G3[s.source], C3[s.source] = a, b
        orc.facet_backward(vertices, sub, colors, G3, C3, CC)
        t1 = T()
        orc.bin_splats(full.mean2d, full.radius, full.depth, full.source, W, H)
        t2 = T()
        orc.composite(full, W, H, background, dtype, tiles=tiles)
        t3 = T()
        orc.composite_backward(full, W, H, background, g_rgb, g_a, dtype, tiles=tiles)
        t4 = T()
        t_bin = t2 - t1
        scale = ntiles / len(tiles)
        t_view = ((t1 - t0) * fstride + 2 * t_bin
                  + max(0.0, t3 - t2 - t_bin) * scale + max(0.0, t4 - t3 - t_bin) * scale)
        conn.send({"view_s": t_view, "sampled_s": t4 - t0, "bin_s": t_bin})


class ViewWorkers:
    """P persistent processes, each timing one view of the workload."""

    def __init__(self, vertices, facets, colors, cams, background, dtype=np.float32, processes=None):
        import multiprocessing as mp
        procs = processes or len(os.sched_getaffinity(0))
        self.procs = max(1, min(procs, len(cams)))
        env = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in env:
            os.environ[k] = "1"
        ctx = mp.get_context("spawn")
        self.conns, self.ps = [], []
        try:
            for i in range(self.procs):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b, np.asarray(vertices), np.asarray(facets),
                                                      np.asarray(colors), cams[i], np.asarray(background),
                                                      dtype, i), daemon=True)
                p.start()
                self.conns.append(a)
                self.ps.append(p)
        finally:
            for k, v in env.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self, face_stride=1, tile_stride=16):
        """One concurrent sample over all workers; returns (views/s, details)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send((face_stride, tile_stride))
        res = [c.recv() for c in self.conns]
        wall = time.perf_counter() - t0
        per_view = [r["view_s"] for r in res]
        return self.procs / max(per_view), {"per_view_s": float(np.mean(per_view)), "wall_s": wall,
                                            "bin_s": float(np.mean([r["bin_s"] for r in res]))}

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.ps:
            p.join(timeout=10)
