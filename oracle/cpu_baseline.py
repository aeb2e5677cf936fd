"""CPU baseline timing of the reference render path — BENCH INFRASTRUCTURE ONLY.

Times the reference's own fwd+bwd (`render_mesh(..., dtype=float32,
return_ctx=True)` + `render_backward`, meshsplat render.py:441-467) on the
host cores, for bench.py's `cpu_baseline` field and its `--impl reference`
arm.  Implementation timed, in order of preference:
* "reference": the real meshsplat package installed in baseline/_ref
  (`pip install --target baseline/_ref`, git-ignored, shipped to the GPU box);
* "port": the pinned numpy restatement oracle/gmr_oracle.py (its fp32 C3 view
  takes 29.1 s here against 30.1 s for the real reference).

No sampling and no extrapolation of work: a view is split into `bands`
horizontal bands of whole tile rows, and each band is rendered by the
reference itself through a crop camera (same pose and focal lengths,
principal point shifted by the band's first row, band height) on the facets
whose projected 3-sigma footprint can reach the band (a conservative float64
pre-selection with a 2-pixel margin, made outside the timed region; the
reference's own culling does the rest).  The bands of a view partition its
pixels, tiles, entries and blend work, so `bands` band renders are one view
of work, with only the facets straddling band edges projected twice.

P persistent worker processes (one per host core, OPENBLAS_NUM_THREADS=1,
capped by free memory) each own one view (view p mod 8 of the config's
cameras).  In step s every worker renders band s mod `bands` of its view, so
all workers do comparable work in a step and `bands` consecutive steps are P
whole views.  Views processed = band renders / bands; views/s = that / the
summed step wall times.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "meshsplat"))


def _band_rows(height, bands):
    """Tile-row ranges [(y0, y1)) of `bands` contiguous bands covering the image."""
    rows = (height + 15) // 16
    cuts = np.linspace(0, rows, bands + 1).round().astype(int)
    return [(16 * a, min(height, 16 * b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _band_facets(vertices, facets, cam, y0, y1):
    """Facets whose float64 projected footprint (3-sigma radius, +2 px) can
    reach rows [y0, y1): a superset of what the reference keeps for the band."""
    from oracle import gmr_oracle as orc
    cloud = orc.facet_gaussians(vertices, facets, np.zeros_like(vertices))
    s = orc.project(cloud, cam, np.float64)
    my, r = s.mean2d[:, 1], s.radius
    ok = (my + r + 2.0 >= y0 - 0.5) & (my - r - 2.0 <= y1 - 0.5)
    return np.sort(np.asarray(s.source)[ok])


def _worker(conn, impl, vertices, facets, colors, cam, background, bands, seed):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    T = time.perf_counter
    rng = np.random.default_rng(seed)
    H, W = cam.height, cam.width
    g_rgb = rng.normal(size=(H, W, 3)).astype(np.float32)
    g_a = rng.normal(size=(H, W)).astype(np.float32)
    bg = np.asarray(background, np.float64)
    if impl == "reference":
        sys.path.insert(0, REF_DIR)
        import meshsplat as ms

        def make_cam(c, y0, h):
            return ms.Camera(rotation=c.rotation, translation=c.translation, fx=c.fx, fy=c.fy, cx=c.cx,
                             cy=c.cy - y0, width=c.width, height=h, near=c.near, far=c.far)

        def run(mesh, c, gr, ga):
            o, ctx = ms.render_mesh(mesh, c, background=bg, dtype=np.float32, return_ctx=True)
            ms.render_backward(ctx, gr, ga)

        def make_mesh(f):
            return ms.TriangleMesh(vertices, f, colors)
    else:
        from oracle import gmr_oracle as orc
        from paper_2602_14493_b200.camera import Camera

        def make_cam(c, y0, h):
            return Camera(rotation=c.rotation, translation=c.translation, fx=c.fx, fy=c.fy, cx=c.cx,
                          cy=c.cy - y0, width=c.width, height=h, near=c.near, far=c.far)

        def run(mesh, c, gr, ga):
            _, _, ctx = orc.render(mesh[0], mesh[1], mesh[2], c, bg, True, np.float32)
            orc.render_grad(ctx, gr, ga)

        def make_mesh(f):
            return (vertices, f, colors)
    # per band: the crop camera, the facet subset as the caller's mesh, the
    # band's upstream gradients (all prepared outside the timed region)
    work = []
    for y0, y1 in _band_rows(H, bands):
        work.append((make_mesh(facets[_band_facets(vertices, facets, cam, y0, y1)]), make_cam(cam, y0, y1 - y0),
                     np.ascontiguousarray(g_rgb[y0:y1]), np.ascontiguousarray(g_a[y0:y1])))
    full = make_mesh(facets)
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        kind, b = msg
        t0 = T()
        if kind == "band":
            run(*work[b % len(work)])
        else:   # one full unsampled view, for the record
            run(full, cam, g_rgb, g_a)
        conn.send(T() - t0)


def default_processes(mem_per_proc_gb=3.0):
    procs = len(os.sched_getaffinity(0))
    try:
        import psutil
        procs = min(procs, max(1, int(psutil.virtual_memory().available / 2 ** 30 / mem_per_proc_gb)))
    except Exception:
        pass
    return max(1, procs)


class BandWorkers:
    """P persistent processes timing band renders of the reference."""

    def __init__(self, vertices, facets, colors, cams, background, bands=10, processes=None, impl=None):
        import multiprocessing as mp
        self.impl = impl or ("reference" if reference_available() else "port")
        self.bands = bands
        self.procs = processes or default_processes()
        ctx = mp.get_context("spawn")
        env = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in env:
            os.environ[k] = "1"
        self.conns, self.ps = [], []
        try:
            for i in range(self.procs):
                a, b = ctx.Pipe()
                p = ctx.Process(target=_worker, args=(b, self.impl, np.asarray(vertices), np.asarray(facets),
                                                      np.asarray(colors), cams[i % len(cams)],
                                                      np.asarray(background), bands, i), daemon=True)
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
        self.band_renders = 0
        self.wall = 0.0
        self.last = []

    def step(self, band):
        """Every worker renders band `band` of its view; returns the step's wall time."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(("band", band))
        self.last = [c.recv() for c in self.conns]
        dt = time.perf_counter() - t0
        self.band_renders += self.procs
        self.wall += dt
        return dt

    def views_per_s(self):
        return (self.band_renders / self.bands) / self.wall if self.wall else 0.0

    def full_view(self):
        """Every worker renders its whole view once; (wall s, per-process s)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(("full", 0))
        per = [c.recv() for c in self.conns]
        return time.perf_counter() - t0, per

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.ps:
            p.join(timeout=10)
