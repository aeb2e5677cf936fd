"""Stress the blend kernels' control paths against the oracle (float64):
dynamic batch cuts (huge splats covering whole tiles), early termination
inside a batch (stacks of opaque splats), partial tiles, multi-view batches
(one device call == sum of single-view reference calls) and determinism."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def _splat_scene(rng, k, lo, hi, cov_scale, opacity, W, H):
    mean2d = rng.uniform(lo, hi, size=(k, 2))
    cov = []
    for _ in range(k):
        a = rng.normal(size=(2, 2))
        cov.append(a @ a.T * cov_scale + np.eye(2) * 0.5)
    return dict(mean2d=mean2d, cov2d=np.array(cov), depth=rng.uniform(1, 5, size=k),
                color=rng.random((k, 3)), opacity=np.full(k, opacity) if np.isscalar(opacity) else opacity,
                source=np.arange(k), g_rgb=rng.normal(size=(H, W, 3)), g_alpha=rng.normal(size=(H, W)))


def _check_splats(gmr, case, W, H, bg=(0.2, 0.1, 0.3)):
    from paper_2602_14493_b200.camera import Camera
    cam = Camera(rotation=np.eye(3), translation=np.zeros(3), fx=40, fy=40, cx=W / 2, cy=H / 2, width=W, height=H)
    s = orc.splats_from_arrays(case["mean2d"], case["cov2d"], case["depth"], case["color"], case["opacity"])
    rgb, alpha = orc.composite(s, W, H, bg)
    gm, gcv, gcol, gop = orc.composite_backward(s, W, H, bg, case["g_rgb"], case["g_alpha"])
    sp = [gmr.Splat2D(m, c, float(d), col, float(o), int(i)) for m, c, d, col, o, i in
          zip(case["mean2d"], case["cov2d"], case["depth"], case["color"], case["opacity"], case["source"])]
    out = gmr.rasterize(sp, cam, bg)
    assert np.abs(out.rgb - rgb).max() <= 1e-10
    assert np.abs(out.alpha - alpha).max() <= 1e-10
    g = gmr.rasterize_backward(sp, cam, out, case["g_rgb"], case["g_alpha"])
    for a, b in zip(g, (gm, gcv, gcol, gop)):
        assert rel(a, b) <= 1e-8


def test_huge_splats_force_batch_cuts(gmr):
    """Splats covering whole tiles: a staged batch's coverage records exceed
    shared memory, so the backward takes fewer entries per batch."""
    rng = np.random.default_rng(1)
    case = _splat_scene(rng, 40, 4, 44, 60.0, rng.uniform(0.02, 0.2, 40), 48, 40)
    _check_splats(gmr, case, 48, 40)


def test_opaque_stacks_terminate_inside_batches(gmr):
    """60 nearly opaque splats stacked on a few pixels: transmittance drops
    below 1e-4 mid-list, later entries are skipped and the tail of the tile
    list never loads (zero partials)."""
    rng = np.random.default_rng(2)
    k = 300
    case = _splat_scene(rng, k, 10, 22, 1.0, 0.97, 32, 32)
    case["mean2d"][:60] = 16.0 + rng.normal(scale=0.3, size=(60, 2))
    _check_splats(gmr, case, 32, 32)


def test_many_low_opacity_layers(gmr):
    rng = np.random.default_rng(3)
    case = _splat_scene(rng, 500, 2, 30, 3.0, 0.05, 32, 32)
    _check_splats(gmr, case, 32, 32)


def test_batched_views_equal_sum_of_single_views(gmr):
    """One device call over 5 views == the reference's serial view loop."""
    from paper_2602_14493_b200 import engine
    import torch
    case = gc.c1_case()
    mesh = gmr.TriangleMesh(case["vertices"], case["facets"], case["colors"])
    cams = gmr.hemisphere_cameras(5, 2.6, (64, 48))
    rng = np.random.default_rng(4)
    g_rgb = rng.normal(size=(5, 48, 64, 3))
    g_a = rng.normal(size=(5, 48, 64))
    pos, col, faces = gmr.api._device_mesh(mesh, np.float64)
    rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 64, 48, (0.1, 0.2, 0.3))
    gp, gcol = engine.render_backward(st, pos, col, faces, rgb, torch.as_tensor(g_rgb).cuda(),
                                      torch.as_tensor(g_a).cuda())
    ogv = np.zeros_like(mesh.vertices)
    ogc = np.zeros_like(mesh.vertices)
    for v, cam in enumerate(cams):
        r, a, ctx = orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, (0.1, 0.2, 0.3))
        assert np.abs(rgb[v].cpu().numpy() - r).max() <= 1e-10
        x, y = orc.render_grad(ctx, g_rgb[v], g_a[v])
        ogv += x
        ogc += y
    assert rel(gp.cpu().numpy(), ogv) <= 1e-8
    assert rel(gcol.cpu().numpy(), ogc) <= 1e-8


def test_backward_is_bit_deterministic_f32(gmr):
    from paper_2602_14493_b200 import engine, make_geodesic_sphere, hemisphere_cameras
    import torch
    m = make_geodesic_sphere(20, seed=2)
    cams = hemisphere_cameras(3, 3.0, (160, 120))
    pos, col, faces = gmr.api._device_mesh(m, np.float32)
    g = torch.randn((3, 120, 160, 3), device="cuda")
    ga = torch.randn((3, 120, 160), device="cuda")
    outs = []
    for _ in range(3):
        rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 160, 120, (0.1, 0.1, 0.1))
        outs.append([x.cpu().numpy() for x in (rgb, alpha) + engine.render_backward(st, pos, col, faces, rgb, g, ga)])
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            np.testing.assert_array_equal(a, b)


def test_sharded_image_loss_gpu_local_fn(gmr):
    """dist.sharded_image_loss with the GPU local_fn (world size 1) == the
    reference's total_loss image terms (golden)."""
    from paper_2602_14493_b200 import dist
    case, g = gc.loss_case(), gc.load("loss_octa_3views_16")
    mesh = gmr.TriangleMesh(case["vertices"], case["facets"], case["colors"])
    fn = dist.gpu_local_image_loss(mesh, background=case["background"], dtype=np.float64)
    c, s, gp, gcol = dist.sharded_image_loss(fn, case["cameras"], case["target_rgb"], case["target_mask"],
                                            len(case["vertices"]), device="cuda")
    assert c == pytest.approx(float(g["color"]), rel=1e-10)
    assert s == pytest.approx(float(g["silhouette"]), rel=1e-10)
    assert rel(gp.cpu().numpy(), g["grad_v"]) <= 1e-8
    assert rel(gcol.cpu().numpy(), g["grad_c"]) <= 1e-8


def test_unreachable_tile_culling_paths_against_oracle(gmr):
    """Splats whose 3-sigma rectangle exceeds 32 tiles (no mask), and thin
    diagonal splats whose rectangles have many unreachable tiles (mask path):
    both must equal the reference semantics exactly (float64)."""
    rng = np.random.default_rng(7)
    W, H = 160, 120
    k_big, k_thin = 12, 60
    mean = np.concatenate([rng.uniform(20, 140, size=(k_big, 2)), rng.uniform(10, 150, size=(k_thin, 2))])
    covs = []
    for _ in range(k_big):
        a = rng.normal(size=(2, 2))
        covs.append(a @ a.T * 300.0 + np.eye(2) * 80.0)
    for _ in range(k_thin):
        th = rng.uniform(0, np.pi)
        R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        covs.append(R @ np.diag([rng.uniform(30, 120), 0.3]) @ R.T)
    k = k_big + k_thin
    case = dict(mean2d=mean, cov2d=np.array(covs), depth=rng.uniform(1, 5, size=k), color=rng.random((k, 3)),
                opacity=rng.uniform(0.05, 0.9, size=k), source=np.arange(k),
                g_rgb=rng.normal(size=(H, W, 3)), g_alpha=rng.normal(size=(H, W)))
    _check_splats(gmr, case, W, H)


@pytest.mark.parametrize("W,H", [(1, 37), (53, 1), (1, 1)])
def test_one_pixel_wide_images(gmr, W, H):
    from paper_2602_14493_b200.camera import Camera
    m = gmr.make_icosphere(80)
    f = 3.0 * max(W, H)
    cam = Camera(rotation=np.eye(3), translation=np.array([0.0, 0.0, 3.0]), fx=f, fy=f,
                 cx=(W - 1) / 2, cy=(H - 1) / 2, width=W, height=H)
    out, ctx = gmr.render_mesh(m, cam, background=(0.3, 0.2, 0.1), return_ctx=True)
    r, a, octx = orc.render(m.vertices, m.facets, m.colors, cam, (0.3, 0.2, 0.1))
    assert np.abs(out.rgb - r).max() <= 1e-10 and np.abs(out.alpha - a).max() <= 1e-10
    rng = np.random.default_rng(0)
    g_rgb, g_a = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W))
    gv, gc = gmr.render_backward(ctx, g_rgb, g_a)
    ogv, ogc = orc.render_grad(octx, g_rgb, g_a)
    assert rel(gv, ogv) <= 1e-8 and rel(gc, ogc) <= 1e-8


@pytest.mark.parametrize("k", [700, 1500, 3000])
def test_large_bins_depth_order(gmr, k):
    """Thousands of splats in one 16x16 tile, depths with many ties: the
    per-tile depth sort (GMR_FLAG_TILE_DEPTH_SORT) runs in shared memory
    (k <= 2048 f32 / 1024 f64) or through global scratch (larger bins); the
    default is the global depth sort.  Both must give the same lists, every
    bin in (depth, source) order (render.py:227), and the f64
    render/backward must match the oracle."""
    from paper_2602_14493_b200 import api, engine
    from paper_2602_14493_b200.camera import Camera
    rng = np.random.default_rng(10 + k)
    W = H = 16
    case = _splat_scene(rng, k, 3, 13, 1.5, rng.uniform(0.004, 0.012, k), W, H)
    case["depth"] = 1.0 + rng.integers(0, 40, k) / 10.0
    cam = Camera(rotation=np.eye(3), translation=np.zeros(3), fx=40, fy=40, cx=W / 2, cy=H / 2, width=W, height=H)
    sp = [gmr.Splat2D(m, c, float(d), col, float(o), int(i)) for m, c, d, col, o, i in
          zip(case["mean2d"], case["cov2d"], case["depth"], case["color"], case["opacity"], case["source"])]
    from paper_2602_14493_b200 import lib
    modes = []
    old = engine.DEFAULT_FLAGS
    engine.AUTO_TILE_ORDER = False
    try:
        for dtype in (np.float32, np.float64):
            for mode in (0, lib.FLAG_TILE_DEPTH_SORT):
                engine.DEFAULT_FLAGS = mode
                t, order, _, _, state = api._raster_device(sp, cam, (0.2, 0.1, 0.3), dtype)
                assert state.raster.flags & lib.FLAG_TILE_DEPTH_SORT == mode
                items, bounds = engine.copy_entries(state, k, False)
                modes.append((dtype, order, items.cpu().numpy().astype(np.int64), bounds.cpu().numpy()))
    finally:
        engine.DEFAULT_FLAGS = old
        engine.AUTO_TILE_ORDER = True
    for (dtype, order, items, bounds), other in zip(modes, modes[1:] + modes[:1]):
        if other[0] == dtype:
            np.testing.assert_array_equal(items, other[2])
        assert bounds[-1] == len(items) and bounds[1] - bounds[0] > 0.9 * k
        d = np.asarray(case["depth"], dtype)[order][items]
        for g in range(len(bounds) - 1):
            dd, ii = d[bounds[g]:bounds[g + 1]], items[bounds[g]:bounds[g + 1]]
            ok = (dd[1:] > dd[:-1]) | ((dd[1:] == dd[:-1]) & (ii[1:] > ii[:-1]))
            assert ok.all(), (dtype, g)
    _check_splats(gmr, case, W, H)


_PDL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2602_14493_b200 as gmr
from paper_2602_14493_b200 import engine
m = gmr.make_geodesic_sphere(20, seed=0)
cams = gmr.hemisphere_cameras(3, 3.0, (96, 80))
dev = torch.device("cuda", 0)
pos = torch.tensor(np.asarray(m.vertices), dtype=torch.float32, device=dev)
col = torch.tensor(np.asarray(m.colors), dtype=torch.float32, device=dev)
faces = torch.tensor(np.asarray(m.facets), dtype=torch.int32, device=dev)
g = torch.randn((3, 80, 96, 3), generator=torch.Generator(device=dev).manual_seed(0), device=dev)
ga = torch.randn((3, 80, 96), generator=torch.Generator(device=dev).manual_seed(1), device=dev)
outs = []
for _ in range(3):   # global depth order first, then per-tile lists
    rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 96, 80, (0.1, 0.2, 0.3))
    gp, gc = engine.render_backward(st, pos, col, faces, rgb, g, ga)
    torch.cuda.synchronize()
    outs += [rgb.cpu().numpy(), alpha.cpu().numpy(), gp.cpu().numpy(), gc.cpu().numpy()]
np.savez(sys.argv[2], *outs)
"""


def test_programmatic_launch_is_bit_identical(gmr, tmp_path):
    """Every kernel waits for its predecessor (griddepcontrol.wait) before
    touching memory, so launching with programmatic stream serialization
    (default) and without it (GMR_PDL=0) gives the same bits."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "pdl.py"
    script.write_text(_PDL_SCRIPT)
    res = {}
    for flag in ("1", "0"):
        out = tmp_path / f"out{flag}.npz"
        env = dict(os.environ, GMR_PDL=flag)
        r = subprocess.run([sys.executable, str(script), root, str(out)], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[flag] = np.load(out)
    for k in res["1"].files:
        assert np.array_equal(res["1"][k], res["0"][k]), k
