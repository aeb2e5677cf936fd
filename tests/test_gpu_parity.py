"""Parity of the CUDA path (through the C ABI) with the reference.

Oracles: the golden fixtures produced by the reference itself
(tests/golden/make_golden.py) and the pinned CPU restatement
(oracle/gmr_oracle.py) on fresh seeded inputs.

Tolerances (stated here, used below):
* float64 path: images max-abs <= 1e-10, vertex/colour gradients relative
  (max|a-b| / max(1, max|b|)) <= 1e-8; tile entries bit-exact.
* float32 path vs the reference's float32 path: images max-abs <= 1e-4 and
  gradients relative <= 1e-3 (BASELINE north star), except at decision
  flips (alpha vs 1/255, transmittance vs 1e-4, the 0.99 clamp) where fp32
  rounding legitimately differs; flipped pixels are counted and bounded.
* binning: bit-exact given the kernel's own projected splats.
"""

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max())) if a.size else 0.0


def _mesh(case):
    from paper_2602_14493_b200 import TriangleMesh
    return TriangleMesh(case["vertices"], case["facets"], case["colors"])


RENDER_CASES = [("c1_icosphere1280_128", gc.c1_case), ("octahedron_32", gc.octahedron_case),
                ("icosphere320_64x48", gc.small_render_case)]


@pytest.mark.parametrize("name,maker", RENDER_CASES)
def test_render_f64_matches_reference(gmr, name, maker):
    case, g = maker(), gc.load(name)
    mesh = _mesh(case)
    out, ctx = gmr.render_mesh(mesh, case["camera"], background=case["background"], dtype=np.float64,
                               return_ctx=True)
    assert out.rgb.dtype == np.float64
    assert np.abs(out.rgb - g["f64_rgb"]).max() <= 1e-10
    assert np.abs(out.alpha - g["f64_alpha"]).max() <= 1e-10
    gv, gcol = gmr.render_backward(ctx, case["g_rgb"], case["g_alpha"])
    assert gv.dtype == np.float64 and gv.shape == g["f64_grad_v"].shape
    assert rel(gv, g["f64_grad_v"]) <= 1e-8
    assert rel(gcol, g["f64_grad_c"]) <= 1e-8
    # tile lists: bit-exact (face ids in (tile, depth, source) order + bounds)
    # with the reference's full _RasterPlan lists
    from paper_2602_14493_b200 import engine, lib
    old = engine.DEFAULT_FLAGS
    engine.DEFAULT_FLAGS = lib.FLAG_FULL_TILE_LISTS
    try:
        out_full, ctx_full = gmr.render_mesh(mesh, case["camera"], background=case["background"],
                                             dtype=np.float64, return_ctx=True)
        items, bounds = engine.copy_entries(ctx_full.state, len(mesh.facets), True)
    finally:
        engine.DEFAULT_FLAGS = old
    np.testing.assert_array_equal(items.cpu().numpy(), g["f64_entry_source"])
    np.testing.assert_array_equal(bounds.cpu().numpy(), g["f64_bounds"])
    # dropping unreachable tiles changes nothing
    np.testing.assert_array_equal(out_full.rgb, out.rgb)
    np.testing.assert_array_equal(out_full.alpha, out.alpha)


@pytest.mark.parametrize("name,maker", RENDER_CASES)
def test_render_f32_matches_reference(gmr, name, maker):
    case, g = maker(), gc.load(name)
    mesh = _mesh(case)
    out, ctx = gmr.render_mesh(mesh, case["camera"], background=case["background"], dtype=np.float32,
                               return_ctx=True)
    assert out.rgb.dtype == np.float32
    d = np.abs(out.rgb.astype(np.float64) - g["f32_rgb"]).max(axis=2)
    da = np.abs(out.alpha.astype(np.float64) - g["f32_alpha"])
    bad = (d > 1e-4) | (da > 1e-4)
    assert bad.sum() <= max(2, 1e-3 * bad.size), (bad.sum(), d.max())
    gv, gcol = gmr.render_backward(ctx, case["g_rgb"], case["g_alpha"])
    if bad.sum() == 0:
        assert rel(gv, g["f32_grad_v"]) <= 1e-3
        assert rel(gcol, g["f32_grad_c"]) <= 1e-3
    else:
        rl2 = np.linalg.norm(gv - g["f32_grad_v"]) / np.linalg.norm(g["f32_grad_v"])
        assert rl2 <= 1e-2


@pytest.mark.parametrize("tile_mode", [False, True])
@pytest.mark.parametrize("name,maker", RENDER_CASES)
def test_binning_bit_exact_f32(gmr, name, maker, tile_mode):
    """Feed the kernel's own fp32 (mean2d, radius, depth) of kept splats to the
    oracle's _RasterPlan restatement: entries and bounds must be identical
    (global and per-tile depth order)."""
    from paper_2602_14493_b200 import engine
    case = maker()
    mesh = _mesh(case)
    pos, col, faces = gmr.api._device_mesh(mesh, np.float32)
    cam = case["camera"]
    from paper_2602_14493_b200 import lib
    flags = lib.FLAG_DEBUG_AUX | lib.FLAG_FULL_TILE_LISTS | (lib.FLAG_TILE_DEPTH_SORT if tile_mode else 0)
    engine.AUTO_TILE_ORDER = False
    try:
        rgb, alpha, st = engine.render_forward(pos, col, faces, [cam], cam.width, cam.height,
                                               case["background"], flags=flags)
    finally:
        engine.AUTO_TILE_ORDER = True
    assert bool(st.raster.flags & lib.FLAG_TILE_DEPTH_SORT) == tile_mode
    rec, rect, cnt, aux = (x.cpu().numpy() for x in engine.copy_splats(st, len(mesh.facets), True))
    kept = np.where(cnt > 0)[0]
    mean2d = rec[kept, 0:2]
    radius, depth = aux[kept, 0], aux[kept, 1]
    # the kernel's depth + screen cull, recomputed in numpy fp32 on its own values
    w, h = np.float32(cam.width), np.float32(cam.height)
    r_all, z_all, m_all = aux[:, 0], aux[:, 1], rec[:, 0:2]
    with np.errstate(invalid="ignore"):
        on = (z_all > np.float32(cam.near)) & (z_all < np.float32(cam.far)) \
            & (m_all[:, 0] + r_all >= -0.5) & (m_all[:, 0] - r_all <= w - np.float32(0.5)) \
            & (m_all[:, 1] + r_all >= -0.5) & (m_all[:, 1] - r_all <= h - np.float32(0.5))
    np.testing.assert_array_equal(np.where(on)[0], kept)
    entry, bounds = orc.bin_splats(mean2d, radius, depth, kept, cam.width, cam.height)
    items, gbounds = engine.copy_entries(st, len(mesh.facets), True)
    np.testing.assert_array_equal(items.cpu().numpy(), kept[entry])
    np.testing.assert_array_equal(gbounds.cpu().numpy(), bounds)


@pytest.mark.parametrize("name,maker", [("splats7_32", gc.splat_case),
                                        ("splats_closed_form_32", gc.closed_form_splat_case)])
def test_rasterize_f64_matches_reference(gmr, name, maker):
    case, g = maker(), gc.load(name)
    sp = [gmr.Splat2D(mean2d=m, cov2d_screen=c, depth=float(d), color=col, opacity=float(o), source=int(s))
          for m, c, d, col, o, s in zip(case["mean2d"], case["cov2d"], case["depth"], case["color"],
                                         case["opacity"], case["source"])]
    cam = case["camera"]
    out = gmr.rasterize(sp[::-1], cam, case["background"])   # input order must not matter
    assert np.abs(out.rgb - g["rgb"]).max() <= 1e-12
    assert np.abs(out.alpha - g["alpha"]).max() <= 1e-12
    gm, gcv, gcol, gop = gmr.rasterize_backward(sp, cam, out, case["g_rgb"], case["g_alpha"])
    for a, k in ((gm, "g_mean2d"), (gcv, "g_cov2d"), (gcol, "g_color"), (gop, "g_opacity")):
        assert rel(a, g[k]) <= 1e-10, k


def test_closed_forms_f64(gmr):
    """reference test_render.py:167-189."""
    cam = gc.identity_camera()
    out = gmr.rasterize([], cam, background=(0.2, 0.4, 0.6))
    assert np.allclose(out.rgb, (0.2, 0.4, 0.6)) and np.all(out.alpha == 0)
    s = lambda m, c, d=1.0, o=1.0, src=-1: gmr.Splat2D(np.array(m, float), np.eye(2) * 2.0, d,
                                                       np.array(c, float), o, src)
    out = gmr.rasterize([s((16, 16), (1, 1, 1))], cam)
    assert out.rgb[16, 16] == pytest.approx([0.99] * 3, abs=1e-12)
    out = gmr.rasterize([s((16, 16), (0, 0, 1), 2.0, 1.0, 1), s((16, 16), (1, 0, 0), 1.0, 1.0, 0)], cam)
    assert out.rgb[16, 16, 0] == pytest.approx(0.99, abs=1e-12)
    assert out.rgb[16, 16, 2] == pytest.approx(0.01 * 0.99, abs=1e-12)
    assert out.alpha[16, 16] == pytest.approx(1 - 1e-4)
    with pytest.raises(ValueError, match="non-finite"):
        gmr.rasterize([s((16, np.nan), (1, 1, 1))], cam)


def test_total_loss_f64_matches_reference(gmr):
    case, g = gc.loss_case(), gc.load("loss_octa_3views_16")
    w = gmr.LossWeights(color=1.0, silhouette=1.0, edge=0.0, laplacian=0.0)
    rep, gv, gcol = gmr.total_loss(_mesh(case), case["cameras"], case["target_rgb"], case["target_mask"],
                                   weights=w, background=case["background"], dtype=np.float64)
    assert rep.color == pytest.approx(float(g["color"]), rel=1e-10)
    assert rep.silhouette == pytest.approx(float(g["silhouette"]), rel=1e-10)
    assert rel(gv, g["grad_v"]) <= 1e-8
    assert rel(gcol, g["grad_c"]) <= 1e-8


def test_convert_f64_matches_reference(gmr):
    case, g = gc.convert_case(), gc.load("convert_random50")
    mesh = _mesh(case)
    cloud = gmr.convert_mesh(mesh)
    np.testing.assert_array_equal(cloud.degenerate, g["degenerate"])
    assert np.abs(cloud.means - g["means"]).max() <= 1e-14
    assert np.abs(cloud.cov3d - g["cov3d"]).max() <= 1e-14
    gv, gcol = gmr.convert_backward(mesh, cloud, case["g_means"], case["g_cov3d"], case["g_colors"])
    assert rel(gv, g["grad_v"]) <= 1e-10
    assert rel(gcol, g["grad_c"]) <= 1e-12


def test_fresh_scene_f64_vs_oracle(gmr):
    """Fresh geodesic scene, non-square image with partial tiles."""
    from paper_2602_14493_b200 import default_intrinsics, look_at, make_geodesic_sphere
    m = make_geodesic_sphere(9, seed=5)
    cam = look_at((1.9, -1.7, 1.3), (0.05, 0, 0), **default_intrinsics(100, 72))
    rng = np.random.default_rng(17)
    g_rgb, g_a = rng.normal(size=(72, 100, 3)), rng.normal(size=(72, 100))
    bg = (0.3, 0.1, 0.2)
    rgb, alpha, octx = orc.render(m.vertices, m.facets, m.colors, cam, bg, True, np.float64)
    ogv, ogc = orc.render_grad(octx, g_rgb, g_a)
    out, ctx = gmr.render_mesh(m, cam, background=bg, return_ctx=True)
    assert np.abs(out.rgb - rgb).max() <= 1e-10
    gv, gcol = gmr.render_backward(ctx, g_rgb, g_a)
    assert rel(gv, ogv) <= 1e-8 and rel(gcol, ogc) <= 1e-8


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_unreachable_tile_culling_is_exact(gmr, dtype):
    """Default lists drop the tiles a splat's padded ellipse cannot reach:
    same images and gradients bit for bit as the reference's full lists,
    and every (tile, face) list is an order-preserving subsequence."""
    import torch
    from paper_2602_14493_b200 import engine, lib
    mesh = gmr.make_geodesic_sphere(40, seed=3)
    cams = gmr.hemisphere_cameras(3, 3.0, (200, 136))
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    pos = torch.tensor(mesh.vertices, dtype=tdt, device="cuda")
    col = torch.tensor(mesh.colors, dtype=tdt, device="cuda")
    faces = torch.tensor(mesh.facets, dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    g_rgb = torch.randn((3, 136, 200, 3), generator=g, device="cuda", dtype=tdt)
    g_a = torch.randn((3, 136, 200), generator=g, device="cuda", dtype=tdt)
    res = {}
    for name, flags in (("cull", 0), ("full", lib.FLAG_FULL_TILE_LISTS)):
        rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 200, 136, (0.1, 0.2, 0.3), flags=flags)
        gp, gc = engine.render_backward(st, pos, col, faces, rgb, g_rgb, g_a)
        items, bounds = engine.copy_entries(st, len(mesh.facets), True)
        res[name] = (rgb, alpha, gp, gc, items.cpu().numpy(), bounds.cpu().numpy(), st.entries)
    for k in range(4):
        assert torch.equal(res["cull"][k], res["full"][k]), k
    ic, bc, ec = res["cull"][4:]
    iff, bf, ef = res["full"][4:]
    assert ec < ef        # some tiles were dropped
    for t in range(len(bf) - 1):
        lc, lf = ic[bc[t]:bc[t + 1]], iff[bf[t]:bf[t + 1]]
        it = iter(lf)
        assert all(any(x == y for y in it) for x in lc), t   # subsequence


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("name,maker", RENDER_CASES)
def test_tile_depth_sort_mode_is_identical(gmr, name, maker, dtype):
    """GMR_FLAG_TILE_DEPTH_SORT (per-tile depth ordering after the tile sort)
    and the default global depth sort give the same (tile, depth, source)
    lists, hence bit-identical images and gradients; in f64 both equal the
    reference's _RasterPlan lists."""
    from paper_2602_14493_b200 import engine, lib
    case = maker()
    mesh = _mesh(case)
    res = []
    old = engine.DEFAULT_FLAGS
    engine.AUTO_TILE_ORDER = False
    try:
        for mode in (0, lib.FLAG_TILE_DEPTH_SORT):
            engine.DEFAULT_FLAGS = lib.FLAG_FULL_TILE_LISTS | mode
            out, ctx = gmr.render_mesh(mesh, case["camera"], background=case["background"], dtype=dtype,
                                       return_ctx=True)
            assert ctx.state.raster.flags & lib.FLAG_TILE_DEPTH_SORT == mode
            items, bounds = engine.copy_entries(ctx.state, len(mesh.facets), True)
            gv, gcol = gmr.render_backward(ctx, case["g_rgb"], case["g_alpha"])
            res.append((items.cpu().numpy(), bounds.cpu().numpy(), out.rgb, out.alpha, gv, gcol))
    finally:
        engine.DEFAULT_FLAGS = old
        engine.AUTO_TILE_ORDER = True
    for a, b in zip(res[0], res[1]):
        np.testing.assert_array_equal(a, b)
    if dtype == np.float64:
        g = gc.load(name)
        np.testing.assert_array_equal(res[1][0], g["f64_entry_source"])
        np.testing.assert_array_equal(res[1][1], g["f64_bounds"])


def test_tile_depth_sort_chosen_from_previous_call(gmr):
    """The engine switches a call shape to per-tile depth ordering once a
    previous forward of that shape reported only short tile lists, and back
    to the global depth sort when a list outgrows the shared-memory sort."""
    import torch
    from paper_2602_14493_b200 import engine, lib
    case = gc.c1_case()
    mesh = _mesh(case)
    engine._order.forget()   # earlier tests' calls of this shape
    flags = []
    for _ in range(3):
        _, ctx = gmr.render_mesh(mesh, case["camera"], background=case["background"], dtype=np.float32,
                                 return_ctx=True)
        torch.cuda.synchronize()
        flags.append(ctx.state.raster.flags & lib.FLAG_TILE_DEPTH_SORT)
    assert flags[0] == 0 and flags[-1] == lib.FLAG_TILE_DEPTH_SORT
    key = next(k for k in engine._order._shapes if k[0] == len(mesh.facets) and k[-1] == torch.float32)
    sh = engine._order._shapes[key]
    sh.pending, sh.last = False, 5000   # as if the last read-back had seen a 5000-entry list
    _, ctx = gmr.render_mesh(mesh, case["camera"], background=case["background"], dtype=np.float32,
                             return_ctx=True)
    assert ctx.state.raster.flags & lib.FLAG_TILE_DEPTH_SORT == 0
