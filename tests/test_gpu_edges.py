"""Edge cases of the boundary and the binning pipeline (float64 vs oracle)."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def test_empty_mesh_renders_background(gmr):
    mesh = gmr.TriangleMesh(np.zeros((3, 3)), np.zeros((0, 3), int))
    cam = gc.identity_camera()
    out, ctx = gmr.render_mesh(mesh, cam, background=(0.2, 0.4, 0.6), return_ctx=True)
    assert np.allclose(out.rgb, (0.2, 0.4, 0.6)) and np.all(out.alpha == 0)
    gv, gcol = gmr.render_backward(ctx, np.ones((32, 32, 3)), np.ones((32, 32)))
    assert np.all(gv == 0) and np.all(gcol == 0)


def test_everything_culled(gmr):
    """reference test_render.py:433-440: mesh behind the camera."""
    m = gmr.make_icosphere(80)
    behind = m.with_vertices(np.asarray(m.vertices) + np.array([0, 0, -10.0]))
    cam = gmr.Camera(rotation=np.eye(3), translation=np.zeros(3), fx=40, fy=40, cx=15.5, cy=15.5, width=32, height=32)
    out, ctx = gmr.render_mesh(behind, cam, background=(0.1, 0.2, 0.3), return_ctx=True)
    assert np.allclose(out.rgb, (0.1, 0.2, 0.3)) and np.all(out.alpha == 0)
    gv, _ = gmr.render_backward(ctx, np.ones((32, 32, 3)), np.ones((32, 32)))
    assert np.all(gv == 0)


def test_many_views_one_call_chunks_cameras(gmr):
    """70 views (> 64 per K1/K5 launch) in one device call == serial reference loop."""
    import torch
    from paper_2602_14493_b200 import engine
    m = gmr.make_icosphere(80)
    mesh = gmr.TriangleMesh(m.vertices, m.facets, gmr.seeded_colors(m.num_vertices, 1))
    cams = gmr.sphere_views(70, 2.8, 24)
    rng = np.random.default_rng(9)
    g_rgb, g_a = rng.normal(size=(70, 24, 24, 3)), rng.normal(size=(70, 24, 24))
    pos, col, faces = gmr.api._device_mesh(mesh, np.float64)
    rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 24, 24, (0.1, 0.1, 0.1))
    gp, gcol = engine.render_backward(st, pos, col, faces, rgb, torch.as_tensor(g_rgb).cuda(),
                                      torch.as_tensor(g_a).cuda())
    ogv = np.zeros_like(mesh.vertices)
    for v in (0, 33, 64, 69):
        r, a, _ = orc.render(mesh.vertices, mesh.facets, mesh.colors, cams[v], (0.1, 0.1, 0.1))
        assert np.abs(rgb[v].cpu().numpy() - r).max() <= 1e-10
    for v, cam in enumerate(cams):
        r, a, ctx = orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, (0.1, 0.1, 0.1))
        ogv += orc.render_grad(ctx, g_rgb[v], g_a[v])[0]
    assert rel(gp.cpu().numpy(), ogv) <= 1e-8


def test_large_partial_tile_image(gmr):
    """Non-multiple-of-16 image (partial tiles on both edges), f64 vs oracle."""
    m = gmr.make_geodesic_sphere(6, seed=4)
    cam = gmr.look_at((0.2, -2.9, 0.7), (0, 0, 0), **gmr.default_intrinsics(301, 187))
    rng = np.random.default_rng(10)
    g_rgb, g_a = rng.normal(size=(187, 301, 3)), rng.normal(size=(187, 301))
    out, ctx = gmr.render_mesh(m, cam, background=(0.3, 0.3, 0.3), return_ctx=True)
    r, a, octx = orc.render(m.vertices, m.facets, m.colors, cam, (0.3, 0.3, 0.3))
    assert np.abs(out.rgb - r).max() <= 1e-10 and np.abs(out.alpha - a).max() <= 1e-10
    gv, gcol = gmr.render_backward(ctx, g_rgb, g_a)
    ogv, ogc = orc.render_grad(octx, g_rgb, g_a)
    assert rel(gv, ogv) <= 1e-8 and rel(gcol, ogc) <= 1e-8


def test_capacity_overflow_recovers(gmr):
    """A forward planned with too small an entry capacity reports the exact
    count; the engine re-plans and re-runs to the same result."""
    from paper_2602_14493_b200 import engine
    case = gc.c1_case()
    mesh = gmr.TriangleMesh(case["vertices"], case["facets"], case["colors"])
    pos, col, faces = gmr.api._device_mesh(mesh, np.float64)
    cam = case["camera"]
    key = (len(mesh.facets), 1, 128, 128, pos.dtype)
    from paper_2602_14493_b200 import lib
    for flags, expect in ((lib.FLAG_FULL_TILE_LISTS, 5997), (0, None)):
        ref, _, st0 = engine.render_forward(pos, col, faces, [cam], 128, 128, case["background"], flags=flags)
        engine._capacity._cap[key] = 17   # far too small
        rgb, _, st = engine.render_forward(pos, col, faces, [cam], 128, 128, case["background"], flags=flags)
        # the reference's E (5,997 at config 1); fewer without unreachable tiles
        assert st.entries == st0.entries == (expect or st0.entries) and st.capacity >= st.entries
        assert expect or st.entries < 5997
        assert np.array_equal(rgb.cpu().numpy(), ref.cpu().numpy())


def test_nan_vertex_is_depth_culled_like_reference(gmr):
    """A NaN mean fails the strict near < z < far test (render.py:108): the
    facet is culled, not reported -- same as the oracle."""
    from paper_2602_14493_b200 import engine
    import torch
    m = gmr.make_icosphere(80)
    v = np.asarray(m.vertices).copy()
    v[3, 0] = np.nan
    cam = gmr.look_at((0, 0, 3), (0, 0, 0), **gmr.default_intrinsics(32, 32))
    pos = torch.tensor(v, device="cuda")
    col = torch.full_like(pos, 0.5)
    faces = torch.tensor(np.asarray(m.facets, np.int32), device="cuda")
    rgb, _, _ = engine.render_forward(pos, col, faces, [cam], 32, 32, (0, 0, 0))
    cloud = orc.facet_gaussians(v, np.asarray(m.facets), np.full_like(v, 0.5))
    s = orc.project(cloud, cam)
    r, _ = orc.composite(s, 32, 32)
    assert np.abs(rgb[0].cpu().numpy() - r).max() <= 1e-10


@pytest.mark.parametrize("scale", [1e19, 1e20, 1e21])
def test_overflowing_splat_raises_reference_error(gmr, scale):
    """A finite but enormous sliver overflows its float32 screen covariance
    while its radius stays +inf, so it is kept: the reference raises
    ValueError("non-finite splat parameter 'cov2d' at splat 0")
    (render.py:191-197) for exactly these inputs; so must the device path."""
    v = np.array([(-scale, 0, 0), (scale, 0, 0), (0, 1, 0)], float)
    mesh = gmr.TriangleMesh(v, [(0, 1, 2)])
    cam = gmr.look_at((0.3, 0.2, 3), (0, 0, 0), **gmr.default_intrinsics(32, 32))
    with pytest.raises(ValueError, match="non-finite splat parameter 'cov2d' at splat 0"):
        gmr.render_mesh(mesh, cam, dtype=np.float32)


def test_nonfinite_error_reports_kept_splat_index(gmr):
    """The reference reports the index into the culled splat batch
    (render.py:191-197), not the face id: with face 0 behind the camera
    (culled) and face 1 kept, the overflowing sliver (face 2) is splat 1.
    Message from the reference itself on these inputs:
    ValueError("non-finite splat parameter 'cov2d' at splat 1")."""
    scale = 1e20
    v = np.array([(0, 0, 5), (0.1, 0, 5), (0, 0.1, 5), (0, 0, 0.5), (0.1, 0, 0.5), (0, 0.1, 0.5),
                  (-scale, 0, 0), (scale, 0, 0), (0, 1, 0)], float)
    mesh = gmr.TriangleMesh(v, [(0, 1, 2), (3, 4, 5), (6, 7, 8)])
    cam = gmr.look_at((0.3, 0.2, 3), (0, 0, 0), **gmr.default_intrinsics(32, 32))
    with pytest.raises(ValueError, match="non-finite splat parameter 'cov2d' at splat 1$"):
        gmr.render_mesh(mesh, cam, dtype=np.float32)


def test_backward_shape_errors_match_reference(gmr):
    case = gc.octahedron_case()
    mesh = gmr.TriangleMesh(case["vertices"], case["facets"], case["colors"])
    out, ctx = gmr.render_mesh(mesh, case["camera"], return_ctx=True)
    with pytest.raises(ValueError, match="upstream gradient shapes"):
        gmr.render_backward(ctx, np.zeros((31, 32, 3)), np.zeros((32, 32)))
    cloud = gmr.convert_mesh(mesh)
    with pytest.raises(ValueError, match="do not match"):
        gmr.convert_backward(mesh, cloud, np.zeros((7, 3)), np.zeros((8, 3, 3)), np.zeros((8, 3)))
    with pytest.raises(ValueError, match="unknown conversion path"):
        gmr.convert_mesh(mesh, path="bogus")


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_distant_mesh_long_tile_lists(gmr, dtype):
    """A 5,120-face sphere far from the camera: every facet lands in the same
    few tiles, so each list holds thousands of entries (beyond the per-tile
    sort's shared memory).  The engine uses the global depth sort for the
    first call and keeps it (the read-back list length is too long); forcing
    the per-tile sort (global-scratch path) must give the same lists, and the
    render must match the oracle."""
    import torch
    from paper_2602_14493_b200 import engine, lib
    m = gmr.make_icosphere(5120)
    mesh = gmr.TriangleMesh(m.vertices, m.facets, gmr.seeded_colors(m.num_vertices, 3))
    cam = gmr.look_at((0.0, -9.0, 2.0), (0, 0, 0), **gmr.default_intrinsics(40, 40))
    rng = np.random.default_rng(4)
    g_rgb, g_a = rng.normal(size=(40, 40, 3)), rng.normal(size=(40, 40))
    res = []
    old = engine.DEFAULT_FLAGS
    engine.AUTO_TILE_ORDER = False
    try:
        for mode in (0, lib.FLAG_TILE_DEPTH_SORT):
            engine.DEFAULT_FLAGS = mode
            out, ctx = gmr.render_mesh(mesh, cam, background=(0.1, 0.1, 0.1), dtype=dtype, return_ctx=True)
            items, bounds = engine.copy_entries(ctx.state, len(mesh.facets), True)
            gv, gc_ = gmr.render_backward(ctx, g_rgb, g_a)
            res.append((items.cpu().numpy(), bounds.cpu().numpy(), out.rgb, gv, gc_))
    finally:
        engine.DEFAULT_FLAGS = old
        engine.AUTO_TILE_ORDER = True
    assert np.diff(res[0][1]).max() > 2048   # the long-list path really ran
    for a, b in zip(res[0], res[1]):
        np.testing.assert_array_equal(a, b)
    r, _, octx = orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, (0.1, 0.1, 0.1), True, dtype)
    ogv = orc.render_grad(octx, g_rgb, g_a)[0]
    itol, gtol = (1e-10, 1e-8) if dtype == np.float64 else (2e-4, 2e-3)
    assert np.abs(res[0][2] - r).max() <= itol
    assert rel(res[0][3], ogv) <= gtol
    # the automatic choice: a list this long keeps the global sort
    engine._order.forget()
    for _ in range(3):
        _, ctx = gmr.render_mesh(mesh, cam, background=(0.1, 0.1, 0.1), dtype=dtype, return_ctx=True)
        torch.cuda.synchronize()
    assert ctx.state.raster.flags & lib.FLAG_TILE_DEPTH_SORT == 0


@pytest.mark.parametrize("seed", range(12))
def test_random_scenes_tile_lists_and_images(gmr, seed):
    """Randomised scenes (mesh size, camera distance incl. close-up and far,
    image sizes that are not tile multiples): in f64 the full tile lists
    equal the oracle's _RasterPlan bit for bit in both depth-order modes,
    and the image matches the oracle."""
    from paper_2602_14493_b200 import engine, lib
    rng = np.random.default_rng(100 + seed)
    n = int(rng.choice([3, 5, 8, 12]))
    mesh = gmr.make_geodesic_sphere(n, seed=seed)
    W, H = int(rng.integers(9, 70)), int(rng.integers(9, 70))
    d = float(rng.choice([1.3, 2.2, 3.5, 9.0]))
    u = rng.normal(size=3)
    eye = d * u / np.linalg.norm(u)
    cam = gmr.look_at(tuple(eye), (0, 0, 0), **gmr.default_intrinsics(W, H))
    bg = tuple(rng.uniform(0, 1, 3))
    cloud = orc.facet_gaussians(mesh.vertices, mesh.facets, mesh.colors)
    s = orc.project(cloud, cam, np.float64)
    entry, bounds = orc.bin_splats(s.mean2d, s.radius, s.depth, s.source, W, H)
    ref_items = np.asarray(s.source)[entry]
    r_ref, a_ref, _ = orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, bg)
    old = engine.DEFAULT_FLAGS
    engine.AUTO_TILE_ORDER = False
    try:
        for mode in (0, lib.FLAG_TILE_DEPTH_SORT):
            engine.DEFAULT_FLAGS = lib.FLAG_FULL_TILE_LISTS | mode
            out, ctx = gmr.render_mesh(mesh, cam, background=bg, dtype=np.float64, return_ctx=True)
            items, gb = engine.copy_entries(ctx.state, len(mesh.facets), True)
            np.testing.assert_array_equal(items.cpu().numpy(), ref_items)
            np.testing.assert_array_equal(gb.cpu().numpy(), bounds)
            assert np.abs(out.rgb - r_ref).max() <= 1e-10
            assert np.abs(out.alpha - a_ref).max() <= 1e-10
    finally:
        engine.DEFAULT_FLAGS = old
        engine.AUTO_TILE_ORDER = True


@pytest.mark.parametrize("seed", range(8))
def test_random_scenes_f32_and_backward_vs_oracle(gmr, seed):
    """Randomised scenes through the full fwd+bwd in both dtypes: f64 within
    1e-10 / 1e-8 of the oracle; f32 against the oracle's own f32 path with the
    flip-aware tolerances of test_gpu_parity (image 1e-4 except on at most
    0.1 % of pixels, gradients 1e-3 relative when nothing flipped)."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.choice([4, 6, 9]))
    mesh = gmr.make_geodesic_sphere(n, seed=seed)
    W, H = int(rng.integers(16, 64)), int(rng.integers(16, 64))
    d = float(rng.choice([1.6, 2.5, 4.0]))
    u = rng.normal(size=3)
    cam = gmr.look_at(tuple(d * u / np.linalg.norm(u)), (0, 0, 0), **gmr.default_intrinsics(W, H))
    bg = tuple(rng.uniform(0, 1, 3))
    g_rgb, g_a = rng.normal(size=(H, W, 3)), rng.normal(size=(H, W))
    for dtype in (np.float64, np.float32):
        r, a, octx = orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, bg, True, dtype)
        ogv, ogc = orc.render_grad(octx, g_rgb, g_a)
        out, ctx = gmr.render_mesh(mesh, cam, background=bg, dtype=dtype, return_ctx=True)
        gv, gcol = gmr.render_backward(ctx, g_rgb, g_a)
        if dtype == np.float64:
            assert np.abs(out.rgb - r).max() <= 1e-10 and np.abs(out.alpha - a).max() <= 1e-10
            assert rel(gv, ogv) <= 1e-8 and rel(gcol, ogc) <= 1e-8
        else:
            dd = np.abs(out.rgb.astype(np.float64) - r).max(axis=2)
            da = np.abs(out.alpha.astype(np.float64) - a)
            bad = (dd > 1e-4) | (da > 1e-4)
            assert bad.sum() <= max(2, 1e-3 * bad.size), (bad.sum(), dd.max())
            if bad.sum() == 0:
                assert rel(gv, ogv) <= 1e-3 and rel(gcol, ogc) <= 1e-3
            else:
                assert np.linalg.norm(gv - ogv) / np.linalg.norm(ogv) <= 1e-2


def test_backward_after_capacity_overflow_is_safe(gmr):
    """A forward planned with too few tile entries and left unchecked
    (check=False), followed directly by the backward: the backward reads
    nothing past the workspace and writes zero gradients; check_status then
    raises CapacityExceeded and a re-run (grown capacity) gives the normal
    result (face_views_backward used to read partials past the
    entry capacity)."""
    import torch
    from paper_2602_14493_b200 import engine
    case = gc.c1_case()
    pos = torch.tensor(case["vertices"], dtype=torch.float32, device="cuda")
    col = torch.tensor(case["colors"], dtype=torch.float32, device="cuda")
    faces = torch.tensor(case["facets"], dtype=torch.int32, device="cuda")
    cam = case["camera"]
    g_rgb = torch.tensor(case["g_rgb"][None], dtype=torch.float32, device="cuda")
    g_a = torch.tensor(case["g_alpha"][None], dtype=torch.float32, device="cuda")
    key = (len(case["facets"]), 1, 128, 128, torch.float32)
    engine._capacity._cap[key] = 16
    rgb, _, st = engine.render_forward(pos, col, faces, [cam], 128, 128, case["background"], check=False)
    gp, gcol = engine.render_backward(st, pos, col, faces, rgb, g_rgb, g_a)
    torch.cuda.synchronize()
    assert float(gp.abs().max()) == 0.0 and float(gcol.abs().max()) == 0.0
    with pytest.raises(engine.CapacityExceeded):
        engine.check_status(st)
    rgb2, _, st2 = engine.render_forward(pos, col, faces, [cam], 128, 128, case["background"], check=False)
    gp2, gc2 = engine.render_backward(st2, pos, col, faces, rgb2, g_rgb, g_a)
    engine.check_status(st2)
    rgb3, _, st3 = engine.render_forward(pos, col, faces, [cam], 128, 128, case["background"])
    gp3, _ = engine.render_backward(st3, pos, col, faces, rgb3, g_rgb, g_a)
    assert torch.equal(rgb2, rgb3) and torch.equal(gp2, gp3)
    assert float(gp2.abs().max()) > 0.0


def test_rasterize_backward_after_capacity_overflow_is_safe(gmr):
    """Splat path (splat_grads) under the same overflow."""
    import torch
    from paper_2602_14493_b200 import engine
    case = gc.splat_case()
    dt = torch.float64
    t = [torch.tensor(np.asarray(case[k]), dtype=dt, device="cuda") for k in ("mean2d", "cov2d", "depth", "color",
                                                                              "opacity")]
    K = int(t[2].shape[0])
    cam = case["camera"]
    key = ("splats", K, cam.width, cam.height, dt)
    engine._capacity._cap[key] = 2
    rgb, alpha, state = engine.rasterize_forward(*t, cam.width, cam.height, case["background"])
    # the checked forward re-planned; force an overflowed state for the backward
    engine._capacity._cap[key] = 2
    lib = engine.L.load()
    import ctypes
    raster = engine.raster_struct(cam.width, cam.height, case["background"], dt)
    sp = engine._splat_struct(*t)
    nb = ctypes.c_size_t()
    engine.L.check(lib.gmr_raster_workspace_size(K, cam.width, cam.height, 2, raster.dtype, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    rgb_o = torch.empty_like(rgb)
    a_o = torch.empty_like(alpha)
    engine.L.check(lib.gmr_rasterize_forward(ctypes.byref(sp), ctypes.byref(raster), engine._ptr(rgb_o),
                                             engine._ptr(a_o), engine._ptr(ws), nb.value, 2, engine._stream()))
    over = engine.ForwardState(ws, 2, raster, None, 1, -1, -1)
    g = torch.ones_like(rgb)
    gm, gcv, gcol, gop = engine.rasterize_backward(over, *t, rgb_o, g, torch.ones_like(alpha))
    torch.cuda.synchronize()
    for x in (gm, gcv, gcol, gop):
        assert float(x.abs().max()) == 0.0
