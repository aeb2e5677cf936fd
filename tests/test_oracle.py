"""Pin the CPU oracle to the real reference.

The fixtures under tests/golden/ were produced by running the reference
itself (tests/golden/make_golden.py).  When /root/reference is importable
(build container) the oracle is also compared to it live on fresh inputs.
"""

import os
import sys

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc

REF_SRC = "/root/reference/pkg/src"


def _render(case, dtype):
    return orc.render(case["vertices"], case["facets"], case["colors"], case["camera"],
                      case["background"], True, dtype)


@pytest.mark.parametrize("name,maker", [
    ("c1_icosphere1280_128", gc.c1_case),
    ("octahedron_32", gc.octahedron_case),
    ("icosphere320_64x48", gc.small_render_case),
])
@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
def test_render_matches_reference_golden(name, maker, tag, dtype):
    case = maker()
    g = gc.load(name)
    rgb, alpha, ctx = _render(case, dtype)
    gv, gcol = orc.render_grad(ctx, case["g_rgb"], case["g_alpha"])
    # binning is integer work: exact
    np.testing.assert_array_equal(ctx.splats.source, g[f"{tag}_source"])
    entry, bounds = orc.bin_splats(ctx.splats.mean2d, ctx.splats.radius, ctx.splats.depth,
                                   ctx.splats.source, case["camera"].width, case["camera"].height)
    np.testing.assert_array_equal(ctx.splats.source[entry], g[f"{tag}_entry_source"])
    np.testing.assert_array_equal(bounds, g[f"{tag}_bounds"])
    # same op order as the reference: agreement to rounding
    tol = 1e-12 if dtype == np.float64 else 1e-6
    np.testing.assert_allclose(rgb, g[f"{tag}_rgb"], rtol=0, atol=tol)
    np.testing.assert_allclose(alpha, g[f"{tag}_alpha"], rtol=0, atol=tol)
    scale = max(1.0, np.abs(g[f"{tag}_grad_v"]).max())
    gtol = 1e-10 if dtype == np.float64 else 1e-5
    np.testing.assert_allclose(gv, g[f"{tag}_grad_v"], rtol=0, atol=gtol * scale)
    np.testing.assert_allclose(gcol, g[f"{tag}_grad_c"], rtol=0, atol=gtol)


@pytest.mark.parametrize("name,maker", [("splats7_32", gc.splat_case),
                                        ("splats_closed_form_32", gc.closed_form_splat_case)])
def test_composite_matches_reference_golden(name, maker):
    case = maker()
    g = gc.load(name)
    s = orc.splats_from_arrays(case["mean2d"], case["cov2d"], case["depth"], case["color"],
                               case["opacity"], case["source"])
    cam = case["camera"]
    rgb, alpha = orc.composite(s, cam.width, cam.height, case["background"])
    np.testing.assert_allclose(rgb, g["rgb"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(alpha, g["alpha"], rtol=0, atol=1e-13)
    gm, gcv, gcol, gop = orc.composite_backward(s, cam.width, cam.height, case["background"],
                                                case["g_rgb"], case["g_alpha"])
    for a, k in ((gm, "g_mean2d"), (gcv, "g_cov2d"), (gcol, "g_color"), (gop, "g_opacity")):
        np.testing.assert_allclose(a, g[k], rtol=0, atol=1e-11)


def test_closed_forms():
    """reference test_render.py:173-189: 0.99 clamp, red over blue."""
    case = gc.closed_form_splat_case()
    s = orc.splats_from_arrays(case["mean2d"], case["cov2d"], case["depth"], case["color"],
                               case["opacity"], case["source"])
    rgb, alpha = orc.composite(s, 32, 32, case["background"])
    assert rgb[16, 16, 0] == pytest.approx(0.99, abs=1e-12)
    assert rgb[16, 16, 2] == pytest.approx(0.01 * 0.99, abs=1e-12)
    assert alpha[16, 16] == pytest.approx(1 - 1e-4)


def test_view_loop_matches_reference_golden():
    case = gc.loss_case()
    g = gc.load("loss_octa_3views_16")
    cv, sv, gv, gcol = orc.views_image_grad(case["vertices"], case["facets"], case["colors"],
                                            case["cameras"], case["target_rgb"],
                                            case["target_mask"], background=case["background"])
    assert cv == pytest.approx(float(g["color"]), rel=1e-12)
    assert sv == pytest.approx(float(g["silhouette"]), rel=1e-12)
    np.testing.assert_allclose(gv, g["grad_v"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(gcol, g["grad_c"], rtol=0, atol=1e-12)


def test_conversion_matches_reference_golden():
    case = gc.convert_case()
    g = gc.load("convert_random50")
    cloud = orc.facet_gaussians(case["vertices"], case["facets"], case["colors"])
    np.testing.assert_array_equal(cloud["degenerate"], g["degenerate"])
    assert cloud["degenerate"][1] and not cloud["degenerate"][2]
    np.testing.assert_allclose(cloud["means"], g["means"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(cloud["cov3d"], g["cov3d"], rtol=0, atol=1e-15)
    gv, gcol = orc.facet_backward(case["vertices"], case["facets"], case["colors"],
                                  case["g_means"], case["g_cov3d"], case["g_colors"])
    np.testing.assert_allclose(gv, g["grad_v"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gcol, g["grad_c"], rtol=0, atol=1e-15)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_live_reference_fresh_inputs():
    """Fresh random scene: oracle vs the reference imported in this container."""
    sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    import meshsplat as ms
    from paper_2602_14493_b200.camera import default_intrinsics, look_at
    from paper_2602_14493_b200.mesh import make_geodesic_sphere
    m = make_geodesic_sphere(6, seed=3)
    cam = look_at((1.1, 2.3, -1.2), (0, 0, 0), **default_intrinsics(40, 56))
    rng = np.random.default_rng(99)
    g_rgb, g_a = rng.normal(size=(56, 40, 3)), rng.normal(size=(56, 40))
    rmesh = ms.TriangleMesh(m.vertices, m.facets, m.colors)
    rcam = ms.Camera(rotation=cam.rotation, translation=cam.translation, fx=cam.fx, fy=cam.fy,
                     cx=cam.cx, cy=cam.cy, width=cam.width, height=cam.height)
    for dt in (np.float64, np.float32):
        o, ctx = ms.render_mesh(rmesh, rcam, background=(0.3, 0.2, 0.1), dtype=dt, return_ctx=True)
        rgv, rgc = ms.render_backward(ctx, g_rgb, g_a)
        rgb, alpha, octx = orc.render(m.vertices, m.facets, m.colors, cam, (0.3, 0.2, 0.1), True, dt)
        gv, gcol = orc.render_grad(octx, g_rgb, g_a)
        np.testing.assert_array_equal(rgb, o.rgb)
        np.testing.assert_array_equal(alpha, o.alpha)
        np.testing.assert_allclose(gv, rgv, rtol=0, atol=1e-9 * max(1, np.abs(rgv).max()))
        np.testing.assert_allclose(gcol, rgc, rtol=0, atol=1e-9)
