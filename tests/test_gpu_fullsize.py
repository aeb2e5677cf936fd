"""Config-3 size (499,280 faces, 800x800): parity and size-independent
properties at the full size, where the numpy oracle would take minutes.

- float64 parity with the reference itself: tests/golden/fullsize_c3_view0
  holds random-projection sketches of the reference's float64 image, alpha
  and gradients for one config-3 view (make_golden.py --fullsize, 70 s of
  CPU); our float64 path matches them to 1e-14 (bound 1e-12);
- float32 precision spread: float32 against float64 moves pixels across the
  alpha floor / stop / clamp thresholds (decision flips), which concentrates
  the gradient difference on a few vertices (99 % of the error norm in 0.1 %
  of them).  At this facet density the reference's OWN float32-vs-float64
  spread is 253 flipped pixels and gradient relative-L2 3.5e-3 / 1.7e-3,
  beyond SURVEY 8c's 1e-3 global figure, so the bound is the reference's
  measured spread x1.5 (same scene, same upstream gradient; ours measured
  299 pixels, 3.55e-3 / 1.71e-3);
- the backward is linear in the upstream image gradients;
- the forward and backward are bit-deterministic, and dropping unreachable
  tiles changes no bit of the outputs.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W = H = 800
VIEWS = 4


@pytest.fixture(scope="module")
def scene(gmr):
    import torch
    mesh = gmr.make_geodesic_sphere(158, seed=0)
    cams = gmr.hemisphere_cameras(VIEWS, 3.0, (W, H))
    faces = torch.tensor(mesh.facets, dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(11)
    g_rgb = torch.randn((VIEWS, H, W, 3), generator=g, device="cuda", dtype=torch.float64)
    g_a = torch.randn((VIEWS, H, W), generator=g, device="cuda", dtype=torch.float64)
    return mesh, cams, faces, g_rgb, g_a


def _run(scene, dtype, flags=0, g_scale=1.0, g_rgb=None, g_a=None):
    import torch
    from paper_2602_14493_b200 import engine
    mesh, cams, faces, gr, ga = scene
    pos = torch.tensor(mesh.vertices, dtype=dtype, device="cuda")
    col = torch.tensor(mesh.colors, dtype=dtype, device="cuda")
    gr = (gr if g_rgb is None else g_rgb).to(dtype) * g_scale
    ga = (ga if g_a is None else g_a).to(dtype) * g_scale
    rgb, alpha, st = engine.render_forward(pos, col, faces, cams, W, H, (0.1, 0.1, 0.1), flags=flags)
    gp, gc = engine.render_backward(st, pos, col, faces, rgb, gr, ga)
    return rgb, alpha, gp, gc


@pytest.fixture(scope="module")
def view0(gmr):
    """One config-3 view in float64 and float32 through the public engine."""
    import torch
    from paper_2602_14493_b200 import engine
    from golden_cases import fullsize_case
    case = fullsize_case()
    faces = torch.tensor(case["facets"], dtype=torch.int32, device="cuda")
    out = {}
    for dt in (torch.float64, torch.float32):
        pos = torch.tensor(case["vertices"], dtype=dt, device="cuda")
        col = torch.tensor(case["colors"], dtype=dt, device="cuda")
        rgb, a, st = engine.render_forward(pos, col, faces, [case["camera"]], W, H, case["background"])
        gr = torch.tensor(case["g_rgb"][None], dtype=dt, device="cuda")
        ga = torch.tensor(case["g_alpha"][None], dtype=dt, device="cuda")
        gp, gc = engine.render_backward(st, pos, col, faces, rgb, gr, ga)
        out[dt] = [x.double().cpu().numpy() for x in (rgb[0], a[0], gp, gc)]
    return out


def test_float64_matches_reference_at_full_size(view0):
    import torch
    from golden_cases import load, sketch
    gold = load("fullsize_c3_view0")
    for i, (name, x) in enumerate(zip(("rgb", "alpha", "gv", "gc"), view0[torch.float64])):
        s, ref = sketch(x, i), gold[f"sketch_{name}"]
        assert np.linalg.norm(s - ref) / np.linalg.norm(ref) <= 1e-12, name


def test_float32_spread_within_reference_spread(view0):
    import torch
    from golden_cases import flip_stats, load
    gold = load("fullsize_c3_view0")
    r32, a32, gv32, gc32 = view0[torch.float32]
    r64, a64, gv64, gc64 = view0[torch.float64]
    st = flip_stats(r32, a32, r64, a64, gv32, gv64, gc32, gc64)
    assert 2 * st["flips"] <= 3 * int(gold["ref32_flips"]), st
    assert st["rel_gv"] <= 1.5 * float(gold["ref32_rel_gv"]), st
    assert st["rel_gc"] <= 1.5 * float(gold["ref32_rel_gc"]), st


def test_backward_is_linear_in_upstream_grads(scene):
    import torch
    mesh, cams, faces, gr, ga = scene
    g = torch.Generator(device="cuda").manual_seed(12)
    gr2 = torch.randn(gr.shape, generator=g, device="cuda", dtype=torch.float64)
    ga2 = torch.randn(ga.shape, generator=g, device="cuda", dtype=torch.float64)
    _, _, p1, c1 = _run(scene, torch.float64)
    _, _, p2, c2 = _run(scene, torch.float64, g_rgb=gr2, g_a=ga2)
    _, _, p12, c12 = _run(scene, torch.float64, g_rgb=gr + gr2, g_a=ga + ga2)
    for a, b in ((p12, p1 + p2), (c12, c1 + c2)):
        assert (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item() <= 1e-12


def test_bit_deterministic_and_cull_invariant_at_full_size(scene):
    import torch
    from paper_2602_14493_b200 import lib
    a = _run(scene, torch.float32)
    b = _run(scene, torch.float32)
    c = _run(scene, torch.float32, flags=lib.FLAG_FULL_TILE_LISTS)
    for x, y, z in zip(a, b, c):
        assert torch.equal(x, y)
        assert torch.equal(x, z)
