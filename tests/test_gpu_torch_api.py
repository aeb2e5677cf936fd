"""The batched torch entry point `render_views` (engine.GMRRender, the path
bench.py's e2e number goes through): forward vs the oracle, autograd vs
`render_backward` and the oracle, partial requires_grad, single-output
losses, input validation."""

import numpy as np
import pytest

from oracle import gmr_oracle as orc

pytestmark = pytest.mark.gpu


def _scene(gmr, dtype):
    import torch
    mesh = gmr.make_geodesic_sphere(12, seed=4)
    cams = gmr.hemisphere_cameras(3, 3.0, (72, 56))
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    pos = torch.tensor(mesh.vertices, dtype=tdt, device="cuda")
    col = torch.tensor(mesh.colors, dtype=tdt, device="cuda")
    faces = torch.tensor(mesh.facets, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(2)
    g_rgb = rng.standard_normal((3, 56, 72, 3))
    g_a = rng.standard_normal((3, 56, 72))
    return mesh, cams, pos, col, faces, g_rgb, g_a


def test_render_views_forward_and_autograd_f64(gmr):
    import torch
    from paper_2602_14493_b200 import engine
    mesh, cams, pos, col, faces, g_rgb, g_a = _scene(gmr, np.float64)
    bg = (0.1, 0.2, 0.3)
    p = pos.clone().requires_grad_(True)
    c = col.clone().requires_grad_(True)
    rgb, alpha = engine.render_views(p, c, faces, cams, 72, 56, bg)
    assert rgb.shape == (3, 56, 72, 3) and alpha.shape == (3, 56, 72) and rgb.dtype == torch.float64
    loss = (rgb * torch.tensor(g_rgb, device="cuda")).sum() + (alpha * torch.tensor(g_a, device="cuda")).sum()
    loss.backward()
    gv = np.zeros((len(mesh.vertices), 3))
    gc = np.zeros((len(mesh.vertices), 3))
    for i, cam in enumerate(cams):
        r, a, ctx = orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, bg, True, np.float64)
        np.testing.assert_allclose(rgb[i].detach().cpu().numpy(), r, rtol=0, atol=1e-10)
        np.testing.assert_allclose(alpha[i].detach().cpu().numpy(), a, rtol=0, atol=1e-10)
        v, cc = orc.render_grad(ctx, g_rgb[i], g_a[i])
        gv += v
        gc += cc
    rel = lambda x, y: np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30)
    assert rel(p.grad.cpu().numpy(), gv) <= 1e-8
    assert rel(c.grad.cpu().numpy(), gc) <= 1e-8


def test_render_views_matches_engine_calls_f32(gmr):
    """autograd = render_forward + render_backward, bit for bit."""
    import torch
    from paper_2602_14493_b200 import engine
    mesh, cams, pos, col, faces, g_rgb, g_a = _scene(gmr, np.float32)
    gr = torch.tensor(g_rgb, dtype=torch.float32, device="cuda")
    ga = torch.tensor(g_a, dtype=torch.float32, device="cuda")
    p = pos.clone().requires_grad_(True)
    c = col.clone().requires_grad_(True)
    rgb, alpha = engine.render_views(p, c, faces, cams, 72, 56)
    torch.autograd.backward([rgb, alpha], [gr, ga])
    rgb2, alpha2, st = engine.render_forward(pos, col, faces, cams, 72, 56, (0.0, 0.0, 0.0))
    gp2, gc2 = engine.render_backward(st, pos, col, faces, rgb2, gr, ga)
    assert torch.equal(rgb.detach(), rgb2) and torch.equal(alpha.detach(), alpha2)
    assert torch.equal(p.grad, gp2) and torch.equal(c.grad, gc2)


@pytest.mark.parametrize("which", ["rgb", "alpha"])
def test_single_output_loss_and_partial_requires_grad(gmr, which):
    """A loss on only one output (the other's grad is None -> zeros), and
    gradients requested for positions only."""
    import torch
    from paper_2602_14493_b200 import engine
    mesh, cams, pos, col, faces, g_rgb, g_a = _scene(gmr, np.float64)
    p = pos.clone().requires_grad_(True)
    rgb, alpha = engine.render_views(p, col, faces, cams, 72, 56)
    out, g = (rgb, g_rgb) if which == "rgb" else (alpha, g_a)
    (out * torch.tensor(g, device="cuda")).sum().backward()
    assert col.grad is None
    z_rgb = np.zeros_like(g_rgb) if which == "alpha" else g_rgb
    z_a = np.zeros_like(g_a) if which == "rgb" else g_a
    gv = sum(orc.render_grad(orc.render(mesh.vertices, mesh.facets, mesh.colors, cam, (0, 0, 0), True,
                                        np.float64)[2], z_rgb[i], z_a[i])[0] for i, cam in enumerate(cams))
    assert np.linalg.norm(p.grad.cpu().numpy() - gv) <= 1e-8 * np.linalg.norm(gv)


def test_render_views_rejects_bad_inputs(gmr):
    import torch
    from paper_2602_14493_b200 import engine
    mesh, cams, pos, col, faces, _, _ = _scene(gmr, np.float32)
    with pytest.raises(ValueError, match="dtype"):
        engine.render_views(pos, col.double(), faces, cams, 72, 56)
    with pytest.raises(ValueError, match="int32"):
        engine.render_views(pos, col, faces.long(), cams, 72, 56)
    with pytest.raises(ValueError, match=r"\[V, 3\]"):
        engine.render_views(pos[:, :2], col, faces, cams, 72, 56)
    with pytest.raises(ValueError, match="same CUDA device"):
        engine.render_views(pos.cpu(), col, faces, cams, 72, 56)
    with pytest.raises(ValueError, match="camera"):
        engine.render_views(pos, col, faces, [], 72, 56)
