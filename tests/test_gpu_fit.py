"""Config 5: the 200-iteration inverse-rendering loop on the device render
path vs the real reference's trajectory (tests/golden/fit_c5_200.npz, made by
make_golden.py --fit; iteration-0 total 1.405564 as recorded in
pkg/test_output.txt:265)."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc

pytestmark = pytest.mark.gpu


def _trajectory_check(ours, ref32, ref64, spread):
    """200 Adam steps on fp32 renders are chaotic: two fp32 implementations
    that differ only in summation order part ways like the reference's own
    fp32 and fp64 runs do (`spread`, up to ~2.4 %).  The short-horizon
    deterministic parity is `test_fit_*_prefix`; here: the trajectory stays
    within twice that spread of the reference's fp32 run or of its fp64 run,
    and the final loss within the spread."""
    d32 = np.abs(ours - ref32) / ref32
    d64 = np.abs(ours - ref64) / ref64
    print(f"trajectory: max |ours-ref32| {d32.max():.4f} @ {d32.argmax()}, |ours-ref64| {d64.max():.4f}, "
          f"reference fp32-vs-fp64 spread {spread:.4f}")
    assert np.all(np.minimum(d32, d64) <= 2.0 * spread)
    assert min(d32[-1], d64[-1]) <= spread


def test_fit_config5_prefix(gmr):
    """The reference run cut to 5 iterations (fit_c5_5.npz): per-iteration
    losses to fp32 rounding and the final vertices/colours to 1e-5."""
    from paper_2602_14493_b200 import fit as gfit
    case, g = gc.fit_case(), gc.load("fit_c5_5")
    init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
    cfg = gfit.FitConfig(iterations=5, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    res = gfit.fit(init, case["cameras"], list(gc.load("fit_c5_200")["target_rgb"]),
                   list(gc.load("fit_c5_200")["target_mask"]), cfg)
    hist = np.array([[h["total"], h["color"], h["silhouette"], h["edge"], h["laplacian"]] for h in res.history])
    np.testing.assert_allclose(hist, g["history"], rtol=2e-5, atol=1e-9)
    np.testing.assert_allclose(res.mesh.vertices, g["vertices"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(res.mesh.colors, g["colors"], rtol=0, atol=1e-5)


def test_fit_config5_loss_parity(gmr):
    """The whole iteration on the GPU (fused losses + gmr_fit_step) tracks
    the reference's 200-iteration trajectory."""
    from paper_2602_14493_b200 import fit as gfit
    case, g = gc.fit_case(), gc.load("fit_c5_200")
    init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
    cfg = gfit.FitConfig(iterations=200, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    res = gfit.fit(init, case["cameras"], list(g["target_rgb"]), list(g["target_mask"]), cfg)
    hist = np.array([[h["total"], h["color"], h["silhouette"], h["edge"], h["laplacian"]] for h in res.history])
    ref = g["history"]
    # same seeded view order, same fp32 render dtype: the first iterations agree
    # to fp32 rounding; later ones drift apart only through optimiser feedback.
    # Tolerance: the reference's OWN fp32-vs-fp64 spread on this loop (up to
    # ~2.4 % along the trajectory), plus margin.
    spread = np.max(np.abs(g["history_f64"] - ref[:, 0]) / ref[:, 0])
    assert spread < 0.03
    assert hist[0, 0] == pytest.approx(1.405564, abs=5e-6), (hist[:3], ref[:3])
    # regulariser values are computed in float64 on the device from float64 parameters
    np.testing.assert_allclose(hist[0, 3:], ref[0, 3:], rtol=1e-10)
    _trajectory_check(hist[:, 0], ref[:, 0], g["history_f64"], spread)
    print(f"fit: final total {hist[-1, 0]:.6f} (reference {ref[-1, 0]:.6f}), {res.wall_time:.3f}s "
          f"vs reference {float(g['wall_time']):.1f}s")


def test_fit_matches_host_optimiser_oracle(gmr):
    """Device optimiser vs the reference's optimiser restated in numpy
    (oracle VectorAdam / ScalarAdam / cosine_lr, optim.py:29-135) driven by
    the same device objective (api.total_loss), float64 state in both."""
    from paper_2602_14493_b200 import fit as gfit
    case, g = gc.fit_case(), gc.load("fit_c5_200")
    init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
    cfg = gfit.FitConfig(iterations=20, batch_size=2, seed=3, log_every=0, lr_positions=1e-2)
    rgbs, masks = list(g["target_rgb"]), list(g["target_mask"])
    b = gfit.fit(init, case["cameras"], rgbs, masks, cfg)
    sampler = gfit._ViewSampler(len(case["cameras"]), cfg.seed)
    popt, copt = orc.VectorAdam(len(init.vertices)), orc.ScalarAdam(init.colors.shape)
    v, c = np.array(init.vertices), np.array(init.colors)
    totals = []
    for it in range(cfg.iterations):
        batch = sampler.next_batch(cfg.batch_size)
        mesh = gmr.TriangleMesh(v, init.facets, c)
        rep, gv, gcol = gmr.total_loss(mesh, [case["cameras"][i] for i in batch], [rgbs[i] for i in batch],
                                       [masks[i] for i in batch], weights=cfg.weights, dtype=np.float32)
        totals.append(rep.total)
        v = popt.step(v, gv, orc.cosine_lr(it, cfg.iterations, cfg.lr_positions))
        c = np.clip(copt.step(c, gcol, orc.cosine_lr(it, cfg.iterations, cfg.lr_colors)), 0.0, 1.0)
    hb = np.array([h["total"] for h in b.history])
    np.testing.assert_allclose(hb, np.array(totals), rtol=1e-4)
    np.testing.assert_allclose(b.mesh.vertices, v, rtol=0, atol=1e-5)


def test_fit_retries_after_capacity_overflow(gmr):
    """A render that overflows its tile-entry capacity is rejected on the
    device (no optimiser step on invalid gradients) and the loop re-runs with
    the capacity the statuses reported: the result equals a run that never
    overflowed."""
    from paper_2602_14493_b200 import engine
    from paper_2602_14493_b200 import fit as gfit
    case, g = gc.fit_case(), gc.load("fit_c5_200")
    init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
    cfg = gfit.FitConfig(iterations=12, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    args = (init, case["cameras"], list(g["target_rgb"]), list(g["target_mask"]), cfg)
    a = gfit.fit(*args, graphs=False)
    key = (len(init.facets), 1, 64, 64, __import__("torch").float32)
    gfit.PRESET_WORST_CASE = False
    try:
        engine._capacity._cap[key] = 64
        b = gfit.fit(*args, graphs=False)
        assert engine._capacity._cap[key] > 64
    finally:
        gfit.PRESET_WORST_CASE = True
    np.testing.assert_array_equal(np.array([h["total"] for h in b.history]), np.array([h["total"] for h in a.history]))
    np.testing.assert_array_equal(b.mesh.vertices, a.mesh.vertices)


def test_fit_graphs_match_eager(gmr):
    """One captured CUDA graph per view, replayed per iteration, gives the
    same trajectory as eager launches (bit-identical kernels and inputs)."""
    from paper_2602_14493_b200 import fit as gfit
    case, g = gc.fit_case(), gc.load("fit_c5_200")
    init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
    cfg = gfit.FitConfig(iterations=40, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    a = gfit.fit(init, case["cameras"], list(g["target_rgb"]), list(g["target_mask"]), cfg, graphs=False)
    b = gfit.fit(init, case["cameras"], list(g["target_rgb"]), list(g["target_mask"]), cfg, graphs=True)
    np.testing.assert_array_equal(np.array([h["total"] for h in b.history]), np.array([h["total"] for h in a.history]))
    np.testing.assert_array_equal(b.mesh.vertices, a.mesh.vertices)
    np.testing.assert_array_equal(b.mesh.colors, a.mesh.colors)
