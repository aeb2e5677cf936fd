"""Gaussian export and evaluation metrics.

Golden: tests/golden/eval_ico320.npz, from the reference's own
export_gaussians / sample_surface / chamfer_distance / normal_consistency /
psnr / ssim / image_metrics (make_golden.py `eval_case`).  CPU tests pin the
oracle (oracle/eval_oracle.py) and the host-side sample stream; GPU tests run
the device kernels (gmr_export_gaussians, gmr_chamfer_nc, gmr_nearest,
gmr_image_metrics)."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import eval_oracle as eo
from paper_2602_14493_b200 import metrics as gm
from paper_2602_14493_b200.mesh import TriangleMesh


def _meshes():
    c = gc.eval_case()
    return c, TriangleMesh(c["gt_vertices"], c["gt_facets"]), \
        TriangleMesh(c["pred_vertices"], c["pred_facets"], c["pred_colors"])


def _parse_ply(raw):
    raw = bytes(raw)
    end = raw.index(b"end_header\n") + len(b"end_header\n")
    return raw[:end], np.frombuffer(raw[end:], "<f4").reshape(-1, 14)


def test_oracle_sample_stream_matches_reference():
    c, gt, pred = _meshes()
    g = gc.load("eval_ico320")
    sp, sn = eo.sample_surface(pred.vertices, pred.facets, 70000, seed=3)
    sel = np.r_[0:100, 65500:65600, 69900:70000]
    np.testing.assert_array_equal(sp[sel], g["samples_sel"])
    np.testing.assert_array_equal(sn[sel], g["snormals_sel"])
    np.testing.assert_array_equal([sp.sum(), (sp * sp).sum(), sn.sum()], g["samples_sum"])


def test_oracle_metrics_match_reference():
    c, gt, pred = _meshes()
    g = gc.load("eval_ico320")
    n = c["n_samples"]

    def pass_(sa, sb):
        pp, pn = eo.sample_surface(pred.vertices, pred.facets, n, seed=sa)
        qp, qn = eo.sample_surface(gt.vertices, gt.facets, n, seed=sb)
        return eo.chamfer_nc_pass(pp, pn, qp, qn)
    a, b = pass_(0, 1), pass_(1, 0)
    assert 0.5 * (a[0] + b[0]) == pytest.approx(float(g["cd"]), rel=1e-14)
    assert 0.5 * (a[1] + b[1]) == pytest.approx(float(g["nc"]), rel=1e-14)
    f = pass_(2, 5)
    assert f[0] == pytest.approx(float(g["cd_fixed"]), rel=1e-14)
    assert f[1] == pytest.approx(float(g["nc_fixed"]), rel=1e-14)
    for i, (x, y) in enumerate(c["images"]):
        assert eo.psnr(x, y) == pytest.approx(float(g[f"psnr{i}"]), rel=1e-14)
        assert eo.ssim(x, y) == pytest.approx(float(g[f"ssim{i}"]), rel=1e-13)


def test_oracle_export_matches_reference_bytes():
    from oracle import gmr_oracle as orc
    c, gt, pred = _meshes()
    g = gc.load("eval_ico320")
    cl = orc.facet_gaussians(pred.vertices, pred.facets, pred.colors)
    np.testing.assert_array_equal(cl["cov3d"], g["cloud_cov3d"])
    rec = eo.export_records(cl["means"], cl["cov3d"], cl["colors"], cl["opacities"])
    head, ref = _parse_ply(g["export_bytes"])
    np.testing.assert_array_equal(rec, ref)
    assert head.decode().splitlines()[2] == f"element vertex {len(rec)}"


def test_input_validation_without_gpu():
    with pytest.raises(ValueError, match="shape mismatch"):
        gm.psnr(np.zeros((4, 4)), np.zeros((4, 5)))
    with pytest.raises(ValueError, match="at least 11"):
        gm.ssim(np.zeros((10, 30)), np.zeros((10, 30)))


@pytest.mark.gpu
def test_device_sample_stream_matches_reference(gmr):
    c, gt, pred = _meshes()
    g = gc.load("eval_ico320")
    sp, sn = gm.sample_surface(pred, 70000, seed=3)
    sel = np.r_[0:100, 65500:65600, 69900:70000]
    np.testing.assert_array_equal(sp[sel], g["samples_sel"])
    np.testing.assert_array_equal(sn[sel], g["snormals_sel"])
    np.testing.assert_array_equal([sp.sum(), (sp * sp).sum(), sn.sum()], g["samples_sum"])
    # a larger mesh (pairwise-sum tree with many leaves, long sequential CDF)
    big = gmr.make_geodesic_sphere(60, seed=2)
    p1, n1 = gm.sample_surface(big, 50000, seed=9)
    p0, n0 = eo.sample_surface(big.vertices, big.facets, 50000, seed=9)
    np.testing.assert_array_equal(p1, p0)
    np.testing.assert_array_equal(n1, n0)
    with pytest.raises(gm.DegenerateGeometryError):
        gm.sample_surface(TriangleMesh(np.zeros((3, 3)), [[0, 1, 2]]), 10)


# ---------------------------------------------------------------------------
# device
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_chamfer_nc_gpu_match_reference(gmr):
    c, gt, pred = _meshes()
    g = gc.load("eval_ico320")
    n = c["n_samples"]
    assert gm.chamfer_distance(pred, gt, n_samples=n, seed=0) == pytest.approx(float(g["cd"]), rel=1e-12)
    assert gm.normal_consistency(pred, gt, n_samples=n, seed=0) == pytest.approx(float(g["nc"]), rel=1e-12)
    cd, nc = gm.chamfer_and_normal_consistency(pred, gt, n_samples=n, seed=2, gt_seed=5)
    assert cd == pytest.approx(float(g["cd_fixed"]), rel=1e-12)
    assert nc == pytest.approx(float(g["nc_fixed"]), rel=1e-12)
    assert gm.chamfer_distance(gt, gt, n_samples=n, seed=4, gt_seed=4) == 0.0
    # swapping the arguments gives the identical value (metrics.py:55-57)
    assert gm.chamfer_distance(gt, pred, n_samples=n, seed=0) == pytest.approx(float(g["cd"]), rel=1e-12)


@pytest.mark.gpu
def test_nearest_gpu_matches_kdtree(gmr):
    import ctypes

    import torch
    from scipy.spatial import cKDTree

    from paper_2602_14493_b200 import lib as L
    rng = np.random.default_rng(5)
    for n, m in ((1, 1), (1000, 777), (70001, 40000)):
        q, p = rng.random((n, 3)), rng.random((m, 3))
        d_ref, i_ref = cKDTree(p).query(q)
        lib = L.load()
        sz = ctypes.c_size_t()
        L.check(lib.gmr_nearest_scratch_size(n, m, ctypes.byref(sz)))
        tq, tp = torch.tensor(q, device="cuda"), torch.tensor(p, device="cuda")
        d2 = torch.empty(n, dtype=torch.float64, device="cuda")
        idx = torch.empty(n, dtype=torch.int32, device="cuda")
        scratch = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
        L.check(lib.gmr_nearest(tq.data_ptr(), n, tp.data_ptr(), m, d2.data_ptr(), idx.data_ptr(),
                                scratch.data_ptr(), sz.value, None))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(idx.cpu().numpy(), i_ref)
        np.testing.assert_allclose(d2.cpu().numpy(), d_ref ** 2, rtol=1e-15, atol=0)


@pytest.mark.gpu
def test_image_metrics_gpu_match_reference(gmr):
    c = gc.eval_case()
    g = gc.load("eval_ico320")
    for i, (x, y) in enumerate(c["images"]):
        assert gm.psnr(x, y) == pytest.approx(float(g[f"psnr{i}"]), rel=1e-13)
        assert gm.ssim(x, y) == pytest.approx(float(g[f"ssim{i}"]), rel=1e-12)
    assert gm.psnr(c["images"][0][0], c["images"][0][0]) == 99.0
    pv, sv = gm.image_metrics([c["images"][0][0], c["images"][2][0]], [c["images"][0][1], c["images"][2][1]])
    np.testing.assert_allclose(pv, g["im_psnr"], rtol=1e-13)
    np.testing.assert_allclose(sv, g["im_ssim"], rtol=1e-12)


@pytest.mark.gpu
def test_export_gpu_matches_reference(gmr, tmp_path):
    from paper_2602_14493_b200 import api
    c, gt, pred = _meshes()
    g = gc.load("eval_ico320")
    cloud = api.convert_mesh(pred)
    np.testing.assert_allclose(cloud.cov3d, g["cloud_cov3d"], rtol=1e-13, atol=1e-28)
    api.export_gaussians(cloud, tmp_path / "g.ply")
    head, rec = _parse_ply(np.frombuffer((tmp_path / "g.ply").read_bytes(), np.uint8))
    ref_head, ref = _parse_ply(g["export_bytes"])
    assert head == ref_head
    # position, colour and opacity fields: identical float32 values
    np.testing.assert_array_equal(rec[:, :7], ref[:, :7])
    # log-scales: the in-plane eigenvalues agree to float32 rounding; the
    # normal-direction one is ~1e-12 inside a ~1e-3 matrix, which any float64
    # eigensolver (LAPACK's or this Jacobi) only resolves to ~eps*|A|/lam
    # ~ 1e-6 relative, i.e. a few float32 ulps of log(scale) ~ -13.8
    np.testing.assert_allclose(rec[:, 7:9], ref[:, 7:9], rtol=0, atol=1e-6)
    np.testing.assert_allclose(rec[:, 9], ref[:, 9], rtol=0, atol=1e-5)
    q = rec[:, 10:14].astype(np.float64)
    np.testing.assert_allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-6)
    assert np.all(q[:, 0] >= 0)
    # the rotation is an eigenbasis: R diag(s^2) R^T reconstructs cov3d
    # (eigenvectors of repeated eigenvalues are not unique, so quaternions are
    # compared through the covariance they encode)
    R = eo.quat_to_rot(q)
    s2 = np.exp(2.0 * rec[:, 7:10].astype(np.float64))
    cov = np.einsum("nij,nj,nkj->nik", R, s2, R)
    scale = np.abs(g["cloud_cov3d"]).max(axis=(1, 2))[:, None, None]
    np.testing.assert_allclose(cov / scale, g["cloud_cov3d"] / scale, rtol=0, atol=5e-6)
    Rr = eo.quat_to_rot(ref[:, 10:14].astype(np.float64))
    cov_r = np.einsum("nij,nj,nkj->nik", Rr, np.exp(2.0 * ref[:, 7:10].astype(np.float64)), Rr)
    np.testing.assert_allclose(cov / scale, cov_r / scale, rtol=0, atol=5e-6)
