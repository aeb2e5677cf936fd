"""Evaluation metrics on the device.

Mirrors the reference's `pkg/src/meshsplat/metrics.py`: squared Chamfer
distance and normal consistency between area-uniform surface samples
(`:40-86`), PSNR and single-scale SSIM (`:89-160`), `image_metrics`
(`:163-172`).

The surface samples are the reference's exact sample sets: the uniforms are
its per-chunk Philox streams keyed by (seed, chunk) (numpy, host), and the
facet CDF, search and triangle fold run on the device with numpy's float64
rounding (`gmr_surface_prepare` / `gmr_surface_sample`; reference
`mesh.py:560-622`).  The nearest-sample queries (the reference's cKDTree
queries) run on the GPU as exact float64 brute force (`gmr_chamfer_nc`),
and PSNR/SSIM as float64 kernels (`gmr_image_metrics`).  Results match the
reference to float64 rounding of the final means.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import lib as L
from .mesh import DEGENERATE_AREA_EPS, TriangleMesh

PSNR_CAP_DB = 99.0
SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03
SSIM_RANGE = 1.0
SAMPLE_CHUNK = 1 << 16
_FALLBACK_NORMAL = np.array([0.0, 0.0, 1.0])

__all__ = ["MetricReport", "DegenerateGeometryError", "mesh_area_and_normals", "sample_surface",
           "chamfer_distance", "normal_consistency", "chamfer_and_normal_consistency", "psnr", "ssim",
           "image_metrics", "PSNR_CAP_DB"]


class DegenerateGeometryError(ValueError):
    """Mesh with zero surface area (reference mesh.py)."""


@dataclass(frozen=True)
class MetricReport:
    cd: float
    nc: float
    psnr_views: tuple
    psnr_mean: float
    ssim_views: tuple
    ssim_mean: float


def mesh_area_and_normals(mesh: TriangleMesh):
    """Per-facet (area, unit normal along the winding, degenerate flag)
    (reference mesh.py:560-577), float64 on the host (a small helper; the
    sampler computes the same quantities on the device)."""
    v, f = mesh.vertices, mesh.facets
    if len(f) == 0:
        return np.zeros(0), np.zeros((0, 3)), np.zeros(0, dtype=bool)
    cr = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    twice = np.linalg.norm(cr, axis=1)
    area = 0.5 * twice
    degen = area < DEGENERATE_AREA_EPS
    nrm = cr / np.where(degen, 1.0, twice)[:, None]
    nrm[degen] = _FALLBACK_NORMAL
    return area, nrm, degen


def uniforms(n: int, seed: int) -> np.ndarray:
    """The reference's sample stream (mesh.py:602-608): chunks of 2^16
    triples, chunk ci from Philox(SeedSequence([seed, ci]))."""
    out = np.empty((n, 3))
    for ci, s in enumerate(range(0, n, SAMPLE_CHUNK)):
        m = min(SAMPLE_CHUNK, n - s)
        out[s:s + m] = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, ci]))).random((m, 3))
    return out


class SurfaceSampler:
    """Device state of `sample_surface` for one mesh: per-facet areas,
    normals, sorted corners and the area CDF, prepared once
    (gmr_surface_prepare, numpy's float64 rounding), then any number of
    sample sets (gmr_surface_sample) from the reference's Philox stream."""

    def __init__(self, mesh: TriangleMesh):
        import torch
        lib = L.load()
        self.dev = _device()
        if len(mesh.facets) == 0:
            raise DegenerateGeometryError("mesh has zero surface area")
        self.pos = torch.tensor(np.asarray(mesh.vertices, np.float64), device=self.dev)
        self.faces = torch.tensor(np.asarray(mesh.facets), dtype=torch.int32, device=self.dev)
        self.F = int(self.faces.shape[0])
        sz = ctypes.c_size_t()
        L.check(lib.gmr_surface_prepare_size(self.F, ctypes.byref(sz)))
        self.prep = torch.empty(sz.value, dtype=torch.uint8, device=self.dev)
        total = torch.empty(1, dtype=torch.float64, device=self.dev)
        L.check(lib.gmr_surface_prepare(self.pos.data_ptr(), self.faces.data_ptr(), int(self.pos.shape[0]), self.F,
                                        self.prep.data_ptr(), sz.value, total.data_ptr(), _stream()))
        if not float(total.item()) > 0.0:
            raise DegenerateGeometryError("mesh has zero surface area")

    def sample(self, n: int, seed: int = 0):
        """(points [n,3], normals [n,3]) float64 device tensors."""
        import torch
        u = torch.tensor(uniforms(n, seed), device=self.dev)
        pts = torch.empty((n, 3), dtype=torch.float64, device=self.dev)
        nrm = torch.empty((n, 3), dtype=torch.float64, device=self.dev)
        L.check(L.load().gmr_surface_sample(self.pos.data_ptr(), self.F, self.prep.data_ptr(), u.data_ptr(), n,
                                            pts.data_ptr(), nrm.data_ptr(), _stream()))
        return pts, nrm


def sample_surface(mesh: TriangleMesh, n: int, seed: int = 0):
    """Area-uniform samples and facet normals (reference mesh.py:580-622):
    the same points and normals, computed on the device.  Returns numpy
    (points (n,3), normals (n,3))."""
    pts, nrm = SurfaceSampler(mesh).sample(n, seed)
    return pts.cpu().numpy(), nrm.cpu().numpy()


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _device():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def _pass_means(pa, na, pb, nb):
    """(mean d2 a->b, mean d2 b->a, mean |cos| a, mean |cos| b) of device
    sample sets (gmr_chamfer_nc)."""
    import torch
    lib = L.load()
    sz = ctypes.c_size_t()
    L.check(lib.gmr_chamfer_scratch_size(len(pa), len(pb), ctypes.byref(sz)))
    scratch = torch.empty(sz.value, dtype=torch.uint8, device=pa.device)
    out = torch.zeros(4, dtype=torch.float64, device=pa.device)
    ptr = lambda x: None if x is None else ctypes.c_void_p(x.data_ptr())
    L.check(lib.gmr_chamfer_nc(ptr(pa), ptr(na), len(pa), ptr(pb), ptr(nb), len(pb), ptr(out), ptr(scratch),
                               sz.value, _stream()))
    return out.cpu().numpy()


def _cd_nc_pass(sp, sg, n_samples, seed_pred, seed_gt, want_nc=True):
    pts_p, nrm_p = sp.sample(n_samples, seed_pred)
    pts_g, nrm_g = sg.sample(n_samples, seed_gt)
    m = _pass_means(pts_p, nrm_p if want_nc else None, pts_g, nrm_g if want_nc else None)
    return 0.5 * (float(m[0]) + float(m[1])), 0.5 * (float(m[2]) + float(m[3]))


def chamfer_and_normal_consistency(pred: TriangleMesh, gt: TriangleMesh, n_samples: int = 100_000,
                                   seed: int = 0, gt_seed: Optional[int] = None):
    """Both metrics from one set of nearest-sample queries (the reference
    runs the same queries twice, once per metric)."""
    sp, sg = SurfaceSampler(pred), SurfaceSampler(gt)
    if gt_seed is not None:
        return _cd_nc_pass(sp, sg, n_samples, seed, gt_seed)
    a = _cd_nc_pass(sp, sg, n_samples, seed, seed + 1)
    b = _cd_nc_pass(sp, sg, n_samples, seed + 1, seed)
    return 0.5 * (a[0] + b[0]), 0.5 * (a[1] + b[1])


def chamfer_distance(pred: TriangleMesh, gt: TriangleMesh, n_samples: int = 100_000, seed: int = 0,
                     gt_seed: Optional[int] = None) -> float:
    """Symmetric squared Chamfer distance (metrics.py:49-66): both stream
    assignments averaged unless `gt_seed` fixes it."""
    sp, sg = SurfaceSampler(pred), SurfaceSampler(gt)
    if gt_seed is not None:
        return _cd_nc_pass(sp, sg, n_samples, seed, gt_seed, False)[0]
    return 0.5 * (_cd_nc_pass(sp, sg, n_samples, seed, seed + 1, False)[0]
                  + _cd_nc_pass(sp, sg, n_samples, seed + 1, seed, False)[0])


def normal_consistency(pred: TriangleMesh, gt: TriangleMesh, n_samples: int = 100_000, seed: int = 0,
                       gt_seed: Optional[int] = None) -> float:
    """Mean |cos| between normals at nearest-sample pairs (metrics.py:79-86)."""
    sp, sg = SurfaceSampler(pred), SurfaceSampler(gt)
    if gt_seed is not None:
        return _cd_nc_pass(sp, sg, n_samples, seed, gt_seed)[1]
    return 0.5 * (_cd_nc_pass(sp, sg, n_samples, seed, seed + 1)[1]
                  + _cd_nc_pass(sp, sg, n_samples, seed + 1, seed)[1])


def _image_stats(a, b, want_ssim):
    """a, b [B,H,W,C] float64 -> (mse [B], ssim [B] or None) on the GPU."""
    import torch
    lib = L.load()
    dev = _device()
    ta = torch.tensor(np.ascontiguousarray(a, np.float64), device=dev)
    tb = torch.tensor(np.ascontiguousarray(b, np.float64), device=dev)
    B, H, W, C = ta.shape
    sz = ctypes.c_size_t()
    L.check(lib.gmr_image_metrics_scratch_size(B, H, W, C, ctypes.byref(sz)))
    scratch = torch.empty(sz.value, dtype=torch.uint8, device=dev)
    mse = torch.empty(B, dtype=torch.float64, device=dev)
    ss = torch.empty(B, dtype=torch.float64, device=dev) if want_ssim else None
    L.check(lib.gmr_image_metrics(ta.data_ptr(), tb.data_ptr(), B, H, W, C, mse.data_ptr(),
                                  None if ss is None else ss.data_ptr(), scratch.data_ptr(), sz.value,
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return mse.cpu().numpy(), None if ss is None else ss.cpu().numpy()


def _as_batch(img_a, img_b):
    a = np.asarray(img_a, dtype=np.float64)
    b = np.asarray(img_b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    return a, b


def _psnr_of(mse: float) -> float:
    if mse == 0.0:
        return PSNR_CAP_DB
    return min(10.0 * np.log10(1.0 / mse), PSNR_CAP_DB)


def psnr(img_a, img_b) -> float:
    """PSNR in dB for unit-range images, capped at 99 dB (metrics.py:89-99)."""
    a, b = _as_batch(img_a, img_b)
    x = a.reshape(1, *a.shape[:2], -1) if a.ndim >= 2 else a.reshape(1, 1, -1, 1)
    y = b.reshape(x.shape)
    return _psnr_of(float(_image_stats(x, y, False)[0][0]))


def _ssim_shape(a):
    if a.ndim == 2:
        a = a[..., None]
    if a.ndim != 3:
        raise ValueError("expected HxW or HxWxC images")
    if min(a.shape[0], a.shape[1]) < SSIM_WINDOW:
        raise ValueError(f"images must be at least {SSIM_WINDOW} pixels on each side")
    return a


def ssim(img_a, img_b) -> float:
    """Single-scale SSIM, Gaussian windows, channel-averaged, interior mean
    (metrics.py:116-160)."""
    a, b = _as_batch(img_a, img_b)
    a, b = _ssim_shape(a), _ssim_shape(b)
    return float(_image_stats(a[None], b[None], True)[1][0])


def image_metrics(rendered: Sequence[np.ndarray], targets: Sequence[np.ndarray]):
    """Per-view PSNR and SSIM (metrics.py:163-172); views of one shape are
    evaluated in one batched device call."""
    if len(rendered) != len(targets):
        raise ValueError("view count mismatch")
    n = len(rendered)
    ps, ss = [0.0] * n, [0.0] * n
    groups = {}
    for i, (r, t) in enumerate(zip(rendered, targets)):
        a, b = _as_batch(r, t)
        a, b = _ssim_shape(a), _ssim_shape(b)
        groups.setdefault(a.shape, []).append((i, a, b))
    for items in groups.values():
        mse, sv = _image_stats(np.stack([x[1] for x in items]), np.stack([x[2] for x in items]), True)
        for (i, _, _), m, s in zip(items, mse, sv):
            ps[i] = _psnr_of(float(m))
            ss[i] = float(s)
    return tuple(ps), tuple(ss)
