"""Export / metrics CPU oracle — TEST INFRASTRUCTURE ONLY.

numpy restatement of the reference's `export_gaussians` (convert.py:444-532)
and of its metrics (metrics.py:40-172).  Only `tests/` may import it, as the
checker.  Nearest-sample queries use scipy's cKDTree, exactly as the
reference does (scipy is the reference's own dependency,
`pkg/pyproject.toml`); the SSIM window filter is restated with explicit
'reflect' indexing instead of scipy.ndimage.

Pinned by tests/golden/eval_ico320.npz (made by the real reference,
tests/golden/make_golden.py `eval_case`) in tests/test_eval.py.
"""

from __future__ import annotations

import numpy as np

S_Z = 1e-6                     # convert.py:27
SH_DC = 0.28209479177387814    # convert.py:29
OPACITY_CLAMP = 1e-6           # convert.py:30
PSNR_CAP_DB = 99.0             # metrics.py:20
SSIM_WINDOW, SSIM_SIGMA, SSIM_K1, SSIM_K2 = 11, 1.5, 0.01, 0.03   # metrics.py:22-26


def quaternions(rot):
    """Rotation matrices -> unit (w, x, y, z), w >= 0 (convert.py:444-481)."""
    m = np.asarray(rot, np.float64)
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    q = np.empty((len(m), 4))
    b0 = tr > 0
    b1 = ~b0 & (m[:, 0, 0] >= m[:, 1, 1]) & (m[:, 0, 0] >= m[:, 2, 2])
    b2 = ~b0 & ~b1 & (m[:, 1, 1] >= m[:, 2, 2])
    b3 = ~(b0 | b1 | b2)
    for sel, diag, cols in ((b0, None, None), (b1, 0, (1, 2)), (b2, 1, (0, 2)), (b3, 2, (0, 1))):
        i = np.where(sel)[0]
        if not len(i):
            continue
        M = m[i]
        if diag is None:
            r = np.sqrt(1.0 + tr[i]) * 2.0
            q[i] = np.stack([0.25 * r, (M[:, 2, 1] - M[:, 1, 2]) / r, (M[:, 0, 2] - M[:, 2, 0]) / r,
                             (M[:, 1, 0] - M[:, 0, 1]) / r], axis=1)
        elif diag == 0:
            r = np.sqrt(1.0 + M[:, 0, 0] - M[:, 1, 1] - M[:, 2, 2]) * 2.0
            q[i] = np.stack([(M[:, 2, 1] - M[:, 1, 2]) / r, 0.25 * r, (M[:, 0, 1] + M[:, 1, 0]) / r,
                             (M[:, 0, 2] + M[:, 2, 0]) / r], axis=1)
        elif diag == 1:
            r = np.sqrt(1.0 + M[:, 1, 1] - M[:, 0, 0] - M[:, 2, 2]) * 2.0
            q[i] = np.stack([(M[:, 0, 2] - M[:, 2, 0]) / r, (M[:, 0, 1] + M[:, 1, 0]) / r, 0.25 * r,
                             (M[:, 1, 2] + M[:, 2, 1]) / r], axis=1)
        else:
            r = np.sqrt(1.0 + M[:, 2, 2] - M[:, 0, 0] - M[:, 1, 1]) * 2.0
            q[i] = np.stack([(M[:, 1, 0] - M[:, 0, 1]) / r, (M[:, 0, 2] + M[:, 2, 0]) / r,
                             (M[:, 1, 2] + M[:, 2, 1]) / r, 0.25 * r], axis=1)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1.0
    return q


def export_records(means, cov3d, colors, opacities):
    """The 14 float32 fields per Gaussian (convert.py:497-532)."""
    lam, vec = np.linalg.eigh(np.asarray(cov3d, np.float64))
    lam, vec = lam[:, ::-1], vec[:, :, ::-1].copy()
    vec[np.linalg.det(vec) < 0, :, 2] *= -1.0
    scales = np.sqrt(np.maximum(lam, S_Z * S_Z * 1e-2))
    op = np.clip(opacities, OPACITY_CLAMP, 1.0 - OPACITY_CLAMP)
    rec = np.empty((len(means), 14), np.float32)
    rec[:, 0:3] = np.asarray(means).astype(np.float32)
    rec[:, 3:6] = (np.asarray(colors) - 0.5) / SH_DC
    rec[:, 6] = np.log(op / (1.0 - op))
    rec[:, 7:10] = np.log(scales)
    rec[:, 10:14] = quaternions(vec)
    return rec


def quat_to_rot(q):
    w, x, y, z = (np.asarray(q, np.float64)[:, k] for k in range(4))
    return np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
                     np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
                     np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)


def chamfer_nc_pass(pts_p, nrm_p, pts_g, nrm_g):
    """One (CD, NC) pass (metrics.py:40-46, :69-77) with cKDTree."""
    from scipy.spatial import cKDTree
    d_pg, i_pg = cKDTree(pts_g).query(pts_p)
    d_gp, i_gp = cKDTree(pts_p).query(pts_g)
    cd = 0.5 * (float(np.mean(d_pg ** 2)) + float(np.mean(d_gp ** 2)))
    nc = 0.5 * (float(np.abs(np.sum(nrm_p * nrm_g[i_pg], axis=1)).mean())
                + float(np.abs(np.sum(nrm_g * nrm_p[i_gp], axis=1)).mean()))
    return cd, nc


def psnr(a, b):
    """metrics.py:89-99."""
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return PSNR_CAP_DB if mse == 0.0 else min(10.0 * np.log10(1.0 / mse), PSNR_CAP_DB)


def _reflect(i, n):
    period = 2 * n
    i = np.mod(i, period)
    return np.where(i < n, i, period - 1 - i)


def _filter(img, k, axis):
    half = len(k) // 2
    n = img.shape[axis]
    out = np.zeros_like(img)
    for t in range(len(k)):
        idx = _reflect(np.arange(n) + t - half, n)
        out += k[t] * np.take(img, idx, axis=axis)
    return out


def ssim(a, b):
    """metrics.py:116-160 (Gaussian window, reflect borders, interior mean)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.ndim == 2:
        a, b = a[..., None], b[..., None]
    half = (SSIM_WINDOW - 1) // 2
    x = np.arange(-half, half + 1, dtype=np.float64)
    k = np.exp(-(x * x) / (2.0 * SSIM_SIGMA ** 2))
    k = k / k.sum()
    w = lambda im: _filter(_filter(im, k, 0), k, 1)
    c1, c2 = SSIM_K1 ** 2, SSIM_K2 ** 2
    scores = []
    for ch in range(a.shape[2]):
        X, Y = a[..., ch], b[..., ch]
        mx, my = w(X), w(Y)
        xx, yy, xy = w(X * X) - mx * mx, w(Y * Y) - my * my, w(X * Y) - mx * my
        smap = ((2 * mx * my + c1) * (2 * xy + c2)) / ((mx ** 2 + my ** 2 + c1) * (xx + yy + c2))
        scores.append(float(np.mean(smap[half:-half, half:-half])))
    return float(np.mean(scores))


def sample_surface(vertices, facets, n, seed=0):
    """Area-uniform samples + facet normals (mesh.py:560-622)."""
    v = np.asarray(vertices, np.float64)
    f = np.asarray(facets, np.int64)
    cr = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    twice = np.linalg.norm(cr, axis=1)
    area = 0.5 * twice
    degen = area < 1e-12
    nrm = cr / np.where(degen, 1.0, twice)[:, None]
    nrm[degen] = (0.0, 0.0, 1.0)
    cdf = np.cumsum(area) / area.sum()
    fs = np.sort(f, axis=1)
    pts, out_n = np.empty((n, 3)), np.empty((n, 3))
    for ci, s in enumerate(range(0, n, 1 << 16)):
        m = min(1 << 16, n - s)
        u = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, ci]))).random((m, 3))
        fi = np.minimum(np.searchsorted(cdf, u[:, 0], side="left"), len(fs) - 1)
        fold = u[:, 1] + u[:, 2] > 1.0
        b1, b2 = np.where(fold, 1.0 - u[:, 1], u[:, 1]), np.where(fold, 1.0 - u[:, 2], u[:, 2])
        a = v[fs[fi, 0]]
        pts[s:s + m] = a + b1[:, None] * (v[fs[fi, 1]] - a) + b2[:, None] * (v[fs[fi, 2]] - a)
        out_n[s:s + m] = nrm[fi]
    return pts, out_n
