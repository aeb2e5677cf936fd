"""GMR CPU oracle — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's render hot path (meshsplat, pure numpy,
`/root/reference/pkg/src/meshsplat`).  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs may import this
module, and only as the checker / the timed CPU baseline.  The product
(`paper_2602_14493_b200`) never imports it and has no CPU fallback.

Parity is pinned: `tests/golden/make_golden.py` runs the real reference (in
the build container, where `/root/reference` exists) on seeded inputs and
commits the outputs; `tests/test_oracle.py` checks this restatement against
those fixtures (and, when the reference is importable, against it directly).

Every function cites the reference lines it restates.  Arithmetic follows the
reference's operation order so fp64 results agree to the last few ulps.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# render.py:26-30, convert.py:27-28, mesh.py:15
TILE = 16
ALPHA_CLAMP = 0.99
CONTRIB_FLOOR = 1.0 / 255.0
TRANSMITTANCE_STOP = 1e-4
DILATION = 0.3
S_Z = 1e-6
DET_EPS = 1e-14
DEGENERATE_AREA_EPS = 1e-12
BCE_CLAMP = 1e-6  # losses.py:20


# ---------------------------------------------------------------------------
# facet -> Gaussian (convert.py:239-276, :313-343)
# ---------------------------------------------------------------------------

def facet_geometry(vertices, facets, rescale=True):
    """Embed-route intermediates per facet (convert.py:239-276)."""
    va = vertices[facets[:, 0]]
    vb = vertices[facets[:, 1]]
    vc = vertices[facets[:, 2]]
    e1 = vb - va
    e2 = vc - va
    e3 = vc - vb
    outer = lambda e: np.einsum("mi,mj->mij", e, e)
    c3 = (outer(e1) + outer(e2) + outer(e3)) / 36.0
    u = np.cross(e1, e2)
    nu = np.linalg.norm(u, axis=1)
    area = 0.5 * nu
    degenerate = area < DEGENERATE_AREA_EPS
    nu_safe = np.where(degenerate, 1.0, nu)
    normal = u / nu_safe[:, None]
    det2d = area * area / 108.0
    clamped = det2d < DET_EPS
    if rescale:
        kappa = area / (np.pi * np.sqrt(np.maximum(det2d, DET_EPS)))
    else:
        kappa = np.ones_like(area)
    cov3d = kappa[:, None, None] * c3 + (S_Z * S_Z) * np.einsum("mi,mj->mij", normal, normal)
    cov3d[degenerate] = S_Z * S_Z * np.eye(3)
    return dict(e1=e1, e2=e2, u=u, nu=nu_safe, normal=normal, area=area, det2d=det2d,
                clamped=clamped, kappa=kappa, c3=c3, cov3d=cov3d, degenerate=degenerate)


def facet_gaussians(vertices, facets, colors, rescale=True):
    """Per-facet (means, cov3d, colors, opacities) of the embed route
    (convert.py:321-326 + :343)."""
    f = facets
    col = (colors[f[:, 0]] + colors[f[:, 1]] + colors[f[:, 2]]) / 3.0
    mean = (vertices[f[:, 0]] + vertices[f[:, 1]] + vertices[f[:, 2]]) / 3.0
    geo = facet_geometry(vertices, facets, rescale)
    return dict(means=mean, cov3d=geo["cov3d"], colors=col, opacities=np.ones(len(f)),
                degenerate=geo["degenerate"], rescale=rescale)


# ---------------------------------------------------------------------------
# EWA projection (render.py:76-145)
# ---------------------------------------------------------------------------

def _conic(cov2d):
    a, b, c = cov2d[:, 0, 0], cov2d[:, 0, 1], cov2d[:, 1, 1]
    det = a * c - b * b
    return np.stack([c / det, -b / det, a / det], axis=1)          # render.py:76-81


def _radius3(cov2d):
    a, b, c = cov2d[:, 0, 0], cov2d[:, 0, 1], cov2d[:, 1, 1]
    return 3.0 * np.sqrt(0.5 * (a + c) + np.hypot(0.5 * (a - c), b))  # render.py:84-88,124


def _jacobian(t, fx, fy):
    """render.py:91-100 (no FoV clamp)."""
    z = t[:, 2]
    jac = np.zeros((len(t), 2, 3), dtype=t.dtype)
    jac[:, 0, 0] = fx / z
    jac[:, 0, 2] = -fx * t[:, 0] / (z * z)
    jac[:, 1, 1] = fy / z
    jac[:, 1, 2] = -fy * t[:, 1] / (z * z)
    return jac


@dataclass
class Splats:
    """Kept splats in source order (render.py:52-73)."""
    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    source: np.ndarray
    t_cam: np.ndarray
    radius: np.ndarray

    def __len__(self):
        return len(self.depth)


def _empty_splats(dtype):
    z = lambda *s: np.zeros(s, dtype=dtype)
    return Splats(z(0, 2), z(0, 2, 2), z(0, 3), z(0), z(0, 3), z(0),
                  np.zeros(0, np.int64), z(0, 3), z(0))


def project(cloud, cam, dtype=np.float64) -> Splats:
    """render.py:103-145: camera transform, strict near/far cull on the mean,
    EWA covariance + 0.3 px^2 dilation, 3-sigma screen cull."""
    rot = np.asarray(cam.rotation).astype(dtype)
    t_all = cloud["means"].astype(dtype) @ rot.T + np.asarray(cam.translation).astype(dtype)
    keep = np.where((t_all[:, 2] > cam.near) & (t_all[:, 2] < cam.far))[0]
    if len(keep) == 0:
        return _empty_splats(dtype)
    t = t_all[keep]
    m2 = _jacobian(t, cam.fx, cam.fy) @ rot
    cov2d = np.einsum("kpi,kij,kqj->kpq", m2, cloud["cov3d"][keep].astype(dtype), m2)
    cov2d[:, 0, 0] += DILATION
    cov2d[:, 1, 1] += DILATION
    z = t[:, 2]
    mean2d = np.stack([cam.fx * t[:, 0] / z + cam.cx, cam.fy * t[:, 1] / z + cam.cy], axis=1)
    radius = _radius3(cov2d)
    onscreen = ((mean2d[:, 0] + radius >= -0.5) & (mean2d[:, 0] - radius <= cam.width - 0.5)
                & (mean2d[:, 1] + radius >= -0.5) & (mean2d[:, 1] - radius <= cam.height - 0.5))
    sel = np.where(onscreen)[0]
    if len(sel) == 0:
        return _empty_splats(dtype)
    src = keep[sel]
    return Splats(mean2d=mean2d[sel], cov2d=cov2d[sel], conic=_conic(cov2d[sel]), depth=z[sel],
                  color=cloud["colors"][src].astype(dtype),
                  opacity=cloud["opacities"][src].astype(dtype),
                  source=src, t_cam=t[sel], radius=radius[sel])


def splats_from_arrays(mean2d, cov2d, depth, color, opacity, source=None, dtype=np.float64):
    """`_batch_from_splats` (render.py:168-188) for array input."""
    mean2d = np.asarray(mean2d, dtype=dtype).reshape(-1, 2)
    k = len(mean2d)
    if k == 0:
        return _empty_splats(dtype)
    cov2d = np.asarray(cov2d, dtype=dtype).reshape(k, 2, 2)
    if source is None:
        source = np.arange(k)
    return Splats(mean2d=mean2d, cov2d=cov2d, conic=_conic(cov2d),
                  depth=np.asarray(depth, dtype=dtype).reshape(k),
                  color=np.asarray(color, dtype=dtype).reshape(k, 3),
                  opacity=np.asarray(opacity, dtype=dtype).reshape(k),
                  source=np.asarray(source, dtype=np.int64).reshape(k),
                  t_cam=np.zeros((k, 3), dtype=dtype), radius=_radius3(cov2d))


def check_finite(s: Splats):
    """render.py:191-197 (same message)."""
    for name in ("mean2d", "cov2d", "conic", "depth", "color", "opacity"):
        bad = ~np.isfinite(getattr(s, name))
        if bad.any():
            raise ValueError(f"non-finite splat parameter {name!r} at splat {int(np.argwhere(bad)[0][0])}")


# ---------------------------------------------------------------------------
# tile binning (render.py:200-232)
# ---------------------------------------------------------------------------

def tile_rects(mean2d, radius, width, height):
    """Inclusive floor-based tile rectangles clipped to the grid
    (render.py:214-217). Returns (tx0, tx1, ty0, ty1) int64."""
    ntx = (width + TILE - 1) // TILE
    nty = (height + TILE - 1) // TILE
    mx, my = mean2d[:, 0], mean2d[:, 1]
    clipx = lambda v: np.clip(np.floor(v / TILE).astype(np.int64), 0, ntx - 1)
    clipy = lambda v: np.clip(np.floor(v / TILE).astype(np.int64), 0, nty - 1)
    return clipx(mx - radius), clipx(mx + radius), clipy(my - radius), clipy(my + radius)


def bin_splats(mean2d, radius, depth, source, width, height):
    """(entry_splat, bounds): entries sorted by (tile, depth, source)
    (render.py:200-229).  entry_splat indexes the splat arrays."""
    ntx = (width + TILE - 1) // TILE
    n_tiles = ntx * ((height + TILE - 1) // TILE)
    k = len(depth)
    if k == 0:
        return np.zeros(0, np.int64), np.zeros(n_tiles + 1, np.int64)
    tx0, tx1, ty0, ty1 = tile_rects(mean2d, radius, width, height)
    nx = tx1 - tx0 + 1
    counts = nx * (ty1 - ty0 + 1)
    owner = np.repeat(np.arange(k), counts)
    first = np.cumsum(counts) - counts
    local = np.arange(int(counts.sum())) - first[owner]
    tile = (ty0[owner] + local // nx[owner]) * ntx + tx0[owner] + local % nx[owner]
    order = np.lexsort((source[owner], depth[owner], tile))
    return owner[order], np.searchsorted(tile[order], np.arange(n_tiles + 1))


# ---------------------------------------------------------------------------
# blend forward / backward (render.py:235-361)
# ---------------------------------------------------------------------------

def _tile_grid(tid, ntx, width, height, dtype):
    ty, tx = divmod(tid, ntx)
    u0, v0 = tx * TILE, ty * TILE
    u1, v1 = min(u0 + TILE, width), min(v0 + TILE, height)
    uu, vv = np.meshgrid(np.arange(u0, u1, dtype=dtype), np.arange(v0, v1, dtype=dtype))
    return uu.ravel(), vv.ravel(), (v0, v1, u0, u1)


def _blend_terms(s: Splats, ids, uu, vv):
    """(pixels x splats) compositing terms of one tile (render.py:244-269)."""
    ca, cb, cc = s.conic[ids, 0], s.conic[ids, 1], s.conic[ids, 2]
    dx = uu[:, None] - s.mean2d[ids, 0][None, :]
    dy = vv[:, None] - s.mean2d[ids, 1][None, :]
    power = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy
    ep = np.exp(power)
    raw = s.opacity[ids] * ep
    alpha = np.minimum(ALPHA_CLAMP, raw)
    visible = alpha >= CONTRIB_FLOOR
    reach = np.cumprod(1.0 - np.where(visible, alpha, 0.0), axis=1)
    used = visible & (reach >= TRANSMITTANCE_STOP)
    keep = np.cumprod(1.0 - np.where(used, alpha, 0.0), axis=1)
    trans = np.empty_like(keep)
    trans[:, 0] = 1.0
    trans[:, 1:] = keep[:, :-1]
    weight = np.where(used, alpha * trans, 0.0)
    return dict(dx=dx, dy=dy, ep=ep, raw=raw, alpha=alpha, used=used, trans=trans,
                weight=weight, t_final=keep[:, -1])


def composite(s: Splats, width, height, background=(0.0, 0.0, 0.0), dtype=np.float64,
              tiles=None):
    """Front-to-back blend over a constant background (render.py:272-291).
    Returns (rgb HxWx3, alpha HxW).  `tiles` (timing only) restricts the
    per-tile loop to a subset of tile ids."""
    check_finite(s)
    bg = np.asarray(background, dtype=dtype)
    rgb = np.empty((height, width, 3), dtype=dtype)
    rgb[:] = bg
    alpha = np.zeros((height, width), dtype=dtype)
    ntx = (width + TILE - 1) // TILE
    entry, bounds = bin_splats(s.mean2d, s.radius, s.depth, s.source, width, height)
    for tid in (range(len(bounds) - 1) if tiles is None else tiles):
        ids = entry[bounds[tid]:bounds[tid + 1]]
        if len(ids) == 0:
            continue
        uu, vv, (r0, r1, c0, c1) = _tile_grid(tid, ntx, width, height, dtype)
        t = _blend_terms(s, ids, uu, vv)
        px = t["weight"] @ s.color[ids] + t["t_final"][:, None] * bg[None, :]
        rgb[r0:r1, c0:c1] = px.reshape(r1 - r0, c1 - c0, 3)
        alpha[r0:r1, c0:c1] = (1.0 - t["t_final"]).reshape(r1 - r0, c1 - c0)
    return rgb, alpha


def composite_backward(s: Splats, width, height, background, grad_rgb, grad_alpha,
                       dtype=np.float64, tiles=None):
    """Screen-space gradients (g_mean2d, g_cov2d, g_color, g_opacity) of
    sum(g_rgb*rgb)+sum(g_alpha*alpha), tile-major accumulation
    (render.py:294-361)."""
    check_finite(s)
    grad_rgb = np.asarray(grad_rgb, dtype=dtype)
    grad_alpha = np.asarray(grad_alpha, dtype=dtype)
    if grad_rgb.shape != (height, width, 3) or grad_alpha.shape != (height, width):
        raise ValueError("upstream gradient shapes do not match the image")
    bg = np.asarray(background, dtype=dtype)
    k = len(s)
    g_mean = np.zeros((k, 2), dtype=dtype)
    g_cov = np.zeros((k, 2, 2), dtype=dtype)
    g_col = np.zeros((k, 3), dtype=dtype)
    g_op = np.zeros(k, dtype=dtype)
    ntx = (width + TILE - 1) // TILE
    entry, bounds = bin_splats(s.mean2d, s.radius, s.depth, s.source, width, height)
    for tid in (range(len(bounds) - 1) if tiles is None else tiles):
        ids = entry[bounds[tid]:bounds[tid + 1]]
        if len(ids) == 0:
            continue
        uu, vv, (r0, r1, c0, c1) = _tile_grid(tid, ntx, width, height, dtype)
        t = _blend_terms(s, ids, uu, vv)
        g_px = grad_rgb[r0:r1, c0:c1].reshape(-1, 3)
        ga_px = grad_alpha[r0:r1, c0:c1].reshape(-1)
        gc = g_px @ s.color[ids].T
        contrib = gc * t["weight"]
        after = np.cumsum(contrib[:, ::-1], axis=1)[:, ::-1] - contrib
        tail = (g_px @ bg - ga_px) * t["t_final"]
        one_minus = 1.0 - np.where(t["used"], t["alpha"], 0.0)
        d_alpha = np.where(t["used"], gc * t["trans"] - (after + tail[:, None]) / one_minus, 0.0)
        live = t["raw"] < ALPHA_CLAMP                                   # clamp gate :336
        d_pow = np.where(live, d_alpha * t["alpha"], 0.0)
        g_op[ids] += np.einsum("pk,pk->k", np.where(live, d_alpha, 0.0), t["ep"])
        g_col[ids] += t["weight"].T @ g_px
        ca, cb, cc = s.conic[ids, 0], s.conic[ids, 1], s.conic[ids, 2]
        dx, dy = t["dx"], t["dy"]
        g_mean[ids, 0] += np.einsum("pk,pk->k", d_pow, ca * dx + cb * dy)
        g_mean[ids, 1] += np.einsum("pk,pk->k", d_pow, cc * dy + cb * dx)
        q00 = -0.5 * np.einsum("pk,pk->k", d_pow, dx * dx)
        q01 = -0.5 * np.einsum("pk,pk->k", d_pow, dx * dy)
        q11 = -0.5 * np.einsum("pk,pk->k", d_pow, dy * dy)
        m = np.empty((len(ids), 2, 2), dtype=dtype)
        m[:, 0, 0], m[:, 0, 1], m[:, 1, 0], m[:, 1, 1] = ca, cb, cb, cc
        q = np.empty_like(m)
        q[:, 0, 0], q[:, 0, 1], q[:, 1, 0], q[:, 1, 1] = q00, q01, q01, q11
        g_cov[ids] += -np.einsum("kab,kbc,kcd->kad", m, q, m)          # dL/dSigma = -M G M
    return g_mean, g_cov, g_col, g_op


# ---------------------------------------------------------------------------
# projection / conversion backward (render.py:364-402, convert.py:371-437)
# ---------------------------------------------------------------------------

def project_backward(s: Splats, cloud, cam, g_mean2d, g_cov2d):
    """(g_mean3d, g_cov3d) aligned with splat order (render.py:364-402)."""
    dtype = s.mean2d.dtype
    rot = np.asarray(cam.rotation).astype(dtype)
    t = s.t_cam
    tx, ty, tz = t[:, 0], t[:, 1], t[:, 2]
    fx, fy = dtype.type(cam.fx), dtype.type(cam.fy)
    m2 = _jacobian(t, cam.fx, cam.fy) @ rot
    cov3d = cloud["cov3d"][s.source].astype(dtype)
    g2 = np.asarray(g_cov2d, dtype=dtype)
    gm = np.asarray(g_mean2d, dtype=dtype)
    g_cov3d = np.einsum("kpq,kpi,kqj->kij", g2, m2, m2)
    g_m2 = np.einsum("kpq,kqi,kij->kpj", g2 + g2.transpose(0, 2, 1), m2, cov3d)
    g_j = np.einsum("kpi,ji->kpj", g_m2, rot)
    iz = 1.0 / tz
    iz2 = iz * iz
    g_tx = -fx * iz2 * g_j[:, 0, 2]
    g_ty = -fy * iz2 * g_j[:, 1, 2]
    g_tz = (-fx * iz2 * g_j[:, 0, 0] - fy * iz2 * g_j[:, 1, 1]
            + 2.0 * fx * tx * iz2 * iz * g_j[:, 0, 2] + 2.0 * fy * ty * iz2 * iz * g_j[:, 1, 2])
    g_tx += gm[:, 0] * fx * iz
    g_ty += gm[:, 1] * fy * iz
    g_tz += -gm[:, 0] * fx * tx * iz2 - gm[:, 1] * fy * ty * iz2
    return np.stack([g_tx, g_ty, g_tz], axis=1) @ rot, g_cov3d


def facet_backward(vertices, facets, colors, grad_means, grad_cov3d, grad_colors, rescale=True):
    """Vertex position / colour gradients (convert.py:371-437), scattered
    corner-major with np.add.at (:427-436)."""
    m = len(facets)
    grad_means = np.asarray(grad_means, dtype=np.float64)
    grad_cov3d = np.asarray(grad_cov3d, dtype=np.float64)
    grad_colors = np.asarray(grad_colors, dtype=np.float64)
    if grad_means.shape != (m, 3) or grad_cov3d.shape != (m, 3, 3) or grad_colors.shape != (m, 3):
        raise ValueError(f"gradient shapes {grad_means.shape}, {grad_cov3d.shape}, "
                         f"{grad_colors.shape} do not match {m} facets")
    geo = facet_geometry(vertices, facets, rescale)
    live = ~geo["degenerate"]
    g = grad_cov3d
    gsym = g + g.transpose(0, 2, 1)
    d_area = np.zeros(m)
    if rescale:
        d_kappa = np.einsum("mij,mij->m", g, geo["c3"])
        hit = geo["clamped"] & live
        d_area[hit] = d_kappa[hit] / (np.pi * np.sqrt(DET_EPS))
    sk = geo["kappa"][:, None, None] * gsym / 36.0
    e1, e2 = geo["e1"], geo["e2"]
    g1 = np.einsum("mij,mj->mi", sk, e1)
    g2 = np.einsum("mij,mj->mi", sk, e2)
    g3 = np.einsum("mij,mj->mi", sk, e2 - e1)
    n = geo["normal"]
    g_n = (S_Z * S_Z) * np.einsum("mij,mj->mi", gsym, n)
    g_u = (g_n - n * np.einsum("mi,mi->m", n, g_n)[:, None]) / geo["nu"][:, None] \
        + 0.5 * d_area[:, None] * n
    g1 += np.cross(e2, g_u)
    g2 += np.cross(g_u, e1)
    for arr in (g1, g2, g3):
        arr[~live] = 0.0
    third = grad_means / 3.0
    corners = (third - g1 - g2, third + g1 - g3, third + g2 + g3)
    gv = np.zeros((len(vertices), 3))
    gc = np.zeros((len(vertices), 3))
    for c in range(3):
        np.add.at(gv, facets[:, c], corners[c])
    for c in range(3):
        np.add.at(gc, facets[:, c], grad_colors / 3.0)
    return gv, gc


# ---------------------------------------------------------------------------
# mesh-level composition (render.py:441-467) and the view loop (losses.py)
# ---------------------------------------------------------------------------

@dataclass
class Ctx:
    vertices: np.ndarray
    facets: np.ndarray
    colors: np.ndarray
    cam: object
    cloud: dict
    splats: Splats
    background: np.ndarray
    dtype: type


def render(vertices, facets, colors, cam, background=(0.0, 0.0, 0.0), rescale=True,
           dtype=np.float64):
    """render_mesh (render.py:441-450). Returns (rgb, alpha, ctx)."""
    vertices = np.asarray(vertices, np.float64)
    facets = np.asarray(facets, np.int64)
    colors = np.asarray(colors, np.float64)
    cloud = facet_gaussians(vertices, facets, colors, rescale)
    s = project(cloud, cam, dtype)
    rgb, alpha = composite(s, cam.width, cam.height, background, dtype)
    return rgb, alpha, Ctx(vertices, facets, colors, cam, cloud, s,
                           np.asarray(background, dtype), dtype)


def render_grad(ctx: Ctx, grad_rgb, grad_alpha):
    """render_backward (render.py:453-467) -> (grad_vertices, grad_colors)."""
    cam = ctx.cam
    g_mean2d, g_cov2d, g_col, _ = composite_backward(
        ctx.splats, cam.width, cam.height, ctx.background, grad_rgb, grad_alpha, ctx.dtype)
    m = len(ctx.facets)
    gm = np.zeros((m, 3))
    gc3 = np.zeros((m, 3, 3))
    gcol = np.zeros((m, 3))
    if len(ctx.splats):
        a, b = project_backward(ctx.splats, ctx.cloud, cam, g_mean2d, g_cov2d)
        gm[ctx.splats.source] = a
        gc3[ctx.splats.source] = b
        gcol[ctx.splats.source] = g_col
    return facet_backward(ctx.vertices, ctx.facets, ctx.colors, gm, gc3, gcol, ctx.cloud["rescale"])


def color_loss(rendered, target):
    """losses.py:43-56."""
    diff = np.asarray(rendered, np.float64) - np.asarray(target, np.float64)
    return float(np.mean(diff * diff)), (2.0 / diff.size) * diff


def silhouette_loss(alpha, mask):
    """losses.py:59-73."""
    alpha = np.asarray(alpha, np.float64)
    mask = np.asarray(mask, np.float64)
    p = np.clip(alpha, BCE_CLAMP, 1.0 - BCE_CLAMP)
    value = float(-np.mean(mask * np.log(p) + (1.0 - mask) * np.log1p(-p)))
    inside = (alpha > BCE_CLAMP) & (alpha < 1.0 - BCE_CLAMP)
    return value, np.where(inside, (-mask / p + (1.0 - mask) / (1.0 - p)) / alpha.size, 0.0)


def views_image_grad(vertices, facets, colors, cams, target_rgb, target_mask,
                     w_color=1.0, w_sil=1.0, background=(0.0, 0.0, 0.0), dtype=np.float64):
    """Image part of total_loss (losses.py:146-164): serial view loop, grads
    scaled by w/n and summed.  Returns (color, silhouette, grad_v, grad_c)."""
    n = len(cams)
    gv = np.zeros((len(vertices), 3))
    gc = np.zeros((len(vertices), 3))
    cval = sval = 0.0
    for cam, rt, mt in zip(cams, target_rgb, target_mask):
        rgb, alpha, ctx = render(vertices, facets, colors, cam, background, True, dtype)
        cv, g_rgb = color_loss(rgb, rt)
        sv, g_a = silhouette_loss(alpha, mt)
        cval += cv
        sval += sv
        a, b = render_grad(ctx, (w_color / n) * g_rgb, (w_sil / n) * g_a)
        gv += a
        gc += b
    return cval / n, sval / n, gv, gc


# ---------------------------------------------------------------------------
# mesh regularisers (losses.py:76-123) and the optimiser (optim.py:29-135),
# checkers for the device kernels of gmr_train.cuh
# ---------------------------------------------------------------------------

def unique_edges(facets):
    """mesh.py:96-106: unique undirected edges, smaller index first, lexsorted."""
    f = np.asarray(facets, np.int64)
    if len(f) == 0:
        return np.zeros((0, 2), np.int64)
    return np.unique(np.sort(f[:, [0, 1, 1, 2, 2, 0]].reshape(-1, 2), axis=1), axis=0)


def edge_length_loss(vertices, facets):
    """losses.py:76-97 (mean length detached; np.add.at scatter order)."""
    v = np.asarray(vertices, np.float64)
    e = unique_edges(facets)
    if len(e) == 0:
        return 0.0, np.zeros_like(v)
    vec = v[e[:, 1]] - v[e[:, 0]]
    length = np.linalg.norm(vec, axis=1)
    dev = length - length.mean()
    coeff = (2.0 / len(e)) * dev / np.maximum(length, 1e-12)
    g = np.zeros_like(v)
    np.add.at(g, e[:, 1], coeff[:, None] * vec)
    np.add.at(g, e[:, 0], -coeff[:, None] * vec)
    return float(np.mean(dev * dev)), g


def laplacian_loss(vertices, facets):
    """losses.py:100-123 (uniform Laplacian over the sorted neighbour lists,
    mesh.py:114-126)."""
    v = np.asarray(vertices, np.float64)
    nv = len(v)
    e = unique_edges(facets)
    both = np.concatenate([e, e[:, ::-1]]) if len(e) else np.zeros((0, 2), np.int64)
    both = both[np.lexsort((both[:, 1], both[:, 0]))]
    deg = np.bincount(both[:, 0], minlength=nv).astype(np.float64)
    has = deg > 0
    nbr = np.zeros_like(v)
    np.add.at(nbr, both[:, 0], v[both[:, 1]])
    lap = np.zeros_like(v)
    lap[has] = v[has] - nbr[has] / deg[has, None]
    scaled = np.where(has[:, None], lap / np.maximum(deg, 1.0)[:, None], 0.0)
    back = np.zeros_like(v)
    np.add.at(back, both[:, 1], scaled[both[:, 0]])
    return float(np.mean(np.sum(lap * lap, axis=1))), (2.0 / nv) * lap - (2.0 / nv) * back


class VectorAdam:
    """optim.py:29-81: Adam with one second moment per vertex row; a step
    with a non-finite gradient is rejected."""

    def __init__(self, n, beta1=0.9, beta2=0.999, eps=1e-8):
        self.b1, self.b2, self.eps = beta1, beta2, eps
        self.m, self.v, self.t = np.zeros((n, 3)), np.zeros(n), 0

    def step(self, p, g, lr):
        if not np.all(np.isfinite(g)):
            return p
        self.t += 1
        self.m = self.b1 * self.m + (1 - self.b1) * g
        self.v = self.b2 * self.v + (1 - self.b2) * np.sum(g * g, axis=1)
        mh = self.m / (1 - self.b1 ** self.t)
        vh = self.v / (1 - self.b2 ** self.t)
        return p - lr * mh / (np.sqrt(vh)[:, None] + self.eps)


class ScalarAdam:
    """optim.py:84-126: per-component Adam."""

    def __init__(self, shape, beta1=0.9, beta2=0.999, eps=1e-8):
        self.b1, self.b2, self.eps = beta1, beta2, eps
        self.m, self.v, self.t = np.zeros(shape), np.zeros(shape), 0

    def step(self, p, g, lr):
        if not np.all(np.isfinite(g)):
            return p
        self.t += 1
        self.m = self.b1 * self.m + (1 - self.b1) * g
        self.v = self.b2 * self.v + (1 - self.b2) * g * g
        mh = self.m / (1 - self.b1 ** self.t)
        vh = self.v / (1 - self.b2 ** self.t)
        return p - lr * mh / (np.sqrt(vh) + self.eps)


def cosine_lr(it, total, base, floor_fraction=0.1):
    """optim.py:129-135."""
    if total <= 1:
        return base
    frac = min(max(it / (total - 1), 0.0), 1.0)
    lo = floor_fraction * base
    return lo + (base - lo) * 0.5 * (1.0 + np.cos(np.pi * frac))
