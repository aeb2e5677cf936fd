"""Drop-in numpy API of the GMR hot path, backed by libgmr.so on the GPU.

Same names, signatures, dtypes and error behaviour as the reference
(`meshsplat`): render.py:441-467 (`render_mesh`, `render_backward`),
render.py:272-361 (`rasterize`, `rasterize_backward`), convert.py:313-437
(`convert_mesh`, `convert_backward`) and losses.py:43-174 (`total_loss`
and its terms).  Inputs are copied to the current CUDA device, all compute
runs in the CUDA library, results come back as numpy arrays.  There is no
CPU fallback: without a CUDA device every call raises.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import engine
from .camera import Camera

TILE = 16
ALPHA_CLAMP = 0.99
CONTRIB_FLOOR = 1.0 / 255.0
TRANSMITTANCE_STOP = 1e-4
DILATION = 0.3
BCE_CLAMP = 1e-6

_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def _torch_dtype(dtype):
    dt = np.dtype(dtype)
    if dt not in _TORCH:
        raise ValueError(f"dtype must be float32 or float64, got {dt}")
    return _TORCH[dt]


def _device():
    engine.L.load()
    return torch.device("cuda", torch.cuda.current_device())


_mesh_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_topo_cache: dict = {}   # id(facets array) -> (weakref to it, int32 faces on device, edges, CSR)


def _facets_entry(facets):
    """Per-topology device/host data, keyed by the facets array object (a
    TriangleMesh rebuilt with new vertices, as in the fit loop, shares it)."""
    key = id(facets)
    hit = _topo_cache.get(key)
    if hit is not None and hit[0]() is facets:
        return hit[1]
    dev = _device()
    entry = {"faces": torch.as_tensor(np.array(facets, dtype=np.int32)).to(dev)}
    try:
        ref = weakref.ref(facets)
    except TypeError:
        return entry
    if len(_topo_cache) > 64:
        _topo_cache.clear()
    _topo_cache[key] = (ref, entry)
    return entry


def _device_mesh(mesh, dtype):
    """(pos, col, faces int32) on the device for an immutable mesh object."""
    tdt = _torch_dtype(dtype)
    dev = _device()
    try:
        per = _mesh_cache.setdefault(mesh, {})
    except TypeError:
        per = {}
    hit = per.get(tdt)
    if hit is None:
        pos = torch.as_tensor(np.array(mesh.vertices, dtype=np.float64), dtype=tdt).to(dev)
        col = torch.as_tensor(np.array(mesh.colors, dtype=np.float64), dtype=tdt).to(dev)
        faces = _facets_entry(mesh.facets)["faces"]
        hit = per[tdt] = (pos, col, faces)
    return hit


@dataclass(frozen=True)
class RenderOutput:
    rgb: np.ndarray
    alpha: np.ndarray
    background: np.ndarray


@dataclass
class RenderContext:
    """Everything render_backward needs (reference render.py:429-438); the
    device part (sorted tile entries, tile ranges, T_final) lives in
    `state.ws` so the backward never re-bins."""
    mesh: object
    camera: Camera
    output: RenderOutput
    dtype: type
    rescale: bool
    state: engine.ForwardState
    rgb_device: torch.Tensor


def render_mesh(mesh, camera, background=(0.0, 0.0, 0.0), rescale: bool = True,
                dtype=np.float64, return_ctx: bool = False):
    """convert -> project -> rasterize on the GPU (reference render.py:441-450)."""
    pos, col, faces = _device_mesh(mesh, dtype)
    bg = np.asarray(background, dtype=dtype)
    rgb, alpha, state = engine.render_forward(
        pos, col, faces, [camera], camera.width, camera.height, bg, rescale,
        item_to_index="kept")
    out = RenderOutput(rgb=rgb[0].cpu().numpy(), alpha=alpha[0].cpu().numpy(), background=bg)
    if not return_ctx:
        return out
    return out, RenderContext(mesh=mesh, camera=camera, output=out, dtype=dtype, rescale=rescale,
                              state=state, rgb_device=rgb)


def render_backward(ctx: RenderContext, grad_rgb, grad_alpha):
    """Pixel gradients -> (grad_vertices (V,3), grad_vertex_colors (V,3)),
    float64 like the reference (render.py:453-467)."""
    cam = ctx.camera
    grad_rgb = np.asarray(grad_rgb)
    grad_alpha = np.asarray(grad_alpha)
    if grad_rgb.shape != (cam.height, cam.width, 3) or grad_alpha.shape != (cam.height, cam.width):
        raise ValueError("upstream gradient shapes do not match the image")
    pos, col, faces = _device_mesh(ctx.mesh, ctx.dtype)
    tdt = _torch_dtype(ctx.dtype)
    dev = pos.device
    g_rgb = torch.as_tensor(np.ascontiguousarray(grad_rgb), dtype=tdt).to(dev)[None]
    g_a = torch.as_tensor(np.ascontiguousarray(grad_alpha), dtype=tdt).to(dev)[None]
    gp, gc = engine.render_backward(ctx.state, pos, col, faces, ctx.rgb_device, g_rgb, g_a)
    return gp.cpu().numpy().astype(np.float64), gc.cpu().numpy().astype(np.float64)


# ---------------------------------------------------------------------------
# splat path: rasterize / rasterize_backward (render.py:168-188, 272-361)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Splat2D:
    mean2d: np.ndarray
    cov2d_screen: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    source: int = -1


def _splat_arrays(splats, dtype):
    if hasattr(splats, "mean2d") and not isinstance(splats, (list, tuple)):
        k = len(splats.depth)
        src = np.asarray(getattr(splats, "source", np.arange(k)), dtype=np.int64)
        return (np.asarray(splats.mean2d, dtype).reshape(k, 2), np.asarray(splats.cov2d, dtype).reshape(k, 2, 2),
                np.asarray(splats.depth, dtype).reshape(k), np.asarray(splats.color, dtype).reshape(k, 3),
                np.asarray(splats.opacity, dtype).reshape(k), src)
    k = len(splats)
    if k == 0:
        z = lambda *s: np.zeros(s, dtype=dtype)
        return z(0, 2), z(0, 2, 2), z(0), z(0, 3), z(0), np.zeros(0, np.int64)
    return (np.stack([np.asarray(s.mean2d, dtype=dtype) for s in splats]),
            np.stack([np.asarray(s.cov2d_screen, dtype=dtype) for s in splats]),
            np.array([s.depth for s in splats], dtype=dtype),
            np.stack([np.asarray(s.color, dtype=dtype) for s in splats]),
            np.array([s.opacity for s in splats], dtype=dtype),
            np.array([s.source if s.source >= 0 else i for i, s in enumerate(splats)], dtype=np.int64))


def _check_finite_host(arrays):
    """render.py:191-197 for the caller's inputs (conic is checked on the device)."""
    names = ("mean2d", "cov2d", None, "depth", "color", "opacity")
    vals = dict(zip(("mean2d", "cov2d", "depth", "color", "opacity"), arrays[:5]))
    for name in names:
        if name is None:
            continue
        bad = ~np.isfinite(vals[name])
        if bad.any():
            raise ValueError(f"non-finite splat parameter {name!r} at splat {int(np.argwhere(bad)[0][0])}")


def _raster_device(splats, camera, background, dtype):
    arrs = _splat_arrays(splats, dtype)
    _check_finite_host(arrs)
    order = np.argsort(arrs[5], kind="stable")   # tie-break by source (render.py:227)
    tdt = _torch_dtype(dtype)
    dev = _device()
    t = [torch.as_tensor(np.ascontiguousarray(a[order]), dtype=tdt).to(dev) for a in arrs[:5]]
    rgb, alpha, state = engine.rasterize_forward(*t, camera.width, camera.height,
                                                 np.asarray(background, dtype=np.float64))
    return t, order, rgb, alpha, state


def rasterize(splats, camera, background=(0.0, 0.0, 0.0), dtype=np.float64) -> RenderOutput:
    """Front-to-back compositing of splats on the GPU (render.py:272-291)."""
    _, _, rgb, alpha, _ = _raster_device(splats, camera, background, dtype)
    return RenderOutput(rgb=rgb.cpu().numpy(), alpha=alpha.cpu().numpy(),
                        background=np.asarray(background, dtype=dtype))


def rasterize_backward(splats, camera, output, grad_rgb, grad_alpha, dtype=np.float64):
    """(g_mean2d, g_cov2d, g_color, g_opacity) in the caller's splat order
    (render.py:294-361)."""
    w, h = camera.width, camera.height
    grad_rgb = np.asarray(grad_rgb, dtype=dtype)
    grad_alpha = np.asarray(grad_alpha, dtype=dtype)
    if grad_rgb.shape != (h, w, 3) or grad_alpha.shape != (h, w):
        raise ValueError("upstream gradient shapes do not match the image")
    bg = np.asarray(output.background, dtype=np.float64)
    t, order, rgb, _, state = _raster_device(splats, camera, bg, dtype)
    tdt = _torch_dtype(dtype)
    g = [torch.as_tensor(np.ascontiguousarray(x), dtype=tdt).to(rgb.device) for x in (grad_rgb, grad_alpha)]
    gm, gc, gcol, gop = engine.rasterize_backward(state, *t, rgb, g[0], g[1])
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    return tuple(x.cpu().numpy()[inv] for x in (gm, gc, gcol, gop))


# ---------------------------------------------------------------------------
# conversion stage (convert.py:313-437, embed route)
# ---------------------------------------------------------------------------

@dataclass
class GaussianCloud:
    means: np.ndarray
    cov3d: np.ndarray
    colors: np.ndarray
    opacities: np.ndarray
    degenerate: np.ndarray
    path: str = "embed"
    rescale: bool = True

    def __len__(self):
        return len(self.means)


def convert_mesh(mesh, path: str = "embed", rescale: bool = True) -> GaussianCloud:
    """Facet -> Gaussian, embed route, float64 (convert.py:313-343)."""
    if path not in ("embed", "eigen"):
        raise ValueError(f"unknown conversion path {path!r}")
    if path == "eigen":
        raise ValueError("the eigen route is a CPU validation path; only 'embed' runs on the device")
    pos, col, faces = _device_mesh(mesh, np.float64)
    means, cov, colors, degen = engine.convert(pos, col, faces, rescale)
    m = len(mesh.facets)
    return GaussianCloud(means=means.cpu().numpy(), cov3d=cov.cpu().numpy(), colors=colors.cpu().numpy(),
                         opacities=np.ones(m), degenerate=degen.cpu().numpy(), path="embed", rescale=rescale)


@dataclass
class SplatBatch:
    """Kept splats of one camera, in cloud order (render.py:52-73)."""
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


def project_cloud(cloud, camera: Camera, dtype=np.float64) -> SplatBatch:
    """EWA projection with depth-window and 3-sigma screen culling
    (render.py:103-145), on the device (gmr_project)."""
    import ctypes
    lib = engine.L.load()
    tdt = _torch_dtype(dtype)
    dev = _device()
    k = len(cloud.means)
    means = torch.as_tensor(np.ascontiguousarray(np.asarray(cloud.means, np.float64).reshape(k, 3)), dtype=tdt).to(dev)
    cov = torch.as_tensor(np.ascontiguousarray(np.asarray(cloud.cov3d, np.float64).reshape(k, 3, 3)), dtype=tdt).to(dev)
    out = {n: torch.zeros(shape, dtype=tdt, device=dev) for n, shape in
           (("mean2d", (k, 2)), ("cov2d", (k, 2, 2)), ("conic", (k, 3)), ("depth", (k,)), ("radius", (k,)),
            ("t_cam", (k, 3)))}
    kept = torch.zeros(k, dtype=torch.uint8, device=dev)
    cam = engine.L.camera_struct([camera])
    engine.L.check(lib.gmr_project(engine._ptr(means), engine._ptr(cov), k, cam, camera.width, camera.height,
                                   engine._DT[tdt], *(engine._ptr(out[n]) for n in
                                                      ("mean2d", "cov2d", "conic", "depth", "radius", "t_cam")),
                                   engine._ptr(kept), engine._stream()))
    idx = np.where(kept.cpu().numpy() > 0)[0]
    host = {n: v.cpu().numpy()[idx] for n, v in out.items()}
    np_dt = np.dtype(dtype)
    return SplatBatch(color=np.asarray(cloud.colors)[idx].astype(np_dt),
                      opacity=np.asarray(cloud.opacities)[idx].astype(np_dt), source=idx.astype(np.int64), **host)


def project_cloud_backward(batch: SplatBatch, cloud, camera: Camera, g_mean2d, g_cov2d):
    """Screen-space gradients of the kept splats -> (g_mean3d, g_cov3d)
    aligned with the batch (render.py:364-402), on the device
    (gmr_project_backward)."""
    lib = engine.L.load()
    np_dt = np.asarray(batch.mean2d).dtype
    tdt = _torch_dtype(np_dt)
    dev = _device()
    k = len(batch)
    t = lambda x, shape: torch.as_tensor(np.ascontiguousarray(np.asarray(x, np.float64).reshape(shape)),
                                         dtype=tdt).to(dev)
    tc = t(batch.t_cam, (k, 3))
    cov = t(np.asarray(cloud.cov3d)[np.asarray(batch.source, np.int64)], (k, 3, 3))
    gm, gc = t(g_mean2d, (k, 2)), t(g_cov2d, (k, 2, 2))
    g3 = torch.zeros((k, 3), dtype=tdt, device=dev)
    gcov = torch.zeros((k, 3, 3), dtype=tdt, device=dev)
    engine.L.check(lib.gmr_project_backward(engine._ptr(tc), engine._ptr(cov), k, engine.L.camera_struct([camera]),
                                            engine._DT[tdt], engine._ptr(gm), engine._ptr(gc), engine._ptr(g3),
                                            engine._ptr(gcov), engine._stream()))
    return g3.cpu().numpy(), gcov.cpu().numpy()


EXPORT_PROPS = ("x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
                "rot_0", "rot_1", "rot_2", "rot_3")


def export_gaussians(cloud, path) -> None:
    """Splat-viewer PLY (binary little-endian, 14 float32 per Gaussian)
    (convert.py:484-532).  The per-Gaussian eigendecomposition, quaternion,
    logit and SH-DC terms run on the device (gmr_export_gaussians); the host
    writes the header and the record bytes."""
    import ctypes

    from . import lib as L
    n = len(cloud.means)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda x, shape: torch.tensor(np.ascontiguousarray(np.asarray(x, np.float64).reshape(shape)), device=dev)
    means, cov = t(cloud.means, (n, 3)), t(cloud.cov3d, (n, 3, 3))
    cols, ops = t(cloud.colors, (n, 3)), t(cloud.opacities, (n,))
    rec = torch.empty((n, len(EXPORT_PROPS)), dtype=torch.float32, device=dev)
    L.check(L.load().gmr_export_gaussians(means.data_ptr(), cov.data_ptr(), cols.data_ptr(), ops.data_ptr(), n,
                                          rec.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    head = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    head += [f"property float {p}" for p in EXPORT_PROPS] + ["end_header"]
    body = rec.cpu().numpy().astype("<f4").tobytes()
    with open(path, "wb") as fh:
        fh.write(("\n".join(head) + "\n").encode("ascii"))
        fh.write(body)


def convert_backward(mesh, cloud, grad_means, grad_cov3ds, grad_colors):
    """Facet grads -> vertex grads in np.add.at order (convert.py:371-437)."""
    if getattr(cloud, "path", "embed") != "embed":
        raise ValueError("convert_backward differentiates the embed path only")
    m = len(mesh.facets)
    gm = np.asarray(grad_means, dtype=np.float64)
    gc = np.asarray(grad_cov3ds, dtype=np.float64)
    gcol = np.asarray(grad_colors, dtype=np.float64)
    if gm.shape != (m, 3) or gc.shape != (m, 3, 3) or gcol.shape != (m, 3):
        raise ValueError(f"gradient shapes {gm.shape}, {gc.shape}, {gcol.shape} do not match {m} facets")
    pos, col, faces = _device_mesh(mesh, np.float64)
    dev = pos.device
    gp, gcv = engine.convert_backward(pos, col, faces, torch.as_tensor(gm).to(dev), torch.as_tensor(gc).to(dev),
                                      torch.as_tensor(gcol).to(dev), getattr(cloud, "rescale", True))
    return gp.cpu().numpy(), gcv.cpu().numpy()


# ---------------------------------------------------------------------------
# objective (losses.py:23-174): B views per device call
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LossWeights:
    color: float = 1.0
    silhouette: float = 1.0
    edge: float = 0.1
    laplacian: float = 0.1


@dataclass(frozen=True)
class LossReport:
    color: float
    silhouette: float
    edge: float
    laplacian: float
    total: float
    n_views: int


def _scratch(n_bytes, dev):
    return torch.empty(max(int(n_bytes), 1), dtype=torch.uint8, device=dev)


def _image_loss(kind, x, t):
    import ctypes
    lib = engine.L.load()
    dev = _device()
    xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    td = torch.as_tensor(np.ascontiguousarray(t, dtype=np.float64)).to(dev)
    n = xd.numel()
    grad = torch.empty_like(xd)
    val = torch.empty(1, dtype=torch.float64, device=dev)
    if n == 0:
        return float("nan"), np.zeros(xd.shape)
    nb = ctypes.c_size_t()
    engine.L.check(lib.gmr_image_loss_scratch_size(n, ctypes.byref(nb)))
    scr = _scratch(nb.value, dev)
    engine.L.check(lib.gmr_image_loss(kind, engine._ptr(xd), engine._ptr(td), n, engine._ptr(grad),
                                      engine._ptr(val), engine._ptr(scr), nb.value, engine._stream()))
    return float(val.item()), grad.cpu().numpy()


def color_loss(rendered, target):
    """Mean squared colour error and its gradient (losses.py:43-56), float64,
    computed on the device (gmr_image_loss kind 0)."""
    rendered, target = np.asarray(rendered), np.asarray(target)
    if rendered.shape != target.shape:
        raise ValueError(f"shape mismatch: {rendered.shape} vs {target.shape}")
    return _image_loss(0, rendered, target)


def silhouette_loss(alpha, mask):
    """Clamped binary cross-entropy of alpha against the mask and its
    gradient (losses.py:59-73), float64, on the device (gmr_image_loss kind 1)."""
    alpha, mask = np.asarray(alpha), np.asarray(mask)
    if alpha.shape != mask.shape:
        raise ValueError(f"shape mismatch: {alpha.shape} vs {mask.shape}")
    return _image_loss(1, alpha, mask)


def _graph(facets, num_vertices):
    """Static mesh graph on the device (edges, np.add.at-order CSRs), cached
    with the facets' other per-topology data."""
    from . import lib as L
    from .mesh import mesh_graph
    ent = _facets_entry(facets)
    hit = ent.get("graph")
    if hit is None or hit[0] != num_vertices:
        dev = _device()
        g = {k: torch.as_tensor(v).to(dev) for k, v in mesh_graph(facets, num_vertices).items()}
        st = L.GmrMeshGraph(g["edges"].data_ptr(), int(g["edges"].shape[0]), g["ve_ptr"].data_ptr(),
                            g["ve_slot"].data_ptr(), g["adj_ptr"].data_ptr(), g["adj"].data_ptr())
        hit = ent["graph"] = (num_vertices, st, g)
    return hit[1]


def _regularizers(facets, vertices, want_edge=True, want_lap=True):
    """(values [2] (edge, laplacian), grad_edge, grad_laplacian) on the
    device for float64 vertices (gmr_mesh_regularizers)."""
    import ctypes
    lib = engine.L.load()
    dev = _device()
    v = torch.as_tensor(np.ascontiguousarray(vertices, dtype=np.float64)).to(dev) \
        if not isinstance(vertices, torch.Tensor) else vertices.to(dev, torch.float64).contiguous()
    nv = int(v.shape[0])
    graph = _graph(facets, nv)
    nb = ctypes.c_size_t()
    engine.L.check(lib.gmr_fit_scratch_size(nv, graph.num_edges, ctypes.byref(nb)))
    scr = _scratch(nb.value, dev)
    vals = torch.empty(2, dtype=torch.float64, device=dev)
    ge = torch.empty_like(v) if want_edge else None
    gl = torch.empty_like(v) if want_lap else None
    engine.L.check(lib.gmr_mesh_regularizers(engine._ptr(v), ctypes.byref(graph), nv, engine._ptr(vals),
                                             engine._ptr(ge), engine._ptr(gl), engine._ptr(scr), nb.value,
                                             engine._stream()))
    return vals, ge, gl


def edge_length_loss(mesh, vertices=None):
    """Edge-length variance regulariser and its gradient (losses.py:76-97),
    on the device (gmr_mesh_regularizers)."""
    verts = np.asarray(mesh.vertices if vertices is None else vertices, dtype=np.float64)
    if len(mesh.facets) == 0 or len(verts) == 0:
        return 0.0, np.zeros_like(verts)
    vals, ge, _ = _regularizers(mesh.facets, verts, want_lap=False)
    return float(vals[0].item()), ge.cpu().numpy()


def laplacian_loss(mesh, vertices=None):
    """Uniform-Laplacian regulariser and its gradient (losses.py:100-123), on
    the device (gmr_mesh_regularizers)."""
    verts = np.asarray(mesh.vertices if vertices is None else vertices, dtype=np.float64)
    if len(verts) == 0:
        return 0.0, np.zeros_like(verts)
    vals, _, gl = _regularizers(mesh.facets, verts, want_edge=False)
    return float(vals[1].item()), gl.cpu().numpy()


def total_loss(mesh, cameras: Sequence[Camera], target_rgb, target_mask, weights: LossWeights = LossWeights(),
               background=(0.0, 0.0, 0.0), rescale: bool = True, dtype=np.float64):
    """Weighted objective over a batch of views (losses.py:126-174).  All
    views of one resolution are rendered and differentiated in ONE device
    call; per-view image grads are scaled by w/n exactly as the reference."""
    if not (len(cameras) == len(target_rgb) == len(target_mask)):
        raise ValueError("cameras and targets must have matching lengths")
    if len(cameras) == 0:
        raise ValueError("need at least one view")
    n = len(cameras)
    pos, col, faces = _device_mesh(mesh, dtype)
    dev = pos.device
    tdt = _torch_dtype(dtype)
    groups = {}
    for i, c in enumerate(cameras):
        groups.setdefault((c.width, c.height), []).append(i)
    gp_acc = torch.zeros((len(mesh.vertices), 3), dtype=torch.float64, device=dev)
    gc_acc = torch.zeros_like(gp_acc)
    cv_acc = torch.zeros((), dtype=torch.float64, device=dev)
    sv_acc = torch.zeros((), dtype=torch.float64, device=dev)
    bg = np.asarray(background, dtype=np.float64)
    for (w, h), idx in groups.items():
        cams = [cameras[i] for i in idx]
        t_rgb = torch.as_tensor(np.stack([np.asarray(target_rgb[i], np.float64) for i in idx]),
                                dtype=tdt).to(dev)
        t_m = torch.as_tensor(np.stack([np.asarray(target_mask[i], np.float64) for i in idx]), dtype=tdt).to(dev)
        if t_rgb.shape != (len(idx), h, w, 3) or t_m.shape != (len(idx), h, w):
            raise ValueError("shape mismatch between renders and targets")
        # losses fused into the blend epilogue (gmr_render_forward_loss)
        rgb, alpha, g_rgb, g_a, sums, state = engine.render_forward_loss(
            pos, col, faces, cams, w, h, bg, t_rgb, t_m, weights.color / n, weights.silhouette / n, rescale)
        cv_acc += sums[0] / (3.0 * w * h)
        sv_acc += sums[1] / (1.0 * w * h)
        gp, gc = engine.render_backward(state, pos, col, faces, rgb, g_rgb, g_a)
        gp_acc += gp.double()
        gc_acc += gc.double()
    # the mesh regularisers on the device too (float64 like the reference)
    nv = len(mesh.vertices)
    if len(mesh.facets) and nv:
        regs, g_edge, g_lap = _regularizers(mesh.facets, mesh.vertices)
        gp_acc += weights.edge * g_edge + weights.laplacian * g_lap
    else:
        regs = torch.zeros(2, dtype=torch.float64, device=dev)
    # one transfer for everything
    flat = torch.cat([cv_acc.view(1), sv_acc.view(1), regs, gp_acc.view(-1), gc_acc.view(-1)]).cpu().numpy()
    cval_sum, sval_sum, edge_val, lap_val = flat[0], flat[1], float(flat[2]), float(flat[3])
    grad_v = flat[4:4 + 3 * nv].reshape(nv, 3).copy()
    grad_c = flat[4 + 3 * nv:].reshape(nv, 3).copy()
    color_val = float(cval_sum / n)
    sil_val = float(sval_sum / n)
    total = (weights.color * color_val + weights.silhouette * sil_val
             + weights.edge * edge_val + weights.laplacian * lap_val)
    return LossReport(color=color_val, silhouette=sil_val, edge=edge_val, laplacian=lap_val,
                      total=total, n_views=n), grad_v, grad_c
