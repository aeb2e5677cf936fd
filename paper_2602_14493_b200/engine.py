"""Device-side driver of libgmr: workspace planning, capacity management,
topology caching, and the torch autograd Function over B views.

PyTorch provides device memory and the current stream only; every FLOP of
the render path runs in libgmr.so (include/gmr.h).  Callers: the numpy
drop-in shim (`api.py`, mirroring reference render.py / convert.py /
losses.py) and the batched torch entry `render_views`.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import lib as L

_DT = {torch.float32: L.GMR_F32, torch.float64: L.GMR_F64}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream():
    """The current CUDA stream of the current device as a void* (the cheap
    raw query: torch.cuda.current_stream() costs ~15 us per call)."""
    if _raw_stream is not None:
        return ctypes.c_void_p(_raw_stream(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


# Extra GmrRaster flags for every call of this process.  Set to
# L.FLAG_FULL_TILE_LISTS to get the reference's exact _RasterPlan tile lists
# (by default splats drop the tiles they cannot reach; outputs are identical).
DEFAULT_FLAGS = 0


def raster_struct(width, height, background, dtype, rescale=True, flags=0) -> L.GmrRaster:
    r = L.GmrRaster()
    r.width, r.height = int(width), int(height)
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    r.background[:] = [float(x) for x in bg]
    r.dtype = _DT[dtype]
    r.rescale = 1 if rescale else 0
    r.flags = int(flags) | DEFAULT_FLAGS
    return r


def mesh_struct(pos, col, faces) -> L.GmrMesh:
    m = L.GmrMesh()
    m.positions, m.colors, m.faces = pos.data_ptr(), col.data_ptr(), faces.data_ptr()
    m.num_vertices, m.num_faces = int(pos.shape[0]), int(faces.shape[0])
    return m


class _Capacity:
    """Entry-capacity estimate per (F, B, W, H): starts at 4 entries per
    item and grows (x1.25 headroom) when a forward reports overflow."""

    def __init__(self):
        self._cap = {}

    def get(self, key, items):
        return self._cap.get(key, 4 * items + 4096)

    def grow(self, key, needed):
        self._cap[key] = int(needed * 1.25) + 4096
        return self._cap[key]

    def note(self, key, cap, used):
        # keep ~25% headroom over what the last call needed
        want = int(used * 1.25) + 4096
        self._cap[key] = want if (cap > 2 * want or cap < want) else cap


_capacity = _Capacity()


class _TileOrder:
    """Chooses GMR_FLAG_TILE_DEPTH_SORT per call shape from the longest tile
    list of an earlier forward of that shape (device status byte 60, copied
    behind the call without a sync; re-read every REFRESH calls).  Per-tile
    depth ordering when every list fits the kernel's shared-memory sort; the
    global depth sort otherwise, and for the first call of a shape.  Both give
    the same lists.  Large batches (>= GLOBAL_ITEMS splats per call) keep the
    global sort: its three range-reduced radix passes over all splats beat
    the per-list sorts there (config 3, 8 views: binning 0.374 vs 0.404 ms;
    config 2 / config 3 batch 1: 0.135 vs 0.137 / 0.117 vs 0.162 ms the other
    way)."""

    LIMIT = {torch.float32: 2048, torch.float64: 1024}
    GLOBAL_ITEMS = 2_000_000
    REFRESH = 64

    class _Shape:
        __slots__ = ("last", "host", "event", "pending", "calls")

        def __init__(self):
            self.last, self.host, self.event, self.pending, self.calls = None, None, None, False, 0

    def __init__(self):
        self._shapes = {}

    def flags(self, key, dtype):
        if not AUTO_TILE_ORDER:
            return 0
        items = key[0] * key[1] if isinstance(key[0], int) else key[1]   # (F, B, ...) or ('splats', K, ...)
        if items >= self.GLOBAL_ITEMS:
            return 0
        sh = self._shapes.get(key)
        if sh is None:
            return 0
        # (no event queries while a graph is being captured)
        if sh.pending and not torch.cuda.is_current_stream_capturing() and sh.event.query():
            sh.last = int(sh.host.view(torch.int32)[0])
            sh.pending = False
        return L.FLAG_TILE_DEPTH_SORT if sh.last is not None and sh.last <= self.LIMIT[dtype] else 0

    def note(self, key, ws):
        if not AUTO_TILE_ORDER or torch.cuda.is_current_stream_capturing():
            return
        sh = self._shapes.get(key)
        if sh is None:
            sh = self._shapes[key] = self._Shape()
            sh.host = torch.empty(4, dtype=torch.uint8, pin_memory=True)
            sh.event = torch.cuda.Event()
        sh.calls += 1
        if sh.pending or (sh.last is not None and sh.calls % self.REFRESH):
            return
        sh.host.copy_(ws[60:64], non_blocking=True)
        sh.event.record()
        sh.pending = True

    def forget(self):
        self._shapes.clear()


_order = _TileOrder()
# False: never add GMR_FLAG_TILE_DEPTH_SORT on our own (tests pin the mode
# through DEFAULT_FLAGS; GMR_TILE_ORDER=global does the same for a process)
AUTO_TILE_ORDER = os.environ.get("GMR_TILE_ORDER", "auto") != "global"
_topologies = {}


def topology(faces: torch.Tensor, num_vertices: int) -> torch.Tensor:
    """Face->vertex CSR (convert.py:427-436 order), cached per faces tensor."""
    key = (faces.data_ptr(), int(faces.shape[0]), int(num_vertices), faces._version)
    topo = _topologies.get(key)
    if topo is None:
        lib = L.load()
        nb = ctypes.c_size_t()
        L.check(lib.gmr_topology_size(faces.shape[0], num_vertices, ctypes.byref(nb)))
        topo = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=faces.device)
        L.check(lib.gmr_topology_build(_ptr(faces), faces.shape[0], num_vertices, _ptr(topo),
                                       nb.value, _stream()))
        if len(_topologies) > 16:
            _topologies.clear()
        _topologies[key] = (topo, faces)  # keep faces alive so the key stays valid
        return topo
    return topo[0]


_FIELDS = ("mean2d", "cov2d", "conic", "depth", "color", "opacity")


@dataclass
class ForwardState:
    """What a forward leaves for its backward (RenderContext device part)."""
    ws: torch.Tensor
    capacity: int
    raster: L.GmrRaster
    cams: ctypes.Array
    views: int
    entries: int
    kept: int


def _status_or_raise(ws, kind, item_to_index=None):
    lib = L.load()
    st = L.GmrStatus()
    code = lib.gmr_status(_ptr(ws), ctypes.byref(st), _stream())
    if code == L.GMR_ENONFINITE:
        idx = st.nonfinite_item if item_to_index is None else item_to_index(st.nonfinite_item)
        raise ValueError(f"non-finite splat parameter {_FIELDS[st.nonfinite_field]!r} at splat {idx}")
    if code not in (L.GMR_OK, L.GMR_ECAPACITY):
        L.check(code)
    return st, code


def render_forward(pos, col, faces, cams, width, height, background, rescale=True, flags=0,
                   item_to_index=None, check=True):
    """B-view forward.  pos/col [V,3] (f32|f64, cuda), faces [F,3] int32.
    Returns (rgb [B,H,W,3], alpha [B,H,W], ForwardState).

    check=False enqueues without waiting for the status (no host sync); the
    caller must then call `check_status(state)` before using any result --
    a capacity overflow or a non-finite splat is reported there."""
    lib = L.load()
    dtype = pos.dtype
    B, F = len(cams), int(faces.shape[0])
    raster = raster_struct(width, height, background, dtype, rescale, flags)
    cam_arr = L.camera_struct(cams)
    mesh = mesh_struct(pos, col, faces)
    key = (F, B, int(width), int(height), dtype)
    raster.flags |= _order.flags(key, dtype)
    cap = _capacity.get(key, F * B)
    rgb = torch.empty((B, height, width, 3), dtype=dtype, device=pos.device)
    alpha = torch.empty((B, height, width), dtype=dtype, device=pos.device)
    if not check:
        nb = ctypes.c_size_t()
        L.check(lib.gmr_render_workspace_size(F, B, width, height, cap, raster.dtype, ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=pos.device)
        L.check(lib.gmr_render_forward(ctypes.byref(mesh), cam_arr, B, ctypes.byref(raster), _ptr(rgb),
                                       _ptr(alpha), _ptr(ws), nb.value, cap, _stream()))
        _order.note(key, ws)
        st = ForwardState(ws, cap, raster, cam_arr, B, -1, -1)
        # the 64-byte device status, copied behind the forward (no sync)
        st.status_host = torch.empty(64, dtype=torch.uint8, pin_memory=True)
        st.status_host.copy_(ws[:64], non_blocking=True)
        st.status_event = torch.cuda.Event()
        st.status_event.record()
        st.key = key
        return rgb, alpha, st
    for _ in range(3):
        nb = ctypes.c_size_t()
        L.check(lib.gmr_render_workspace_size(F, B, width, height, cap, raster.dtype, ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=pos.device)
        # the status arrives as soon as binning has counted the entries: the
        # call is validated while the forward still sorts and blends, so the
        # caller's next launches queue behind it without draining the stream
        status = torch.empty(64, dtype=torch.uint8, pin_memory=True)
        ev = torch.cuda.Event()
        ev.record()   # torch creates the CUDA event lazily, on its first record
        assert ev.cuda_event, "CUDA event not created"
        L.check(lib.gmr_render_forward_ex(ctypes.byref(mesh), cam_arr, B, ctypes.byref(raster), _ptr(rgb),
                                          _ptr(alpha), _ptr(ws), nb.value, cap, ctypes.c_void_p(status.data_ptr()),
                                          ctypes.c_void_p(ev.cuda_event), _stream()))
        _order.note(key, ws)
        ev.synchronize()
        entries, kept, bad, overflow = _parse_status(status.numpy())
        for field in range(6):
            if bad[field] != 0xFFFFFFFF:
                item = int(bad[field])
                if item_to_index == "kept":
                    # the reference reports the index into the view's culled
                    # splat batch (render.py:191-197): rank among kept faces
                    fs = ForwardState(ws, cap, raster, cam_arr, B, -1, -1)
                    cnt = copy_splats(fs, F, True)[2].cpu().numpy()
                    v0 = (item // max(F, 1)) * F
                    idx = int(np.count_nonzero(cnt[v0:item] > 0))
                else:
                    idx = item if item_to_index is None else item_to_index(item)
                raise ValueError(f"non-finite splat parameter {_FIELDS[field]!r} at splat {idx}")
        if not overflow:
            _capacity.note(key, cap, entries)
            return rgb, alpha, ForwardState(ws, cap, raster, cam_arr, B, entries, kept)
        cap = _capacity.grow(key, entries)
    raise RuntimeError("tile-entry capacity did not converge")


def _parse_status(raw):
    """(entries, kept, first non-finite item per field, overflow) of the
    64-byte device status (DevStatus in csrc/gmr_common.cuh)."""
    entries, kept = (int(x) for x in raw[:16].view(np.uint64))
    words = raw[16:48].view(np.uint32)
    return entries, kept, words[:6], int(words[6])


def render_forward_loss(pos, col, faces, cams, width, height, background, target_rgb, target_mask,
                        scale_rgb, scale_alpha, rescale=True, check=True):
    """B-view forward with the colour/silhouette losses fused into the blend
    epilogue.  target_rgb [B,H,W,3] / target_mask [B,H,W] on the device in the
    render dtype.  Returns (rgb, alpha, g_rgb, g_alpha, loss_sums [2] f64 on
    the device: sum of squared colour errors, sum of BCE terms), state).
    check: True = validate now (host sync), False = copy the status behind the
    call (`check_status` later), None = leave it in the workspace."""
    lib = L.load()
    dtype = pos.dtype
    B, F = len(cams), int(faces.shape[0])
    raster = raster_struct(width, height, background, dtype, rescale, 0)
    cam_arr = L.camera_struct(cams)
    mesh = mesh_struct(pos, col, faces)
    key = (F, B, int(width), int(height), dtype)
    raster.flags |= _order.flags(key, dtype)
    dev = pos.device
    rgb = torch.empty((B, height, width, 3), dtype=dtype, device=dev)
    alpha = torch.empty((B, height, width), dtype=dtype, device=dev)
    g_rgb = torch.empty_like(rgb)
    g_a = torch.empty_like(alpha)
    sums = torch.empty(2, dtype=torch.float64, device=dev)
    t_rgb = target_rgb.to(dtype).contiguous()
    t_m = target_mask.to(dtype).contiguous()
    cap = _capacity.get(key, F * B)
    for _ in range(3):
        nb = ctypes.c_size_t()
        L.check(lib.gmr_render_workspace_size(F, B, width, height, cap, raster.dtype, ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
        L.check(lib.gmr_render_forward_loss(ctypes.byref(mesh), cam_arr, B, ctypes.byref(raster), _ptr(t_rgb),
                                            _ptr(t_m), float(scale_rgb), float(scale_alpha), _ptr(rgb), _ptr(alpha),
                                            _ptr(g_rgb), _ptr(g_a), _ptr(sums), _ptr(ws), nb.value, cap, _stream()))
        _order.note(key, ws)
        st = ForwardState(ws, cap, raster, cam_arr, B, -1, -1)
        if check is None:
            # status stays on the device (ws[:64]); the caller validates it
            # (graph-captured loops copy it with gmr_fit_step_scheduled)
            st.key = key
            return rgb, alpha, g_rgb, g_a, sums, st
        if not check:
            st.status_host = torch.empty(64, dtype=torch.uint8, pin_memory=True)
            st.status_host.copy_(ws[:64], non_blocking=True)
            st.status_event = torch.cuda.Event()
            st.status_event.record()
            st.key = key
            return rgb, alpha, g_rgb, g_a, sums, st
        s_, code = _status_or_raise(ws, "mesh")
        if code == L.GMR_OK:
            _capacity.note(key, cap, s_.entries)
            st.entries, st.kept = s_.entries, s_.kept
            return rgb, alpha, g_rgb, g_a, sums, st
        cap = _capacity.grow(key, s_.entries)
    raise RuntimeError("tile-entry capacity did not converge")


def render_images_u8(pos, col, faces, cams, width, height, background, rescale=True):
    """B-view forward straight to 8-bit images (rgb8 [B,H,W,3], alpha8
    [B,H,W] uint8 on the device), quantised in the blend epilogue the way
    the reference's dataset writer does (dataset.py:59-61)."""
    lib = L.load()
    dtype = pos.dtype
    B, F = len(cams), int(faces.shape[0])
    raster = raster_struct(width, height, background, dtype, rescale, 0)
    cam_arr = L.camera_struct(cams)
    mesh = mesh_struct(pos, col, faces)
    key = (F, B, int(width), int(height), dtype)
    raster.flags |= _order.flags(key, dtype)
    cap = _capacity.get(key, F * B)
    rgb8 = torch.empty((B, height, width, 3), dtype=torch.uint8, device=pos.device)
    a8 = torch.empty((B, height, width), dtype=torch.uint8, device=pos.device)
    for _ in range(3):
        nb = ctypes.c_size_t()
        L.check(lib.gmr_render_workspace_size(F, B, width, height, cap, raster.dtype, ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=pos.device)
        L.check(lib.gmr_render_images_u8(ctypes.byref(mesh), cam_arr, B, ctypes.byref(raster), _ptr(rgb8),
                                         _ptr(a8), _ptr(ws), nb.value, cap, _stream()))
        _order.note(key, ws)
        st, code = _status_or_raise(ws, "mesh")
        if code == L.GMR_OK:
            _capacity.note(key, cap, st.entries)
            return rgb8, a8
        cap = _capacity.grow(key, st.entries)
    raise RuntimeError("tile-entry capacity did not converge")


class CapacityExceeded(RuntimeError):
    """A deferred-check forward needed more tile entries than it was planned
    for; its outputs are invalid.  The capacity has been raised: re-run."""


def check_status(state: ForwardState, key=None):
    """Validate a forward launched with check=False.  Waits only for that
    forward (its status copy event), not for work enqueued after it."""
    key = getattr(state, "key", key)
    state.status_event.synchronize()
    entries, kept, bad, overflow = _parse_status(state.status_host.numpy())
    state.entries, state.kept = entries, kept
    for field in range(6):
        if bad[field] != 0xFFFFFFFF:
            raise ValueError(f"non-finite splat parameter {_FIELDS[field]!r} at splat {int(bad[field])}")
    if overflow:
        _capacity.grow(key, entries)
        raise CapacityExceeded(f"{entries} tile entries > capacity {state.capacity}")
    _capacity.note(key, state.capacity, entries)
    return state


def render_backward(state: ForwardState, pos, col, faces, rgb, g_rgb, g_alpha):
    """Vertex position/colour grads [V,3] summed over the state's views."""
    lib = L.load()
    dtype = pos.dtype
    g_rgb = g_rgb.to(dtype).contiguous()
    g_alpha = g_alpha.to(dtype).contiguous()
    topo = topology(faces, pos.shape[0])
    g_pos = torch.empty_like(pos)
    g_col = torch.empty_like(col)
    mesh = mesh_struct(pos, col, faces)
    L.check(lib.gmr_render_backward(ctypes.byref(mesh), state.cams, state.views,
                                    ctypes.byref(state.raster), _ptr(rgb), _ptr(g_rgb), _ptr(g_alpha),
                                    _ptr(g_pos), _ptr(g_col), _ptr(topo), _ptr(state.ws),
                                    state.ws.numel(), state.capacity, _stream()))
    return g_pos, g_col


class GMRRender(torch.autograd.Function):
    """rgb [B,H,W,3], alpha [B,H,W] = render(pos [V,3], col [V,3]; faces, cams)
    with autograd to pos and col (reference render_mesh/render_backward
    summed over views, losses.py:151-162)."""

    @staticmethod
    def forward(ctx, pos, col, faces, cams, width, height, background, rescale):
        pos_c, col_c = pos.detach().contiguous(), col.detach().contiguous()
        rgb, alpha, state = render_forward(pos_c, col_c, faces, cams, width, height, background, rescale)
        ctx.state = state
        ctx.save_for_backward(pos_c, col_c, faces, rgb)
        return rgb, alpha

    @staticmethod
    def backward(ctx, g_rgb, g_alpha):
        pos, col, faces, rgb = ctx.saved_tensors
        if g_rgb is None:
            g_rgb = torch.zeros_like(rgb)
        if g_alpha is None:
            g_alpha = torch.zeros(rgb.shape[:-1], dtype=rgb.dtype, device=rgb.device)
        g_pos, g_col = render_backward(ctx.state, pos, col, faces, rgb, g_rgb, g_alpha)
        return g_pos, g_col, None, None, None, None, None, None


def _check_mesh_tensors(pos, col, faces):
    if not (isinstance(pos, torch.Tensor) and isinstance(col, torch.Tensor) and isinstance(faces, torch.Tensor)):
        raise TypeError("pos, col and faces must be torch tensors")
    if pos.dtype not in _DT:
        raise ValueError(f"pos must be float32 or float64, got {pos.dtype}")
    if col.dtype != pos.dtype:
        raise ValueError(f"col dtype {col.dtype} != pos dtype {pos.dtype}")
    if faces.dtype != torch.int32:
        raise ValueError(f"faces must be int32, got {faces.dtype}")
    if pos.dim() != 2 or pos.shape[1] != 3 or col.shape != pos.shape:
        raise ValueError(f"pos and col must both be [V, 3], got {tuple(pos.shape)} and {tuple(col.shape)}")
    if faces.dim() != 2 or faces.shape[1] != 3:
        raise ValueError(f"faces must be [F, 3], got {tuple(faces.shape)}")
    if not (pos.is_cuda and col.device == pos.device and faces.device == pos.device):
        raise ValueError("pos, col and faces must be on the same CUDA device")


def render_views(pos, col, faces, cams, width, height, background=(0.0, 0.0, 0.0), rescale=True):
    """Batched torch entry: B views of one mesh, differentiable in pos/col.
    pos, col [V,3] float32|float64 (same dtype), faces [F,3] int32, all on one
    CUDA device.  Returns rgb [B,H,W,3], alpha [B,H,W] in pos's dtype."""
    _check_mesh_tensors(pos, col, faces)
    if len(cams) == 0:
        raise ValueError("need at least one camera")
    return GMRRender.apply(pos, col, faces, list(cams), int(width), int(height),
                           tuple(np.asarray(background, dtype=np.float64).reshape(3)), bool(rescale))


# ---------------------------------------------------------------------------
# splat path (rasterize / rasterize_backward stage functions)
# ---------------------------------------------------------------------------

def _splat_struct(mean2d, cov2d, depth, color, opacity):
    s = L.GmrSplats()
    s.mean2d, s.cov2d, s.depth = mean2d.data_ptr(), cov2d.data_ptr(), depth.data_ptr()
    s.color, s.opacity, s.count = color.data_ptr(), opacity.data_ptr(), int(depth.shape[0])
    return s


def rasterize_forward(mean2d, cov2d, depth, color, opacity, width, height, background):
    lib = L.load()
    dtype = mean2d.dtype
    K = int(depth.shape[0])
    raster = raster_struct(width, height, background, dtype)
    sp = _splat_struct(mean2d, cov2d, depth, color, opacity)
    key = ("splats", K, int(width), int(height), dtype)
    raster.flags |= _order.flags(key, dtype)
    cap = _capacity.get(key, K)
    rgb = torch.empty((height, width, 3), dtype=dtype, device=mean2d.device)
    alpha = torch.empty((height, width), dtype=dtype, device=mean2d.device)
    for _ in range(3):
        nb = ctypes.c_size_t()
        L.check(lib.gmr_raster_workspace_size(K, width, height, cap, raster.dtype, ctypes.byref(nb)))
        ws = torch.empty(nb.value, dtype=torch.uint8, device=mean2d.device)
        L.check(lib.gmr_rasterize_forward(ctypes.byref(sp), ctypes.byref(raster), _ptr(rgb), _ptr(alpha),
                                          _ptr(ws), nb.value, cap, _stream()))
        _order.note(key, ws)
        st, code = _status_or_raise(ws, "splats")
        if code == L.GMR_OK:
            _capacity.note(key, cap, st.entries)
            return rgb, alpha, ForwardState(ws, cap, raster, None, 1, st.entries, st.kept)
        cap = _capacity.grow(key, st.entries)
    raise RuntimeError("tile-entry capacity did not converge")


def rasterize_backward(state, mean2d, cov2d, depth, color, opacity, rgb, g_rgb, g_alpha):
    lib = L.load()
    K = int(depth.shape[0])
    dt = mean2d.dtype
    gm = torch.empty((K, 2), dtype=dt, device=mean2d.device)
    gc = torch.empty((K, 2, 2), dtype=dt, device=mean2d.device)
    gcol = torch.empty((K, 3), dtype=dt, device=mean2d.device)
    gop = torch.empty((K,), dtype=dt, device=mean2d.device)
    sp = _splat_struct(mean2d, cov2d, depth, color, opacity)
    L.check(lib.gmr_rasterize_backward(ctypes.byref(sp), ctypes.byref(state.raster), _ptr(rgb),
                                       _ptr(g_rgb.to(dt).contiguous()), _ptr(g_alpha.to(dt).contiguous()),
                                       _ptr(gm), _ptr(gc), _ptr(gcol), _ptr(gop), _ptr(state.ws),
                                       state.ws.numel(), state.capacity, _stream()))
    return gm, gc, gcol, gop


# ---------------------------------------------------------------------------
# inspection (bit-exact binning checks)
# ---------------------------------------------------------------------------

def copy_entries(state: ForwardState, items_per_view: int, mesh_path: bool):
    lib = L.load()
    dev = state.ws.device
    items = torch.empty(max(state.entries, 1), dtype=torch.int32, device=dev)
    bins = (((state.raster.width + 15) // 16) * ((state.raster.height + 15) // 16)) * state.views
    bounds = torch.empty(bins + 1, dtype=torch.int32, device=dev)
    L.check(lib.gmr_copy_entries(_ptr(state.ws), items_per_view, state.views, ctypes.byref(state.raster),
                                 state.capacity, int(mesh_path), _ptr(items), _ptr(bounds), _stream()))
    return items[:state.entries], bounds


def copy_splats(state: ForwardState, items_per_view: int, mesh_path: bool):
    lib = L.load()
    dev = state.ws.device
    dt = torch.float64 if state.raster.dtype == L.GMR_F64 else torch.float32
    n = items_per_view * state.views
    rec = torch.empty((n, 8), dtype=dt, device=dev)
    rect = torch.empty((n, 2), dtype=torch.int32, device=dev)
    cnt = torch.empty(n, dtype=torch.int32, device=dev)
    aux = torch.empty((n, 2), dtype=dt, device=dev)
    L.check(lib.gmr_copy_splats(_ptr(state.ws), items_per_view, state.views, ctypes.byref(state.raster),
                                state.capacity, int(mesh_path), _ptr(rec), _ptr(rect), _ptr(cnt), _ptr(aux),
                                _stream()))
    return rec, rect, cnt, aux


def convert(pos, col, faces, rescale=True):
    lib = L.load()
    F = int(faces.shape[0])
    dt = pos.dtype
    means = torch.empty((F, 3), dtype=dt, device=pos.device)
    cov = torch.empty((F, 3, 3), dtype=dt, device=pos.device)
    colors = torch.empty((F, 3), dtype=dt, device=pos.device)
    degen = torch.empty(F, dtype=torch.uint8, device=pos.device)
    mesh = mesh_struct(pos, col, faces)
    L.check(lib.gmr_convert(ctypes.byref(mesh), int(rescale), _DT[dt], _ptr(means), _ptr(cov), _ptr(colors),
                            _ptr(degen), _stream()))
    return means, cov, colors, degen.bool()


def convert_backward(pos, col, faces, g_means, g_cov, g_colors, rescale=True):
    lib = L.load()
    dt = pos.dtype
    topo = topology(faces, pos.shape[0])
    nb = ctypes.c_size_t()
    L.check(lib.gmr_convert_scratch_size(faces.shape[0], _DT[dt], ctypes.byref(nb)))
    scratch = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=pos.device)
    gp = torch.empty_like(pos)
    gc = torch.empty_like(col)
    mesh = mesh_struct(pos, col, faces)
    L.check(lib.gmr_convert_backward(ctypes.byref(mesh), int(rescale), _DT[dt], _ptr(g_means.to(dt).contiguous()),
                                     _ptr(g_cov.to(dt).contiguous()), _ptr(g_colors.to(dt).contiguous()),
                                     _ptr(gp), _ptr(gc), _ptr(topo), _ptr(scratch), nb.value, _stream()))
    return gp, gc
