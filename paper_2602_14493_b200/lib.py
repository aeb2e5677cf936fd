"""ctypes binding of libgmr.so (the C ABI declared in include/gmr.h).

This is the reference-side binding a maintainer would add: plain pointers,
sizes and a stream handle cross the boundary; no torch types.  The product
path has no CPU fallback: `load()` raises if the library or a CUDA device is
missing.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMR_LIB_PATH") or os.path.join(_HERE, "libgmr.so")

GMR_OK = 0
GMR_EINVAL = -1
GMR_ENONFINITE = -2
GMR_EWORKSPACE = -3
GMR_ECUDA = -4
GMR_ECAPACITY = -5
GMR_F32 = 0
GMR_F64 = 1
FLAG_DEBUG_AUX = 1
FLAG_FULL_TILE_LISTS = 2
FLAG_TILE_DEPTH_SORT = 4
STAGES = ("convert_project", "depth_sort", "scan_emit", "tile_sort_ranges", "blend_forward",
          "blend_backward", "face_backward", "vertex_gather")

c_i32, c_i64, c_sz, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p


class GmrCamera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("near_plane", ctypes.c_double), ("far_plane", ctypes.c_double)]


class GmrMesh(ctypes.Structure):
    _fields_ = [("positions", c_vp), ("colors", c_vp), ("faces", c_vp),
                ("num_vertices", c_i64), ("num_faces", c_i64)]


class GmrRaster(ctypes.Structure):
    _fields_ = [("width", c_i32), ("height", c_i32), ("background", ctypes.c_double * 3),
                ("dtype", c_i32), ("rescale", c_i32), ("flags", c_i32)]


class GmrStatus(ctypes.Structure):
    _fields_ = [("entries", c_i64), ("entry_capacity", c_i64), ("kept", c_i64),
                ("overflow", c_i32), ("nonfinite_field", c_i32), ("nonfinite_item", c_i64)]


class GmrFitState(ctypes.Structure):
    _fields_ = [("positions", c_vp), ("colors", c_vp), ("positions_f32", c_vp), ("colors_f32", c_vp),
                ("m_pos", c_vp), ("v_pos", c_vp), ("m_col", c_vp), ("v_col", c_vp),
                ("step_counts", c_vp), ("flags", c_vp)]


class GmrMeshGraph(ctypes.Structure):
    _fields_ = [("edges", c_vp), ("num_edges", c_i64), ("ve_ptr", c_vp), ("ve_slot", c_vp),
                ("adj_ptr", c_vp), ("adj", c_vp)]


class GmrSplats(ctypes.Structure):
    _fields_ = [("mean2d", c_vp), ("cov2d", c_vp), ("depth", c_vp), ("color", c_vp),
                ("opacity", c_vp), ("count", c_i64)]


P = ctypes.POINTER
_SIGNATURES = {
    "gmr_last_error": ([], ctypes.c_char_p),
    "gmr_version": ([], ctypes.c_char_p),
    "gmr_timing_enable": ([c_i32], None),
    "gmr_launch_count": ([], c_i64),
    "gmr_timing_read": ([P(ctypes.c_double), P(c_i64), c_i32, c_i32], c_i32),
    "gmr_render_workspace_size": ([c_i64, c_i32, c_i32, c_i32, c_i64, c_i32, P(c_sz)], c_i32),
    "gmr_render_forward": ([P(GmrMesh), P(GmrCamera), c_i32, P(GmrRaster), c_vp, c_vp, c_vp,
                            c_sz, c_i64, c_vp], c_i32),
    "gmr_status": ([c_vp, P(GmrStatus), c_vp], c_i32),
    "gmr_fit_scratch_size": ([c_i64, c_i64, P(c_sz)], c_i32),
    "gmr_fit_step": ([P(GmrFitState), P(GmrMeshGraph), c_i64, c_vp, c_vp, c_vp] + [ctypes.c_double] * 11
                     + [c_i32, c_vp, c_vp, c_sz, c_vp], c_i32),
    "gmr_fit_step_scheduled": ([P(GmrFitState), P(GmrMeshGraph), c_i64, c_vp, c_vp, c_vp] + [ctypes.c_double] * 6
                               + [c_vp, c_vp] + [ctypes.c_double] * 3 + [c_i32, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp],
                               c_i32),
    "gmr_project": ([c_vp, c_vp, c_i64, P(GmrCamera), c_i32, c_i32, c_i32] + [c_vp] * 7 + [c_vp], c_i32),
    "gmr_project_backward": ([c_vp, c_vp, c_i64, P(GmrCamera), c_i32, c_vp, c_vp, c_vp, c_vp, c_vp], c_i32),
    "gmr_mesh_regularizers": ([c_vp, P(GmrMeshGraph), c_i64, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp], c_i32),
    "gmr_image_loss_scratch_size": ([c_i64, P(c_sz)], c_i32),
    "gmr_image_loss": ([c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_sz, c_vp], c_i32),
    "gmr_render_forward_loss": ([P(GmrMesh), P(GmrCamera), c_i32, P(GmrRaster), c_vp, c_vp, ctypes.c_double,
                                 ctypes.c_double, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_i64, c_vp], c_i32),
    "gmr_render_forward_ex": ([P(GmrMesh), P(GmrCamera), c_i32, P(GmrRaster), c_vp, c_vp, c_vp, c_sz, c_i64,
                               c_vp, c_vp, c_vp], c_i32),
    "gmr_render_images_u8": ([P(GmrMesh), P(GmrCamera), c_i32, P(GmrRaster), c_vp, c_vp, c_vp, c_sz, c_i64,
                              c_vp], c_i32),
    "gmr_topology_size": ([c_i64, c_i64, P(c_sz)], c_i32),
    "gmr_export_gaussians": ([c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp], c_i32),
    "gmr_surface_prepare_size": ([c_i64, P(c_sz)], c_i32),
    "gmr_surface_prepare": ([c_vp, c_vp, c_i64, c_i64, c_vp, c_sz, c_vp, c_vp], c_i32),
    "gmr_surface_sample": ([c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp], c_i32),
    "gmr_nearest_scratch_size": ([c_i64, c_i64, P(c_sz)], c_i32),
    "gmr_nearest": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_sz, c_vp], c_i32),
    "gmr_chamfer_scratch_size": ([c_i64, c_i64, P(c_sz)], c_i32),
    "gmr_chamfer_nc": ([c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_sz, c_vp], c_i32),
    "gmr_image_metrics_scratch_size": ([c_i32, c_i32, c_i32, c_i32, P(c_sz)], c_i32),
    "gmr_image_metrics": ([c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_sz, c_vp], c_i32),
    "gmr_topology_build": ([c_vp, c_i64, c_i64, c_vp, c_sz, c_vp], c_i32),
    "gmr_render_backward": ([P(GmrMesh), P(GmrCamera), c_i32, P(GmrRaster), c_vp, c_vp, c_vp,
                             c_vp, c_vp, c_vp, c_vp, c_sz, c_i64, c_vp], c_i32),
    "gmr_raster_workspace_size": ([c_i64, c_i32, c_i32, c_i64, c_i32, P(c_sz)], c_i32),
    "gmr_rasterize_forward": ([P(GmrSplats), P(GmrRaster), c_vp, c_vp, c_vp, c_sz, c_i64,
                               c_vp], c_i32),
    "gmr_rasterize_backward": ([P(GmrSplats), P(GmrRaster), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                c_vp, c_vp, c_sz, c_i64, c_vp], c_i32),
    "gmr_copy_entries": ([c_vp, c_i64, c_i32, P(GmrRaster), c_i64, c_i32, c_vp, c_vp, c_vp],
                         c_i32),
    "gmr_copy_splats": ([c_vp, c_i64, c_i32, P(GmrRaster), c_i64, c_i32, c_vp, c_vp, c_vp, c_vp,
                         c_vp], c_i32),
    "gmr_convert": ([P(GmrMesh), c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp], c_i32),
    "gmr_convert_scratch_size": ([c_i64, c_i32, P(c_sz)], c_i32),
    "gmr_convert_backward": ([P(GmrMesh), c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                              c_vp, c_sz, c_vp], c_i32),
}

_lib = None


class GmrError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"gmr error {code}: {message}")
        self.code = code


def load_cdll(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library and bind every symbol (no GPU needed)."""
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                           " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def load() -> ctypes.CDLL:
    """The CUDA product library; raises unless a CUDA device is present."""
    global _lib
    if _lib is None:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2602_14493_b200 needs a CUDA device (sm_100a); no CPU fallback")
        _lib = load_cdll()
    return _lib


def check(code: int):
    if code != GMR_OK:
        msg = _lib.gmr_last_error().decode() if _lib is not None else "?"
        raise GmrError(code, msg)


def camera_struct(cams) -> ctypes.Array:
    """GmrCamera[n] (18 float64 each: R row-major, t, fx, fy, cx, cy, near,
    far) filled from one packed array."""
    n = len(cams)
    vals = np.empty((n, 18), np.float64)
    for i, c in enumerate(cams):
        vals[i, 0:9] = np.asarray(c.rotation, np.float64).reshape(-1)
        vals[i, 9:12] = np.asarray(c.translation, np.float64).reshape(-1)
        vals[i, 12:] = (c.fx, c.fy, c.cx, c.cy, c.near, c.far)
    return (GmrCamera * n).from_buffer_copy(vals.tobytes())
