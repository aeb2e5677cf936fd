"""CPU-side checks of the boundary: libgmr.so loads without a GPU and exports
every symbol include/gmr.h declares; host containers and generators behave
like the reference's."""

import os
import re

import numpy as np
import pytest

from paper_2602_14493_b200 import lib
from paper_2602_14493_b200.camera import CameraError, Camera, default_intrinsics, look_at
from paper_2602_14493_b200.mesh import MeshError, TriangleMesh, make_geodesic_sphere, make_icosphere

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gmr.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gmr_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("gmr_render_forward", "gmr_render_backward", "gmr_rasterize_forward",
              "gmr_rasterize_backward", "gmr_status", "gmr_topology_build", "gmr_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(lib.LIB_PATH):
        from paper_2602_14493_b200 import build
        build.build()
    cdll = lib.load_cdll()
    for s in declared_symbols():
        assert hasattr(cdll, s), s
    assert set(declared_symbols()) == set(lib._SIGNATURES), "ctypes binding out of sync with gmr.h"
    assert b"sm_100a" in cdll.gmr_version()


def test_argument_errors_without_gpu():
    """Validation happens before any CUDA call: usable on a CPU box."""
    cdll = lib.load_cdll()
    import ctypes
    nb = ctypes.c_size_t()
    assert cdll.gmr_render_workspace_size(-1, 1, 8, 8, 0, 0, ctypes.byref(nb)) == lib.GMR_EINVAL
    assert b"bad workspace" in cdll.gmr_last_error()
    assert cdll.gmr_render_workspace_size(100, 2, 32, 32, 1000, 0, ctypes.byref(nb)) == lib.GMR_OK
    small = nb.value
    assert cdll.gmr_render_workspace_size(100, 2, 32, 32, 100000, 0, ctypes.byref(nb)) == lib.GMR_OK
    assert nb.value > small
    assert cdll.gmr_render_workspace_size(100, 2, 32, 32, 1 << 32, 0, ctypes.byref(nb)) == lib.GMR_EINVAL
    assert b"2^32" in cdll.gmr_last_error()
    assert cdll.gmr_raster_workspace_size(10, 32, 32, 1 << 33, 0, ctypes.byref(nb)) == lib.GMR_EINVAL
    r = lib.GmrRaster()
    r.width, r.height, r.dtype = 0, 8, 0
    m = lib.GmrMesh()
    assert cdll.gmr_render_forward(ctypes.byref(m), None, 1, ctypes.byref(r), None, None, None, 0, 0,
                                   None) == lib.GMR_EINVAL


def test_camera_validation_matches_reference():
    with pytest.raises(CameraError):
        Camera(rotation=np.eye(3) + 1e-6, translation=np.zeros(3), fx=1, fy=1, cx=0, cy=0, width=4, height=4)
    with pytest.raises(CameraError):
        Camera(rotation=np.eye(3), translation=np.zeros(3), fx=1, fy=1, cx=0, cy=0, width=4, height=4,
               near=2.0, far=1.0)
    cam = look_at((0, 0, 3), (0, 0, 0), **default_intrinsics(64, 64))
    assert np.allclose(cam.position, (0, 0, 3))
    assert cam.world_to_camera(np.zeros(3))[2] == pytest.approx(3.0)


def test_mesh_validation_matches_reference():
    with pytest.raises(MeshError):
        TriangleMesh(np.eye(3), [(0, 1, 3)])
    with pytest.raises(MeshError):
        TriangleMesh(np.eye(3), [(0, 1, 1)])
    with pytest.raises(MeshError):
        TriangleMesh(np.eye(3), [(0, 1, 2)], colors=np.full((3, 3), 2.0))
    m = make_icosphere(1280)
    assert (m.num_facets, m.num_vertices) == (1280, 642)


@pytest.mark.parametrize("n", [1, 2, 7, 20])
def test_geodesic_sphere_is_closed_and_outward(n):
    m = make_geodesic_sphere(n)
    assert m.num_facets == 20 * n * n and m.num_vertices == 10 * n * n + 2
    f, v = m.facets, m.vertices
    e = np.sort(f[:, [0, 1, 1, 2, 2, 0]].reshape(-1, 2), axis=1)
    _, counts = np.unique(e, axis=0, return_counts=True)
    assert set(counts.tolist()) == {2}
    nrm = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    assert ((nrm * v[f].mean(axis=1)).sum(axis=1) > 0).all()
    assert np.all(m.colors >= 0.1) and np.all(m.colors <= 0.9)
