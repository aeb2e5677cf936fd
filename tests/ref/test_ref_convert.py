"""The reference's conversion-backward tests, run against the CUDA drop-in.

Adapted from /root/reference/pkg/tests/test_convert.py:324-432
(`_conversion_loss` and TestConvertBackward, including the clamped-kappa
branch, shared vertices and degenerate facets): bodies and tolerances are the
reference's; imports rebound (meshsplat_shim).  The clamped-branch case
computes the facet area directly instead of through the reference's
internal `triangle_moments`.
"""

import numpy as np
import pytest

from fd_utils import finite_difference_gradient, relative_error
from meshsplat_shim import TriangleMesh, convert_backward, convert_mesh, make_icosphere

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(gmr):
    return gmr


def _conversion_loss(mesh_verts, facets, colors, gm, gc, gcol, rescale=True):
    mesh = TriangleMesh(mesh_verts, facets, colors)
    cloud = convert_mesh(mesh, rescale=rescale)
    return float(np.sum(gm * cloud.means)) + float(np.sum(gc * cloud.cov3d)) + float(np.sum(gcol * cloud.colors))


def test_mean_only_single_facet():
    mesh = TriangleMesh(np.eye(3), [(0, 1, 2)])
    cloud = convert_mesh(mesh)
    gm = np.array([[1.0, 2.0, 3.0]])
    gv, gcol = convert_backward(mesh, cloud, gm, np.zeros((1, 3, 3)), np.zeros((1, 3)))
    for r in range(3):
        assert np.allclose(gv[r], gm[0] / 3)
    assert np.allclose(gcol, 0.0)


def test_zero_upstream_zero_out():
    mesh = make_icosphere(20)
    cloud = convert_mesh(mesh)
    gv, gcol = convert_backward(mesh, cloud, np.zeros((20, 3)), np.zeros((20, 3, 3)), np.zeros((20, 3)))
    assert np.all(gv == 0) and np.all(gcol == 0)


def test_color_backward_is_thirds():
    mesh = TriangleMesh(np.eye(3), [(0, 1, 2)])
    cloud = convert_mesh(mesh)
    gcol_up = np.array([[0.3, -0.6, 0.9]])
    _, gcol = convert_backward(mesh, cloud, np.zeros((1, 3)), np.zeros((1, 3, 3)), gcol_up)
    assert np.allclose(gcol, np.repeat(gcol_up / 3, 3, axis=0))


def test_finite_difference_oracle():
    rng = np.random.default_rng(42)
    facets = np.array([(0, 1, 2)])
    worst = 0.0
    for _ in range(50):
        verts, colors = rng.normal(size=(3, 3)), rng.random((3, 3))
        gm, gc, gcol = rng.normal(size=(1, 3)), rng.normal(size=(1, 3, 3)), rng.normal(size=(1, 3))
        mesh = TriangleMesh(verts, facets, colors)
        gv, _ = convert_backward(mesh, convert_mesh(mesh), gm, gc, gcol)
        num = finite_difference_gradient(lambda x: _conversion_loss(x, facets, colors, gm, gc, gcol),
                                         verts.copy(), eps=1e-5)
        worst = max(worst, relative_error(gv, num))
    assert worst < 1e-5


def test_finite_difference_no_rescale():
    rng = np.random.default_rng(43)
    facets = np.array([(0, 1, 2)])
    for _ in range(10):
        verts, colors = rng.normal(size=(3, 3)), rng.random((3, 3))
        gm, gc, gcol = rng.normal(size=(1, 3)), rng.normal(size=(1, 3, 3)), rng.normal(size=(1, 3))
        mesh = TriangleMesh(verts, facets, colors)
        cloud = convert_mesh(mesh, rescale=False)
        gv, _ = convert_backward(mesh, cloud, gm, gc, gcol)
        num = finite_difference_gradient(lambda x: _conversion_loss(x, facets, colors, gm, gc, gcol, rescale=False),
                                         verts.copy(), eps=1e-5)
        assert relative_error(gv, num) < 1e-5


def test_finite_difference_clamped_branch():
    rng = np.random.default_rng(44)
    facets = np.array([(0, 1, 2)])
    base = rng.normal(size=(3, 3))
    area = 0.5 * np.linalg.norm(np.cross(base[1] - base[0], base[2] - base[0]))
    verts = base * np.sqrt(1e-7 / area)
    colors = rng.random((3, 3))
    gm, gc, gcol = rng.normal(size=(1, 3)), rng.normal(size=(1, 3, 3)), rng.normal(size=(1, 3))
    mesh = TriangleMesh(verts, facets, colors)
    cloud = convert_mesh(mesh)
    assert not cloud.degenerate[0]
    gv, _ = convert_backward(mesh, cloud, gm, gc, gcol)
    num = finite_difference_gradient(lambda x: _conversion_loss(x, facets, colors, gm, gc, gcol),
                                     verts.copy(), eps=1e-9)
    assert relative_error(gv, num) < 1e-3


def test_shared_vertex_accumulation():
    verts = np.array([(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0.5)], dtype=float)
    facets = np.array([(0, 1, 2), (1, 3, 2)])
    mesh = TriangleMesh(verts, facets)
    cloud = convert_mesh(mesh)
    rng = np.random.default_rng(45)
    gm, gc, gcol = rng.normal(size=(2, 3)), rng.normal(size=(2, 3, 3)), np.zeros((2, 3))
    gv, _ = convert_backward(mesh, cloud, gm, gc, gcol)
    num = finite_difference_gradient(lambda x: _conversion_loss(x, facets, mesh.colors, gm, gc, gcol),
                                     verts.copy(), eps=1e-5)
    assert relative_error(gv, num) < 1e-5


def test_degenerate_still_gets_mean_grad():
    verts = np.array([(0, 0, 0), (1, 0, 0), (2, 0, 0)], dtype=float)
    mesh = TriangleMesh(verts, [(0, 1, 2)])
    gv, _ = convert_backward(mesh, convert_mesh(mesh), np.ones((1, 3)), np.ones((1, 3, 3)), np.zeros((1, 3)))
    assert np.allclose(gv, 1 / 3)


def test_shape_mismatch_rejected():
    mesh = make_icosphere(20)
    cloud = convert_mesh(mesh)
    with pytest.raises(ValueError):
        convert_backward(mesh, cloud, np.zeros((19, 3)), np.zeros((20, 3, 3)), np.zeros((20, 3)))
