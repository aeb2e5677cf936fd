"""The names the reference's own test modules import from `meshsplat`,
bound to the CUDA drop-in (paper_2602_14493_b200), so those tests run
against the device path (the shim keeps the
reference's names and signatures "so the reference's own tests can be
pointed at it").  Test infrastructure only."""

from dataclasses import dataclass, field

import numpy as np

from paper_2602_14493_b200.api import (ALPHA_CLAMP, DILATION, GaussianCloud, LossWeights, RenderOutput,  # noqa: F401
                                       Splat2D, SplatBatch, color_loss, convert_backward, convert_mesh,
                                       edge_length_loss, laplacian_loss, project_cloud, project_cloud_backward,
                                       rasterize, rasterize_backward, render_backward, render_mesh,
                                       silhouette_loss, total_loss)
from paper_2602_14493_b200.camera import Camera, CameraError, default_intrinsics, look_at  # noqa: F401
from paper_2602_14493_b200.mesh import TriangleMesh, make_grid_cube, make_icosphere  # noqa: F401


@dataclass
class FacetGaussian:
    """meshsplat.convert.FacetGaussian (the fields the projection uses)."""
    mean: np.ndarray
    cov3d: np.ndarray
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    scales: np.ndarray = field(default_factory=lambda: np.full(3, 0.1))
    opacity: float = 1.0
    color_dc: np.ndarray = field(default_factory=lambda: np.full(3, 0.5))
    source_facet: int = -1
    degenerate: bool = False


def _cloud(g):
    return GaussianCloud(means=np.asarray(g.mean, np.float64)[None], cov3d=np.asarray(g.cov3d, np.float64)[None],
                         colors=np.asarray(g.color_dc, np.float64)[None], opacities=np.array([float(g.opacity)]),
                         degenerate=np.array([bool(g.degenerate)]))


def project_gaussian(g, camera):
    """render.py:148-165: one Gaussian through project_cloud; None if culled."""
    b = project_cloud(_cloud(g), camera)
    if len(b) == 0:
        return None
    return Splat2D(mean2d=b.mean2d[0], cov2d_screen=b.cov2d[0], depth=float(b.depth[0]), color=b.color[0],
                   opacity=float(b.opacity[0]), source=g.source_facet)


def project_backward(g, camera, grad_mean2d, grad_cov2d):
    """render.py:405-426: project_cloud_backward for one Gaussian (zero grads
    when it is culled)."""
    cloud = _cloud(g)
    b = project_cloud(cloud, camera)
    if len(b) == 0:
        return np.zeros(3), np.zeros((3, 3))
    g3, gc3 = project_cloud_backward(b, cloud, camera, np.asarray(grad_mean2d, np.float64)[None],
                                     np.asarray(grad_cov2d, np.float64)[None])
    return g3[0], gc3[0]
