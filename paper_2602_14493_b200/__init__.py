"""paper_2602_14493_b200 — B200-native Gaussian Mesh Renderer hot path.

Drop-in for the reference renderer's API (meshsplat render/convert/losses):
mesh + cameras -> image, with gradients to the vertices, computed by
hand-written sm_100a CUDA kernels in libgmr.so (C ABI: include/gmr.h).
"""

from . import lib
from .camera import (Camera, CameraError, default_intrinsics, fibonacci_hemisphere,
                     hemisphere_cameras, look_at, sphere_views)
from .mesh import MeshError, TriangleMesh, make_geodesic_sphere, make_icosphere, seeded_colors

_API = ("RenderOutput", "RenderContext", "Splat2D", "SplatBatch", "GaussianCloud", "LossWeights", "LossReport",
        "project_cloud", "project_cloud_backward",
        "render_mesh", "render_backward", "rasterize", "rasterize_backward", "convert_mesh",
        "convert_backward", "total_loss", "color_loss", "silhouette_loss", "edge_length_loss",
        "laplacian_loss", "export_gaussians", "ALPHA_CLAMP", "CONTRIB_FLOOR", "TRANSMITTANCE_STOP", "DILATION", "TILE")
_ENGINE = ("render_views", "GMRRender")


def __getattr__(name):
    # torch-backed modules load on first use so `import paper_2602_14493_b200`
    # stays cheap on machines that only build
    if name in _API:
        from . import api
        return getattr(api, name)
    if name in _ENGINE:
        from . import engine
        return getattr(engine, name)
    if name in ("api", "engine", "dist", "metrics", "dataset", "fit"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)


__all__ = list(_API) + list(_ENGINE) + [
    "lib", "Camera", "CameraError", "look_at", "default_intrinsics", "fibonacci_hemisphere",
    "hemisphere_cameras", "sphere_views", "TriangleMesh", "MeshError", "make_icosphere",
    "make_geodesic_sphere", "seeded_colors"]
