"""Batched ground-truth view rendering.

`make_views` keeps the reference's dataset writer (`pkg/src/meshsplat/
dataset.py:118-164`): normalise the mesh, render it from a Fibonacci
hemisphere of cameras, write one RGB and one mask PNG per view, the camera
file, the normalised target mesh and a metadata file -- byte-identical files.

Rendering is the device forward (K1-K3) over many views per call, with the
8-bit quantisation of `_save_png` (`:59-61`) fused into the blend epilogue
(`gmr_render_images_u8`), so only uint8 images cross PCIe.  PNG encoding
(PIL) runs on host threads while the device renders the next group of
views.  The default render dtype is float64, as the reference's
`render_mesh` default (`render.py:442`).  Reading datasets back is outside
the hot path and not provided.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .camera import fibonacci_hemisphere, hemisphere_cameras, save_cameras
from .mesh import TriangleMesh, normalize_mesh

VERSION = "0.1.0"

__all__ = ["ViewDataset", "make_views", "render_view_images", "fibonacci_hemisphere", "hemisphere_cameras"]


def _png(path, image_u8) -> None:
    from PIL import Image
    Image.fromarray(image_u8).save(path)


@dataclass(frozen=True)
class ViewDataset:
    """What make_views wrote (the reference's return type, dataset.py:71-97,
    without its readers)."""
    root: Path
    cameras: tuple
    rgb_paths: tuple
    mask_paths: tuple
    metadata: dict

    def __len__(self):
        return len(self.cameras)


def _views_per_call(F: int, W: int, H: int, n: int) -> int:
    # keep one call's items (F x B) and pixels (W x H x B) in a few hundred MB
    # of workspace; the view loop inside a call is already batched
    return max(1, min(n, 1024, (1 << 25) // max(F, 1), (1 << 27) // max(W * H, 1)))


def render_view_images(mesh: TriangleMesh, cameras, background=(0.0, 0.0, 0.0), dtype=np.float64,
                       on_group=None):
    """Render every camera on the device and return (rgb8 [N,H,W,3],
    mask8 [N,H,W]) uint8 host arrays, quantised like `_save_png`.  All
    cameras must share one resolution.  `on_group(first, rgb8, mask8)` is
    called for each finished group of views (host arrays), in order."""
    import torch

    from . import engine
    cams = list(cameras)
    if not cams:
        raise ValueError("need at least one view")
    W, H = cams[0].width, cams[0].height
    if any((c.width, c.height) != (W, H) for c in cams):
        raise ValueError("all cameras must share one resolution")
    tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    dev = torch.device("cuda", torch.cuda.current_device())
    pos = torch.tensor(np.asarray(mesh.vertices), dtype=tdt, device=dev)
    col = torch.tensor(np.asarray(mesh.colors), dtype=tdt, device=dev)
    faces = torch.tensor(np.asarray(mesh.facets), dtype=torch.int32, device=dev)
    bg = tuple(float(x) for x in np.asarray(background, np.float64).reshape(3))
    N = len(cams)
    out_rgb = np.empty((N, H, W, 3), np.uint8)
    out_a = np.empty((N, H, W), np.uint8)
    step = _views_per_call(int(faces.shape[0]), W, H, N)
    host = [(torch.empty((step, H, W, 3), dtype=torch.uint8, pin_memory=True),
             torch.empty((step, H, W), dtype=torch.uint8, pin_memory=True)) for _ in range(2)]
    pending = None
    for k, v0 in enumerate(range(0, N, step)):
        nv = min(step, N - v0)
        rgb8, a8 = engine.render_images_u8(pos, col, faces, cams[v0:v0 + nv], W, H, bg)
        hr, ha = host[k % 2]
        hr[:nv].copy_(rgb8, non_blocking=True)
        ha[:nv].copy_(a8, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        if pending is not None:
            _drain(pending, out_rgb, out_a, on_group)
        pending = (ev, v0, nv, hr, ha)
    _drain(pending, out_rgb, out_a, on_group)
    return out_rgb, out_a


def _drain(pending, out_rgb, out_a, on_group):
    ev, v0, nv, hr, ha = pending
    ev.synchronize()
    out_rgb[v0:v0 + nv] = hr[:nv].numpy()
    out_a[v0:v0 + nv] = ha[:nv].numpy()
    if on_group is not None:
        on_group(v0, out_rgb[v0:v0 + nv], out_a[v0:v0 + nv])


def _write_metadata(path: Path, meta: dict) -> None:
    """`key = value` lines in key order (the reference's metadata.txt)."""
    path.write_text("".join(f"{k} = {meta[k]}\n" for k in sorted(meta)))


def _write_ply_ascii(mesh: TriangleMesh, path: Path) -> None:
    """The normalised target mesh as the reference writes it (mesh.py:395-421
    format): ASCII PLY, double xyz + rgb as %.17g, triangle index lists."""
    with open(path, "w") as fh:
        fh.write("ply\nformat ascii 1.0\ncomment meshsplat\n"
                 f"element vertex {mesh.num_vertices}\n"
                 + "".join(f"property double {p}\n" for p in ("x", "y", "z", "red", "green", "blue"))
                 + f"element face {mesh.num_facets}\nproperty list uchar int vertex_indices\nend_header\n")
        np.savetxt(fh, np.concatenate([mesh.vertices, mesh.colors], axis=1), fmt="%.17g", delimiter=" ")
        np.savetxt(fh, np.asarray(mesh.facets, np.int64), fmt="3 %d %d %d")


def make_views(mesh, n_views: int = 253, resolution=(256, 256), radius: float = 3.0, up: str = "z",
               seed: int = 0, out_dir=None, background=(0.0, 0.0, 0.0), dtype=np.float64,
               png_threads: int | None = None) -> ViewDataset:
    """Normalise `mesh` (a TriangleMesh), render
    `n_views` hemisphere views on the device and write the dataset directory
    (dataset.py:118-164: view_%04d.png, mask_%04d.png, cameras.txt,
    target_mesh.ply, metadata.txt)."""
    if out_dir is None:
        raise ValueError("out_dir is required")
    if not isinstance(mesh, TriangleMesh):
        raise TypeError("make_views takes a TriangleMesh (mesh file readers are outside the hot path)")
    if isinstance(resolution, int):
        resolution = (resolution, resolution)
    mesh, _ = normalize_mesh(mesh)
    cams = hemisphere_cameras(n_views, radius, resolution, up)
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    rgb_paths = tuple(out / f"view_{i:04d}.png" for i in range(n_views))
    mask_paths = tuple(out / f"mask_{i:04d}.png" for i in range(n_views))
    jobs = []
    with ThreadPoolExecutor(max_workers=png_threads or min(16, os.cpu_count() or 1)) as pool:
        def encode(first, rgb8, mask8):
            for j in range(len(rgb8)):
                jobs.append(pool.submit(_png, rgb_paths[first + j], rgb8[j]))
                jobs.append(pool.submit(_png, mask_paths[first + j], mask8[j]))
        render_view_images(mesh, cams, background, dtype, on_group=encode)
        for j in jobs:
            j.result()
    save_cameras(cams, out / "cameras.txt")
    _write_ply_ascii(mesh, out / "target_mesh.ply")
    meta = {"n_views": n_views, "width": resolution[0], "height": resolution[1], "radius": radius,
            "up": up, "seed": seed, "version": VERSION}
    _write_metadata(out / "metadata.txt", meta)
    return ViewDataset(root=out, cameras=tuple(cams), rgb_paths=rgb_paths, mask_paths=mask_paths,
                       metadata=meta)
