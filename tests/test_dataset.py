"""batched ground-truth view rendering (make_views).

Golden: tests/golden/views_ico320_13.npz, written by the reference's own
make_views (dataset.py:118-164) -- decoded PNGs, SHA-256 of every file and
the text files.  CPU tests pin the oracle and the host-side formats; the GPU
test runs the device path (gmr_render_images_u8) and requires identical
images and identical file bytes."""

import hashlib
import os

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc
from paper_2602_14493_b200 import camera as gcam
from paper_2602_14493_b200 import mesh as gmesh


def _case():
    c = gc.views_case()
    m = gmesh.TriangleMesh(c["vertices"], c["facets"], c["colors"])
    return c, m


def _png_levels(x):
    # dataset.py:59-61
    return np.round(np.clip(np.asarray(x, np.float64), 0.0, 1.0) * 255.0).astype(np.uint8)


def test_oracle_views_match_reference_pngs():
    c, m = _case()
    g = gc.load("views_ico320_13")
    nm, _ = gmesh.normalize_mesh(m)
    cams = gcam.hemisphere_cameras(c["n_views"], c["radius"], c["resolution"])
    for i in (0, 5, 12):
        rgb, alpha, _ = orc.render(nm.vertices, nm.facets, nm.colors, cams[i], c["background"], True, np.float64)
        np.testing.assert_array_equal(_png_levels(rgb), g["rgb"][i])
        np.testing.assert_array_equal(_png_levels(alpha), g["mask"][i])


def test_camera_mesh_and_metadata_files_match_reference(tmp_path):
    c, m = _case()
    g = gc.load("views_ico320_13")
    nm, _ = gmesh.normalize_mesh(m)
    cams = gcam.hemisphere_cameras(c["n_views"], c["radius"], c["resolution"])
    gcam.save_cameras(cams, tmp_path / "cameras.txt")
    gmesh.save_mesh(nm, tmp_path / "target_mesh.ply")
    assert (tmp_path / "cameras.txt").read_text() == str(g["cameras_txt"])
    assert (tmp_path / "target_mesh.ply").read_text() == str(g["ply_txt"])
    back = gcam.load_cameras(tmp_path / "cameras.txt")
    for a, b in zip(back, cams):
        np.testing.assert_array_equal(a.rotation, b.rotation)
        np.testing.assert_array_equal(a.translation, b.translation)
        assert (a.fx, a.fy, a.cx, a.cy, a.width, a.height) == (b.fx, b.fy, b.cx, b.cy, b.width, b.height)
    r = gmesh.load_mesh(tmp_path / "target_mesh.ply")
    np.testing.assert_array_equal(r.vertices, nm.vertices)
    np.testing.assert_array_equal(r.colors, nm.colors)
    np.testing.assert_array_equal(r.facets, nm.facets)
    from paper_2602_14493_b200 import dataset
    dataset._write_metadata(tmp_path / "metadata.txt",
                            {"n_views": c["n_views"], "width": 64, "height": 48, "radius": 3.0, "up": "z",
                             "seed": 0, "version": dataset.VERSION})
    assert (tmp_path / "metadata.txt").read_text() == str(g["metadata_txt"])


def test_mesh_readers(tmp_path):
    (tmp_path / "q.obj").write_text("# quad\nv 0 0 0 1 0 0\nv 1 0 0 0 1 0\nv 1 1 0 0 0 1\nv 0 1 0 1 1 1\n"
                                   "f 1/1 2/2 3/3 4/4\n")
    m = gmesh.load_mesh(tmp_path / "q.obj")
    assert m.facets.tolist() == [[0, 1, 2], [0, 2, 3]]
    np.testing.assert_array_equal(m.colors[1], [0, 1, 0])
    # binary little-endian PLY with uchar colours
    head = ("ply\nformat binary_little_endian 1.0\nelement vertex 3\nproperty float x\nproperty float y\n"
            "property float z\nproperty uchar red\nproperty uchar green\nproperty uchar blue\n"
            "element face 1\nproperty list uchar int vertex_indices\nend_header\n").encode()
    vt = np.zeros(3, dtype=[("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("r", "u1"), ("g", "u1"), ("b", "u1")])
    vt["x"] = [0, 1, 0]
    vt["y"] = [0, 0, 1]
    vt["r"] = [255, 0, 51]
    body = vt.tobytes() + bytes([3]) + np.array([0, 1, 2], "<i4").tobytes()
    (tmp_path / "t.ply").write_bytes(head + body)
    t = gmesh.load_mesh(tmp_path / "t.ply")
    assert t.facets.tolist() == [[0, 1, 2]]
    np.testing.assert_allclose(t.colors[:, 0], [1.0, 0.0, 0.2])
    with pytest.raises(gmesh.MeshParseError):
        (tmp_path / "bad.obj").write_text("v 0 0 0\nf 1 2 3\n")
        gmesh.load_mesh(tmp_path / "bad.obj")
    with pytest.raises(gmesh.MeshParseError):
        gmesh.load_mesh(tmp_path / "x.stl")


def test_load_views_and_splits(tmp_path):
    from PIL import Image

    from paper_2602_14493_b200 import dataset
    c, m = _case()
    g = gc.load("views_ico320_13")
    cams = gcam.hemisphere_cameras(c["n_views"], c["radius"], c["resolution"])
    gcam.save_cameras(cams, tmp_path / "cameras.txt")
    for i in range(c["n_views"]):
        Image.fromarray(g["rgb"][i]).save(tmp_path / f"view_{i:04d}.png")
        Image.fromarray(g["mask"][i]).save(tmp_path / f"mask_{i:04d}.png")
    ds = dataset.load_views(tmp_path)
    assert len(ds) == 13
    assert ds.train_indices == g["train"].tolist() and ds.holdout_indices == g["holdout"].tolist()
    np.testing.assert_array_equal(ds.load_rgb(3), g["rgb"][3] / 255.0)
    os.remove(tmp_path / "mask_0004.png")
    with pytest.raises(FileNotFoundError):
        dataset.load_views(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("as_path", [False, True])
def test_make_views_gpu_matches_reference_files(gmr, tmp_path, as_path):
    from paper_2602_14493_b200 import dataset
    c, m = _case()
    g = gc.load("views_ico320_13")
    src = m
    if as_path:
        src = tmp_path / "in.ply"
        gmesh.save_mesh(m, src)
    out = tmp_path / "ds"
    ds = dataset.make_views(src, n_views=c["n_views"], resolution=c["resolution"], radius=c["radius"],
                            out_dir=out, background=c["background"])
    rgb = np.array([np.asarray(__import__("PIL.Image").Image.open(p)) for p in ds.rgb_paths])
    mask = np.array([np.asarray(__import__("PIL.Image").Image.open(p)) for p in ds.mask_paths])
    np.testing.assert_array_equal(rgb, g["rgb"])
    np.testing.assert_array_equal(mask, g["mask"])
    names = sorted(n for n in os.listdir(out) if n != "in.ply")
    assert names == g["names"].tolist()
    sha = [hashlib.sha256((out / n).read_bytes()).hexdigest() for n in names]
    assert sha == g["sha"].tolist()


@pytest.mark.gpu
def test_render_view_images_batched_f32(gmr):
    """float32 fast path, many views in one call: every view equals a
    single-view call (no cross-view interaction in the batched binning)."""
    from paper_2602_14493_b200 import dataset
    m = gmr.make_geodesic_sphere(20, seed=1)
    cams = gcam.hemisphere_cameras(40, 3.0, (96, 80))
    rgb, a = dataset.render_view_images(m, cams, (0.1, 0.1, 0.1), np.float32)
    for i in (0, 17, 39):
        r1, a1 = dataset.render_view_images(m, [cams[i]], (0.1, 0.1, 0.1), np.float32)
        np.testing.assert_array_equal(rgb[i], r1[0])
        np.testing.assert_array_equal(a[i], a1[0])
