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
    from paper_2602_14493_b200 import dataset
    c, m = _case()
    g = gc.load("views_ico320_13")
    nm, _ = gmesh.normalize_mesh(m)
    cams = gcam.hemisphere_cameras(c["n_views"], c["radius"], c["resolution"])
    gcam.save_cameras(cams, tmp_path / "cameras.txt")
    dataset._write_ply_ascii(nm, tmp_path / "target_mesh.ply")
    assert (tmp_path / "cameras.txt").read_text() == str(g["cameras_txt"])
    assert (tmp_path / "target_mesh.ply").read_text() == str(g["ply_txt"])
    dataset._write_metadata(tmp_path / "metadata.txt",
                            {"n_views": c["n_views"], "width": 64, "height": 48, "radius": 3.0, "up": "z",
                             "seed": 0, "version": dataset.VERSION})
    assert (tmp_path / "metadata.txt").read_text() == str(g["metadata_txt"])


def test_make_views_takes_a_mesh(tmp_path):
    from paper_2602_14493_b200 import dataset
    with pytest.raises(TypeError):
        dataset.make_views(str(tmp_path / "in.ply"), n_views=2, out_dir=tmp_path / "ds")


@pytest.mark.gpu
def test_make_views_gpu_matches_reference_files(gmr, tmp_path):
    from paper_2602_14493_b200 import dataset
    c, m = _case()
    g = gc.load("views_ico320_13")
    out = tmp_path / "ds"
    ds = dataset.make_views(m, n_views=c["n_views"], resolution=c["resolution"], radius=c["radius"],
                            out_dir=out, background=c["background"])
    rgb = np.array([np.asarray(__import__("PIL.Image").Image.open(p)) for p in ds.rgb_paths])
    mask = np.array([np.asarray(__import__("PIL.Image").Image.open(p)) for p in ds.mask_paths])
    np.testing.assert_array_equal(rgb, g["rgb"])
    np.testing.assert_array_equal(mask, g["mask"])
    names = sorted(os.listdir(out))
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
