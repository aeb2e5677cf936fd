"""Deterministic inputs of the golden fixtures (shared by make_golden.py,
which feeds them to the real reference, and by the tests, which feed them to
the oracle and to the CUDA path).  Pure numpy + the product's own container
types; nothing here reads /root/reference."""

from __future__ import annotations

import os
import sys

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2602_14493_b200.camera import Camera, default_intrinsics, look_at  # noqa: E402
from paper_2602_14493_b200.mesh import make_icosphere  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    with np.load(os.path.join(HERE, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def identity_camera(width=32, height=32, f=40.0):
    """reference tests/test_render.py:26-31."""
    return Camera(rotation=np.eye(3), translation=np.zeros(3), fx=f, fy=f,
                  cx=(width - 1) / 2, cy=(height - 1) / 2, width=width, height=height)


def octahedron_mesh():
    """reference tests/test_render.py:34-44."""
    v = np.array([(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)], float)
    f = np.array([(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4),
                  (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)])
    col = np.random.default_rng(0).random((6, 3)) * 0.8 + 0.1
    return v, f, col


def _grads(rng, h, w):
    return rng.normal(size=(h, w, 3)), rng.normal(size=(h, w))


def c1_case():
    """Config 1: icosphere L3 (1,280 F), 128^2, camera of BASELINE.md §2."""
    m = make_icosphere(1280)
    col = np.random.default_rng(0).uniform(0.1, 0.9, size=(m.num_vertices, 3))
    cam = look_at((0.3, -2.4, 1.6), (0, 0, 0), **default_intrinsics(128, 128))
    g_rgb, g_a = _grads(np.random.default_rng(0), 128, 128)
    return dict(vertices=np.asarray(m.vertices), facets=np.asarray(m.facets), colors=col,
                camera=cam, background=np.array([0.1, 0.1, 0.1]), g_rgb=g_rgb, g_alpha=g_a)


def octahedron_case():
    """reference tests/test_render.py:442-450."""
    v, f, col = octahedron_mesh()
    cam = look_at((1.7, -2.2, 1.4), (0, 0, 0), **default_intrinsics(32, 32))
    g_rgb, g_a = _grads(np.random.default_rng(7), 32, 32)
    return dict(vertices=v, facets=f, colors=col, camera=cam,
                background=np.array([0.1, 0.1, 0.1]), g_rgb=g_rgb, g_alpha=g_a)


def small_render_case():
    """Non-square image with a partial tile row (reference test_render.py:236-243 camera)."""
    m = make_icosphere(320)
    col = np.random.default_rng(3).uniform(0.1, 0.9, size=(m.num_vertices, 3))
    cam = look_at((0.5, -2.5, 1.5), (0, 0, 0), **default_intrinsics(64, 48))
    g_rgb, g_a = _grads(np.random.default_rng(11), 48, 64)
    return dict(vertices=np.asarray(m.vertices), facets=np.asarray(m.facets), colors=col,
                camera=cam, background=np.array([0.2, 0.3, 0.4]), g_rgb=g_rgb, g_alpha=g_a)


def splat_case():
    """Seven random splats (reference test_render.py:326-349 generator)."""
    rng = np.random.default_rng(5)
    bg = rng.random(3)
    mean2d, cov2d, depth, color, opacity = [], [], [], [], []
    for _ in range(7):
        a = rng.normal(size=(2, 2))
        cov2d.append(a @ a.T + 1.5 * np.eye(2))
        mean2d.append(rng.uniform(6, 26, size=2))
        depth.append(float(rng.uniform(1, 5)))
        color.append(rng.random(3))
        opacity.append(float(rng.uniform(0.25, 0.65)))
    g_rgb, g_a = rng.normal(size=(32, 32, 3)), rng.normal(size=(32, 32))
    return dict(camera=identity_camera(), background=bg, mean2d=np.array(mean2d),
                cov2d=np.array(cov2d), depth=np.array(depth), color=np.array(color),
                opacity=np.array(opacity), source=np.arange(7), g_rgb=g_rgb, g_alpha=g_a)


def closed_form_splat_case():
    """Opaque red over blue at a pixel centre, a depth tie, a clamp pixel and
    a faint splat (reference test_render.py:173-199)."""
    mean2d = np.array([(16, 16), (16, 16), (5, 5), (5, 5), (26, 8), (8, 26)], float)
    cov2d = np.array([np.eye(2) * 2.0] * 6)
    depth = np.array([2.0, 1.0, 1.0, 1.0, 3.0, 1.5])
    color = np.array([(0, 0, 1), (1, 0, 0), (1, 0, 0), (0, 0, 1), (1, 1, 1), (0.2, 0.9, 0.4)], float)
    opacity = np.array([1.0, 1.0, 0.7, 0.7, 1.0, 0.005])
    rng = np.random.default_rng(12)
    return dict(camera=identity_camera(), background=np.array([0.0, 0.0, 0.0]), mean2d=mean2d,
                cov2d=cov2d, depth=depth, color=color, opacity=opacity, source=np.arange(6),
                g_rgb=rng.normal(size=(32, 32, 3)), g_alpha=rng.normal(size=(32, 32)))


def loss_case():
    """total_loss batch (reference test_losses.py:158-170 style), 3 views 16^2."""
    v, f, col = octahedron_mesh()
    rng = np.random.default_rng(4)
    cams, rgbs, masks = [], [], []
    for _ in range(3):
        p = rng.normal(size=3)
        cams.append(look_at(p / np.linalg.norm(p) * 2.6, (0, 0, 0), **default_intrinsics(16, 16)))
        rgbs.append(rng.random((16, 16, 3)))
        masks.append((rng.random((16, 16)) > 0.4).astype(float))
    return dict(vertices=v, facets=f, colors=col, cameras=cams, target_rgb=rgbs,
                target_mask=masks, background=np.array([0.1, 0.1, 0.1]))


def convert_case():
    """50 random facets plus a degenerate and a clamped-kappa facet
    (reference test_convert.py:360-417)."""
    rng = np.random.default_rng(42)
    v = rng.normal(size=(150, 3))
    f = np.arange(150).reshape(50, 3)
    v[3:6] = [(0, 0, 0), (1, 0, 0), (2, 0, 0)]                  # collinear -> degenerate
    v[6:9] = rng.normal(size=(3, 3)) * 1e-3                      # area ~1e-6 -> clamped
    col = rng.random((150, 3))
    return dict(vertices=v, facets=f, colors=col, g_means=rng.normal(size=(50, 3)),
                g_cov3d=rng.normal(size=(50, 3, 3)), g_colors=rng.normal(size=(50, 3)))


def _mesh_dict(m):
    return dict(vertices=np.asarray(m.vertices), facets=np.asarray(m.facets), colors=np.asarray(m.colors))


def fit_case():
    """Config 5 inputs (reference tests/test_acceptance.py:57-93)."""
    from paper_2602_14493_b200.camera import sphere_views
    from paper_2602_14493_b200.mesh import TriangleMesh, make_grid_cube_normalized
    target = make_grid_cube_normalized(4)
    init = make_icosphere(1280)
    return dict(target=_mesh_dict(target), init=_mesh_dict(init), cameras=sphere_views(20, 3.0, 64))


def views_case():
    """SURVEY §8f row 3 (make_views, dataset.py:118-164): a seeded-colour
    icosphere(320) stretched off-centre (so normalize_mesh does work), 13
    hemisphere views at 64x48 on a non-black background (13 > HOLDOUT_STRIDE:
    two hold-out views)."""
    m = make_icosphere(320)
    v = m.vertices * np.array([1.3, 0.8, 1.0]) + np.array([0.2, -0.1, 0.05])
    col = np.random.default_rng(7).random((len(v), 3)) * 0.8 + 0.1
    return dict(vertices=v, facets=m.facets, colors=col, n_views=13, resolution=(64, 48),
                radius=3.0, background=(0.1, 0.2, 0.3))


def eval_case():
    """a target icosphere(320) and a prediction with seeded
    vertex noise and one collapsed (degenerate) facet; image pairs of three
    shapes for PSNR / SSIM."""
    gt = make_icosphere(320)
    rng = np.random.default_rng(11)
    pv = gt.vertices + 0.02 * rng.standard_normal(gt.vertices.shape)
    pf = np.array(gt.facets)
    pv[pf[7, 2]] = 0.5 * (pv[pf[7, 0]] + pv[pf[7, 1]])   # facet 7 becomes degenerate
    col = rng.random((len(pv), 3)) * 0.8 + 0.1
    imgs = []
    for shape in ((32, 24, 3), (17, 40), (64, 48, 3)):
        a = rng.random(shape)
        b = np.clip(a + 0.05 * rng.standard_normal(shape), 0, 1)
        imgs.append((a, b))
    return dict(gt_vertices=gt.vertices, gt_facets=gt.facets, pred_vertices=pv, pred_facets=pf, pred_colors=col,
                n_samples=3000, images=imgs)


def fullsize_case():
    """Config 3 cut to one view (BASELINE configs[3]: geodesic sphere of
    frequency 158 = 499,280 facets, 800x800): the scene, background and a
    seeded upstream gradient for the full-size parity sketch."""
    from paper_2602_14493_b200.camera import hemisphere_cameras
    from paper_2602_14493_b200.mesh import make_geodesic_sphere
    mesh = make_geodesic_sphere(158, seed=0)
    cam = hemisphere_cameras(1, 3.0, (800, 800))[0]
    rng = np.random.default_rng(11)
    return dict(vertices=mesh.vertices, facets=mesh.facets, colors=mesh.colors, camera=cam,
                background=(0.1, 0.1, 0.1), g_rgb=rng.standard_normal((800, 800, 3)),
                g_alpha=rng.standard_normal((800, 800)))


SKETCH_ROWS = 16


def sketch(x, seed):
    """A seeded Gaussian random projection (SKETCH_ROWS x x.size) of a
    flattened float64 array.  ||sketch(a) - sketch(b)|| / ||sketch(b)||
    estimates the relative L2 distance of a and b (Johnson-Lindenstrauss, a
    few tens of percent at 16 rows), so a few KB stand in for a 36 MB
    fixture.  Generated row by row to bound memory."""
    x = np.asarray(x, dtype=np.float64).ravel()
    rng = np.random.default_rng(seed)
    return np.array([rng.standard_normal(x.size) @ x for _ in range(SKETCH_ROWS)])


def flip_stats(rgb_a, alpha_a, rgb_b, alpha_b, gv_a, gv_b, gc_a, gc_b):
    """Precision-spread summary of two renders of one scene: pixels whose
    colour or alpha differ by more than 1e-4 (decision flips), the covered
    pixel count, and the global relative L2 of both gradients."""
    d = np.maximum(np.abs(rgb_a - rgb_b).max(-1), np.abs(alpha_a - alpha_b))
    rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
    return dict(flips=int((d > 1e-4).sum()), covered=int((alpha_b > 0).sum()),
                rel_gv=rel(gv_a, gv_b), rel_gc=rel(gc_a, gc_b))


WIDE_SKETCH_ROWS = 64


def wide_sketch(x, seed):
    """`sketch` with WIDE_SKETCH_ROWS rows (relative-L2 estimates to ~15 %)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    rng = np.random.default_rng(seed)
    return np.array([rng.standard_normal(x.size) @ x for _ in range(WIDE_SKETCH_ROWS)])


def quantize_unit(x):
    """[0, 1] image -> uint16 steps of 1/65535 (max error 7.7e-6, far inside
    the 1e-4 image tolerance; background regions compress to nothing)."""
    return np.round(np.clip(np.asarray(x, np.float64), 0.0, 1.0) * 65535.0).astype(np.uint16)


def vertex_subset(num_vertices, frac=0.1, seed=5):
    """A seeded sorted subset of vertex ids stored exactly in full-size fixtures."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(num_vertices, size=max(1, int(frac * num_vertices)), replace=False))


def c2_case():
    """Config 2: icosphere L6 (81,920 F), 8 hemisphere views 512x512
    (SURVEY 8d), seeded colours, N(0,1) upstream grads per view (seed 21);
    the reference's view loop (losses.py:151-162) sums the per-view grads."""
    from paper_2602_14493_b200.camera import hemisphere_cameras
    m = make_icosphere(81920)
    col = np.random.default_rng(0).uniform(0.1, 0.9, size=(m.num_vertices, 3))
    cams = hemisphere_cameras(8, 3.0, (512, 512))
    rng = np.random.default_rng(21)
    return dict(vertices=np.asarray(m.vertices), facets=np.asarray(m.facets), colors=col, cameras=cams,
                background=(0.1, 0.1, 0.1), g_rgb=rng.standard_normal((8, 512, 512, 3)),
                g_alpha=rng.standard_normal((8, 512, 512)))


def c4_case():
    """Config 4 cut to one view: geodesic sphere n=316 (1,997,120 F), 1024x1024,
    the first full-sphere Fibonacci camera of 64 (test_acceptance.py:61-67)."""
    from paper_2602_14493_b200.camera import sphere_views
    from paper_2602_14493_b200.mesh import make_geodesic_sphere
    mesh = make_geodesic_sphere(316, seed=0)
    cam = sphere_views(64, 3.0, 1024)[0]
    rng = np.random.default_rng(31)
    return dict(vertices=mesh.vertices, facets=mesh.facets, colors=mesh.colors, camera=cam,
                background=(0.1, 0.1, 0.1), g_rgb=rng.standard_normal((1024, 1024, 3)),
                g_alpha=rng.standard_normal((1024, 1024)))
