"""Generate golden fixtures by running the REAL reference (meshsplat).

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box never needs /root/reference: tests
read these committed fixtures.  Inputs are regenerated deterministically by
`golden_cases.py` (shared with the tests), so only outputs are stored.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("GMR_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, HERE)
sys.dont_write_bytecode = True

import meshsplat as ms  # noqa: E402  (the reference)
from meshsplat.render import Splat2D, _RasterPlan, rasterize_backward  # noqa: E402

import golden_cases as gc  # noqa: E402


def ref_mesh(case):
    return ms.TriangleMesh(case["vertices"], case["facets"], case["colors"])


def ref_cam(c):
    return ms.Camera(rotation=c.rotation, translation=c.translation, fx=c.fx, fy=c.fy,
                     cx=c.cx, cy=c.cy, width=c.width, height=c.height, near=c.near, far=c.far)


def render_case(name, case, dtypes=(np.float64, np.float32)):
    mesh = ref_mesh(case)
    cam = ref_cam(case["camera"])
    out = {}
    for dt in dtypes:
        tag = "f64" if dt == np.float64 else "f32"
        o, ctx = ms.render_mesh(mesh, cam, background=case["background"], dtype=dt, return_ctx=True)
        gv, gcol = ms.render_backward(ctx, case["g_rgb"], case["g_alpha"])
        plan = _RasterPlan(ctx.batch, cam.width, cam.height)
        out[f"{tag}_rgb"] = o.rgb
        out[f"{tag}_alpha"] = o.alpha
        out[f"{tag}_grad_v"] = gv
        out[f"{tag}_grad_c"] = gcol
        out[f"{tag}_source"] = ctx.batch.source
        out[f"{tag}_mean2d"] = ctx.batch.mean2d
        out[f"{tag}_radius"] = ctx.batch.radius
        out[f"{tag}_depth"] = ctx.batch.depth
        out[f"{tag}_entry_source"] = ctx.batch.source[plan.entry_splat]
        out[f"{tag}_bounds"] = plan.bounds
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: v.shape for k, v in out.items()})


def splat_case(name, case):
    cam = ref_cam(case["camera"])
    sp = [Splat2D(mean2d=m, cov2d_screen=c, depth=float(d), color=col, opacity=float(o), source=int(s))
          for m, c, d, col, o, s in zip(case["mean2d"], case["cov2d"], case["depth"],
                                         case["color"], case["opacity"], case["source"])]
    o = ms.rasterize(sp, cam, case["background"])
    gm, gcv, gcol, gop = rasterize_backward(sp, cam, o, case["g_rgb"], case["g_alpha"])
    out = dict(rgb=o.rgb, alpha=o.alpha, g_mean2d=gm, g_cov2d=gcv, g_color=gcol, g_opacity=gop)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: v.shape for k, v in out.items()})


def loss_case(name, case):
    mesh = ref_mesh(case)
    cams = [ref_cam(c) for c in case["cameras"]]
    w = ms.LossWeights(color=1.0, silhouette=1.0, edge=0.0, laplacian=0.0)
    rep, gv, gcol = ms.total_loss(mesh, cams, case["target_rgb"], case["target_mask"],
                                  weights=w, background=case["background"], dtype=np.float64)
    out = dict(color=rep.color, silhouette=rep.silhouette, grad_v=gv, grad_c=gcol)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: np.shape(v) for k, v in out.items()})


def convert_case(name, case):
    mesh = ref_mesh(case)
    cloud = ms.convert_mesh(mesh)
    gv, gcol = ms.convert_backward(mesh, cloud, case["g_means"], case["g_cov3d"], case["g_colors"])
    out = dict(means=cloud.means, cov3d=cloud.cov3d, colors=cloud.colors,
               degenerate=cloud.degenerate, grad_v=gv, grad_c=gcol)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: v.shape for k, v in out.items()})


def fit_case(name, iterations=200):
    """Config 5: icosphere(1280) -> normalised 4x4 grid cube, 20 views 64^2,
    FitConfig(iterations=200, batch_size=1, lr_positions=1e-2, seed=0)
    (reference tests/test_acceptance.py:57-93)."""
    from meshsplat.optim import FitConfig, fit
    case = gc.fit_case()
    target = ref_mesh(case["target"])
    cams = [ref_cam(c) for c in case["cameras"]]
    views = [ms.render_mesh(target, c, dtype=np.float64) for c in cams]
    init = ref_mesh(case["init"])
    cfg = FitConfig(iterations=iterations, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    res = fit(init, cams, [v.rgb for v in views], [v.alpha for v in views], cfg)
    hist = np.array([[h["total"], h["color"], h["silhouette"], h["edge"], h["laplacian"]] for h in res.history])
    # the same loop rendered in float64: the reference's own precision spread
    cfg64 = FitConfig(iterations=iterations, batch_size=1, seed=0, log_every=0, lr_positions=1e-2,
                      dtype="float64")
    res64 = fit(init, cams, [v.rgb for v in views], [v.alpha for v in views], cfg64)
    hist64 = np.array([h["total"] for h in res64.history])
    out = dict(history=hist, history_f64=hist64, final_vertices=res.mesh.vertices, final_colors=res.mesh.colors,
               target_rgb=np.array([v.rgb for v in views]), target_mask=np.array([v.alpha for v in views]),
               wall_time=res.wall_time)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, hist[0], hist[-1], res.wall_time)


def views_case(name):
    """make_views (dataset.py:118-164) into a temp dir: the decoded 8-bit
    images, the SHA-256 of every written file, and the text files."""
    import hashlib
    import tempfile
    c = gc.views_case()
    with tempfile.TemporaryDirectory() as d:
        ds = ms.make_views(ms.TriangleMesh(c["vertices"], c["facets"], c["colors"]), n_views=c["n_views"],
                           resolution=c["resolution"], radius=c["radius"], out_dir=d,
                           background=c["background"])
        from PIL import Image
        rgb = np.array([np.asarray(Image.open(p)) for p in ds.rgb_paths])
        mask = np.array([np.asarray(Image.open(p)) for p in ds.mask_paths])
        names = sorted(os.listdir(d))
        sha = np.array([hashlib.sha256(open(os.path.join(d, n), "rb").read()).hexdigest() for n in names])
        cams = open(os.path.join(d, "cameras.txt")).read()
        meta = open(os.path.join(d, "metadata.txt")).read()
        ply = open(os.path.join(d, "target_mesh.ply")).read()
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), rgb=rgb, mask=mask, names=np.array(names), sha=sha,
                        cameras_txt=np.array(cams), metadata_txt=np.array(meta), ply_txt=np.array(ply),
                        train=np.array(ds.train_indices), holdout=np.array(ds.holdout_indices))
    print(name, rgb.shape, mask.shape, len(names))


def eval_case(name):
    """export_gaussians (convert.py:497-532), sample_surface (mesh.py:580-622),
    chamfer_distance / normal_consistency (metrics.py:40-86), psnr / ssim /
    image_metrics (metrics.py:89-172)."""
    import tempfile
    from meshsplat import metrics as mt
    from meshsplat.mesh import sample_surface
    c = gc.eval_case()
    gt = ms.TriangleMesh(c["gt_vertices"], c["gt_facets"])
    pred = ms.TriangleMesh(c["pred_vertices"], c["pred_facets"], c["pred_colors"])
    n = c["n_samples"]
    out = {}
    sp, sn = sample_surface(pred, 70000, seed=3)   # two 2^16-sample chunks
    sel = np.r_[0:100, 65500:65600, 69900:70000]
    out["samples_sel"], out["snormals_sel"] = sp[sel], sn[sel]
    out["samples_sum"] = np.array([sp.sum(), (sp * sp).sum(), sn.sum()])
    out["cd"] = mt.chamfer_distance(pred, gt, n_samples=n, seed=0)
    out["nc"] = mt.normal_consistency(pred, gt, n_samples=n, seed=0)
    out["cd_fixed"] = mt.chamfer_distance(pred, gt, n_samples=n, seed=2, gt_seed=5)
    out["nc_fixed"] = mt.normal_consistency(pred, gt, n_samples=n, seed=2, gt_seed=5)
    out["cd_self"] = mt.chamfer_distance(gt, gt, n_samples=n, seed=4, gt_seed=4)
    for i, (a, b) in enumerate(c["images"]):
        out[f"psnr{i}"] = mt.psnr(a, b)
        out[f"ssim{i}"] = mt.ssim(a, b)
    out["psnr_same"] = mt.psnr(c["images"][0][0], c["images"][0][0])
    pv, sv = mt.image_metrics([c["images"][0][0], c["images"][2][0]], [c["images"][0][1], c["images"][2][1]])
    out["im_psnr"], out["im_ssim"] = np.array(pv), np.array(sv)
    cloud = ms.convert_mesh(pred)
    with tempfile.TemporaryDirectory() as d:
        ms.export_gaussians(cloud, os.path.join(d, "g.ply"))
        out["export_bytes"] = np.frombuffer(open(os.path.join(d, "g.ply"), "rb").read(), np.uint8)
    out["cloud_cov3d"] = cloud.cov3d
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: (np.shape(v) if np.ndim(v) else float(v)) for k, v in out.items()})


def fit_prefix_case(name, iterations=5):
    """Config 5 cut to a few iterations (the cosine schedule is over
    `iterations`, so this is its own run): history, vertices and colours for
    a tight short-horizon parity check before the trajectory turns chaotic."""
    from meshsplat.optim import FitConfig, fit
    case = gc.fit_case()
    target = ref_mesh(case["target"])
    cams = [ref_cam(c) for c in case["cameras"]]
    views = [ms.render_mesh(target, c, dtype=np.float64) for c in cams]
    init = ref_mesh(case["init"])
    cfg = FitConfig(iterations=iterations, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    res = fit(init, cams, [v.rgb for v in views], [v.alpha for v in views], cfg)
    hist = np.array([[h["total"], h["color"], h["silhouette"], h["edge"], h["laplacian"]] for h in res.history])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), history=hist, vertices=res.mesh.vertices,
                        colors=res.mesh.colors)
    print(name, hist[:, 0])


def fullsize_case(name):
    """Config 3, one view, through the reference in float64 and float32
    (~70 s of CPU): random-projection sketches of the float64 outputs (the
    GPU test pins its own float64 path to them) and the reference's own
    float32-vs-float64 spread (the GPU test bounds its float32 spread by it)."""
    case = gc.fullsize_case()
    mesh = ref_mesh(case)
    cam = ref_cam(case["camera"])
    res = {}
    for dt in (np.float64, np.float32):
        o, ctx = ms.render_mesh(mesh, cam, background=case["background"], dtype=dt, return_ctx=True)
        gv, gcol = ms.render_backward(ctx, case["g_rgb"].astype(dt), case["g_alpha"].astype(dt))
        res[dt] = [np.asarray(a, dtype=np.float64) for a in (o.rgb, o.alpha, gv, gcol)]
    (r64, a64, gv64, gc64), (r32, a32, gv32, gc32) = res[np.float64], res[np.float32]
    out = {f"sketch_{n}": gc.sketch(a, i) for i, (n, a) in enumerate(zip(("rgb", "alpha", "gv", "gc"), res[np.float64]))}
    out.update({f"ref32_{k}": v for k, v in gc.flip_stats(r32, a32, r64, a64, gv32, gv64, gc32, gc64).items()})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: (v if np.ndim(v) == 0 else v.shape) for k, v in out.items()})


def fullsize_f32_case(name):
    """Config 3 view 0 through the reference in float32 only, stored so the
    GPU float32 path can be compared with it DIRECTLY (SURVEY 8c contract):
    the image and alpha quantised to 1/65535 (uint16), both gradients at a
    seeded 10 % vertex subset exactly plus 64-row sketches of the full
    vectors, and the reference's float32 tile lists (face ids in (tile,
    depth, source) order + bounds) to count differing entries."""
    case = gc.fullsize_case()
    mesh = ref_mesh(case)
    cam = ref_cam(case["camera"])
    dt = np.float32
    o, ctx = ms.render_mesh(mesh, cam, background=case["background"], dtype=dt, return_ctx=True)
    gv, gcol = ms.render_backward(ctx, case["g_rgb"].astype(dt), case["g_alpha"].astype(dt))
    plan = _RasterPlan(ctx.batch, cam.width, cam.height)
    sub = gc.vertex_subset(len(case["vertices"]))
    out = dict(rgb_u16=gc.quantize_unit(o.rgb), alpha_u16=gc.quantize_unit(o.alpha),
               gv_sub=np.asarray(gv, np.float32)[sub], gc_sub=np.asarray(gcol, np.float32)[sub],
               gv_sketch=gc.wide_sketch(gv, 100), gc_sketch=gc.wide_sketch(gcol, 101),
               entry_face=ctx.batch.source[plan.entry_splat].astype(np.int32),
               bounds=np.asarray(plan.bounds, np.int32))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: v.shape for k, v in out.items()})


def c2_case(name):
    """Config 2 (8 views 512^2, 81,920 F) through the reference, float64 and
    float32: per-view sketches of the images, sketches of the view-summed
    vertex gradients (the losses.py:151-162 loop with unit weights), and the
    reference's own float32-vs-float64 spread."""
    case = gc.c2_case()
    mesh = ref_mesh(case)
    res = {}
    for dt in (np.float64, np.float32):
        rgbs, alphas, gv_sum, gc_sum = [], [], 0.0, 0.0
        for v, c in enumerate(case["cameras"]):
            cam = ref_cam(c)
            o, ctx = ms.render_mesh(mesh, cam, background=case["background"], dtype=dt, return_ctx=True)
            gv, gcol = ms.render_backward(ctx, case["g_rgb"][v].astype(dt), case["g_alpha"][v].astype(dt))
            rgbs.append(np.asarray(o.rgb, np.float64))
            alphas.append(np.asarray(o.alpha, np.float64))
            gv_sum = gv_sum + np.asarray(gv, np.float64)
            gc_sum = gc_sum + np.asarray(gcol, np.float64)
        res[dt] = (np.array(rgbs), np.array(alphas), gv_sum, gc_sum)
    out = {}
    for tag, dt in (("f64", np.float64), ("f32", np.float32)):
        r, a, gv, gcol = res[dt]
        out[f"{tag}_rgb"] = np.array([gc.wide_sketch(x, 200 + i) for i, x in enumerate(r)])
        out[f"{tag}_alpha"] = np.array([gc.wide_sketch(x, 300 + i) for i, x in enumerate(a)])
        out[f"{tag}_gv"] = gc.wide_sketch(gv, 400)
        out[f"{tag}_gc"] = gc.wide_sketch(gcol, 401)
    r64, a64, gv64, gc64 = res[np.float64]
    r32, a32, gv32, gc32 = res[np.float32]
    out.update({f"ref32_{k}": v for k, v in gc.flip_stats(r32, a32, r64, a64, gv32, gv64, gc32, gc64).items()})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: (v if np.ndim(v) == 0 else v.shape) for k, v in out.items()})


def c4_case(name):
    """Config 4 cut to one view (1,997,120 F, 1024^2) through the reference
    in float64: sketches of image, alpha and both gradients."""
    case = gc.c4_case()
    mesh = ref_mesh(case)
    cam = ref_cam(case["camera"])
    o, ctx = ms.render_mesh(mesh, cam, background=case["background"], dtype=np.float64, return_ctx=True)
    gv, gcol = ms.render_backward(ctx, case["g_rgb"], case["g_alpha"])
    out = {f"sketch_{n}": gc.sketch(a, i) for i, (n, a) in enumerate(zip(("rgb", "alpha", "gv", "gc"),
                                                                          (o.rgb, o.alpha, gv, gcol)))}
    out["entries"] = np.int64(len(_RasterPlan(ctx.batch, cam.width, cam.height).entry_splat))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    # --only: just the large cases named by their flags
    if "--only" not in sys.argv:
        render_case("c1_icosphere1280_128", gc.c1_case())
        render_case("octahedron_32", gc.octahedron_case())
        render_case("icosphere320_64x48", gc.small_render_case())
        splat_case("splats7_32", gc.splat_case())
        splat_case("splats_closed_form_32", gc.closed_form_splat_case())
        loss_case("loss_octa_3views_16", gc.loss_case())
        convert_case("convert_random50", gc.convert_case())
        views_case("views_ico320_13")
        eval_case("eval_ico320")
    if "--fullsize" in sys.argv:
        fullsize_case("fullsize_c3_view0")
    if "--fullsize-f32" in sys.argv:
        fullsize_f32_case("fullsize_c3_view0_f32")
    if "--c2" in sys.argv:
        c2_case("c2_8views_512")
    if "--c4" in sys.argv:
        c4_case("c4_view0_1024")
    if "--fit" in sys.argv:
        fit_case("fit_c5_200")
        fit_prefix_case("fit_c5_5", 5)
