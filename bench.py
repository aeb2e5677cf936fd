#!/usr/bin/env python
"""GMR hot-path benchmark: forward+backward views/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl gmr|reference]

A step = forward + backward of one batch of views of the config's mesh
(device-resident inputs), ending with the vertex-gradient sum over the batch
(and, for N > 1 ranks, an NCCL all-reduce of [grad_pos | grad_col]).  Views
are sharded across ranks (weak scaling: `views` per GPU).  `value` = views
of all ranks / max-over-ranks device time.  `e2e` = the same metric through
the public torch API (`render_views` + autograd) with pinned host inputs
copied in and gradients copied out every step.  `roofline` = the dominant
stage's algorithmic bytes per launch / its CUDA-event time (timed live in
the library on the launching stream), against MEASURED_PEAKS.json.

`--impl reference` times the reference algorithm on the host cores (the
pinned numpy restatement in oracle/, one process per core, one view each;
bounded sample, see oracle/cpu_baseline.py).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(mesh=("icosphere", 1280), res=128, views=1,
               desc="config1: icosphere subdiv-3 (1,280 faces), 128x128"),
    "c2": dict(mesh=("icosphere", 81920), res=512, views=8,
               desc="config2: icosphere subdiv-6 (81,920 faces), 512x512"),
    "c3": dict(mesh=("geodesic", 158), res=800, views=8,
               desc="config3: geodesic displaced sphere n=158 (499,280 faces, 249,642 vertices), 800x800"),
    "c3b1": dict(mesh=("geodesic", 158), res=800, views=1,
                 desc="config3 batch 1: geodesic displaced sphere n=158 (499,280 faces), 800x800"),
    "c4": dict(mesh=("geodesic", 316), res=1024, views=8, cams="sphere",
               desc="config4: geodesic displaced sphere n=316 (1,997,120 faces), 1024x1024, full-sphere Fibonacci "
                    "cameras (SURVEY 8d)"),
    # BASELINE configs[3] as stated: 64 views in total, sharded over the ranks
    "c4s": dict(mesh=("geodesic", 316), res=1024, views=64, total_views=True, chunk=16, cams="sphere",
                desc="config4: geodesic displaced sphere n=316 (1,997,120 faces), 1024x1024, full-sphere Fibonacci "
                     "cameras (SURVEY 8d), 64 views in total"),
    "views": dict(mesh=("geodesic", 158), res=256, views=253,
                  desc="SURVEY 8f row 3: make_views of the config-3 mesh (499,280 faces), 253 hemisphere views "
                       "256x256, float64 like the reference, 8-bit images to host"),
    "eval": dict(mesh=("geodesic", 158), res=0, views=0,
                 desc="SURVEY 8f row 4: chamfer_distance + normal_consistency at the reference default "
                      "n_samples=100,000 (both stream assignments), config-3 mesh vs a noisy copy"),
    "c5": dict(mesh=("fit", 1280), res=64, views=1,
               desc="config5: 200-iteration batch-1 inverse-rendering loop, icosphere(1280) -> grid cube, 20 views 64x64"),
}
METRIC = "fwd+bwd views/sec @500K faces 800x800; HBM GB/s vs peak; 1/2/4/8 GPU"
BG = (0.1, 0.1, 0.1)


def build_mesh(cfg):
    import paper_2602_14493_b200 as gmr
    kind, n = cfg["mesh"]
    if kind == "geodesic":
        return gmr.make_geodesic_sphere(n, seed=0)
    m = gmr.make_icosphere(n)
    return gmr.TriangleMesh(m.vertices, m.facets, gmr.seeded_colors(m.num_vertices, 0))


def all_cams(cfg, total):
    import paper_2602_14493_b200 as gmr
    if cfg.get("cams") == "sphere":   # C4: full-sphere Fibonacci lattice (reference test_acceptance.py:61-67)
        from paper_2602_14493_b200.camera import sphere_views
        return sphere_views(total, 3.0, cfg["res"])
    return gmr.hemisphere_cameras(total, 3.0, (cfg["res"], cfg["res"]))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.samples = []
        self.proc = None
        self.window = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(gpu_index), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append((time.time(), parts))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def summary(self):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0, t1 = self.window or (0, 1e30)
        inside = [p for t, p in self.samples if t0 - 0.05 <= t <= t1 + 0.05] or [p for _, p in self.samples[-3:]]
        sm = sorted(float(p[0]) for p in inside if p[0].replace(".", "").isdigit())
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for p in inside for i in range(4) if "Active" in p[2 + i]
                          and "Not" not in p[2 + i]})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(inside[0][1]) if inside[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(inside)}


# Stage groups of the library's CUDA-event timers (lib.STAGES) that SURVEY
# §8(d)'s per-kernel byte model prices as one kernel.
STAGE_GROUPS = {
    "convert_project": ("convert_project",),                          # K1
    "binning": ("depth_sort", "scan_emit", "tile_sort_ranges"),       # K2
    "blend_forward": ("blend_forward",),                              # K3
    "blend_backward": ("blend_backward",),                            # K4
    "face_vertex_backward": ("face_backward", "vertex_gather"),       # K5 + K6
}


def section8d_bytes(F, V, B, W, H, E, T):
    """SURVEY §8(d) compulsory bytes per launch of each stage group (fp32
    values, int32 indices, each logical array crossing a kernel boundary
    once): per view K1 60F+24V, K2 24F+44E+8T, K3 8T+36E+24WH,
    K4 24WH+8T+36E+32F, K5/K6 44F+36V.  E is summed over the B views."""
    WH = W * H
    return {
        "convert_project": B * (60 * F + 24 * V),
        "binning": B * (24 * F + 8 * T) + 44 * E,
        "blend_forward": B * (8 * T + 24 * WH) + 36 * E,
        "blend_backward": B * (24 * WH + 8 * T + 32 * F) + 36 * E,
        "face_vertex_backward": B * (44 * F + 36 * V),
    }


def implementation_bytes(F, V, B, W, H, E, bins, tile_depth_sort=True):
    """What the implementation moves per launch (diagnostic beside the
    §8(d) model: coverage masks, entry partials, double-buffered sorts)."""
    n = F * B
    px = W * H * B
    entry_passes = max(1, (max(1, (bins - 1).bit_length()) + 7) // 8)
    return {
        "convert_project": 12 * F + 24 * V + 16 * F + 52 * n,
        "binning": (12 * E if tile_depth_sort else 80 * n) + (32 if tile_depth_sort else 36) * n + 8 * E
        + 20 * entry_passes * E + 4 * E + 4 * bins,
        "blend_forward": 8 * bins + 52 * E + 20 * px,
        "blend_backward": 8 * bins + 96 * E + 32 * px,
        "face_vertex_backward": 24 * F + 24 * V + 40 * n + 32 * E + 72 * F + 4 * V + 12 * F + 72 * F + 24 * V,
    }


def survey_bytes_per_view(F, V, E_view, T, W, H):
    """SURVEY §8d compulsory bytes of the whole fwd+bwd per view."""
    return 160 * F + 60 * V + 116 * E_view + 24 * T + 48 * W * H


def load_counters(config):
    """ncu counters of the dominant kernels for THIS config (profiles/
    traffic_r02.json, keyed by config name), or None."""
    tf = os.path.join(ROOT, "profiles", "traffic_r02.json")
    try:
        with open(tf) as f:
            return json.load(f).get(config)
    except Exception:
        return None


def static_config(cfg, name, world):
    """The `config` object both arms print (run-independent keys only)."""
    F, V = {("geodesic", 158): (499280, 249642), ("geodesic", 316): (1997120, 998562),
            ("icosphere", 1280): (1280, 642), ("icosphere", 81920): (81920, 40962)}.get(cfg["mesh"], (None, None))
    total = cfg.get("total_views", False)
    per = cfg["views"] // world if total else cfg["views"]
    return {"workload": cfg["desc"] + (f", {cfg['views']} views sharded over the GPUs" if total else
                                       f", {cfg['views']} views per GPU per step (hemisphere cameras r=3)"),
            "name": name, "faces": F, "vertices": V, "views_per_gpu": per, "resolution": [cfg["res"], cfg["res"]],
            "l2": "inputs+workspace per step > 126 MB L2 (no flush needed)",
            "parallelism": f"views sharded over {world} GPU(s), one NCCL all-reduce of vertex grads per step"}


def run_gmr(args, cfg):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2602_14493_b200 as gmr
    from paper_2602_14493_b200 import dist as gdist
    from paper_2602_14493_b200 import engine, lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the multi-rank path (NCCL init, per-step all-reduce, max over ranks);
    # GMR_BENCH_DIST=1 exercises it even with one rank under torchrun
    multi = world > 1 or os.environ.get("GMR_BENCH_DIST") == "1"
    if multi:
        # NCCL's init lines (rank count, transport) go to stderr for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # stdout carries only the JSON line
        dist.init_process_group("nccl", device_id=dev)
    L = lib.load()
    mesh = build_mesh(cfg)
    W = H = cfg["res"]
    if cfg.get("total_views"):   # strong scaling: a fixed set of views split over the ranks
        lo, hi = gdist.shard_range(cfg["views"], rank, world)
        cams = all_cams(cfg, cfg["views"])[lo:hi]
    else:                        # weak scaling: `views` per rank
        cams = all_cams(cfg, cfg["views"] * world)[rank * cfg["views"]:(rank + 1) * cfg["views"]]
    B = len(cams)
    chunk = cfg.get("chunk") or B
    total_views = cfg["views"] if cfg.get("total_views") else cfg["views"] * world
    pos = torch.tensor(np.asarray(mesh.vertices), dtype=torch.float32, device=dev)
    col = torch.tensor(np.asarray(mesh.colors), dtype=torch.float32, device=dev)
    faces = torch.tensor(np.asarray(mesh.facets), dtype=torch.int32, device=dev)
    F, V = faces.shape[0], pos.shape[0]
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    g_rgb = torch.randn((B, H, W, 3), generator=gen, device=dev)
    g_a = torch.randn((B, H, W), generator=gen, device=dev)
    T = ((W + 15) // 16) * ((H + 15) // 16)

    pending = []
    last = {}

    def step(final=False, flags=0, views=None):
        # forward and backward of every chunk enqueued back to back; each
        # forward's status (entry capacity, non-finite splats) is validated
        # one step behind, so the device never drains between steps
        nv = B if views is None else views
        gp = gc = None
        states, reds = [], []
        for c0 in range(0, nv, chunk):
            c1 = min(nv, c0 + chunk)
            rgb, alpha, st = engine.render_forward(pos, col, faces, cams[c0:c1], W, H, BG, flags=flags, check=False)
            a, b = engine.render_backward(st, pos, col, faces, rgb, g_rgb[c0:c1], g_a[c0:c1])
            if multi and nv > chunk:
                # this view group's reduction runs on NCCL's stream while the
                # next group renders
                reds.append(gdist.allreduce_vertex_grads(a, b, async_op=True))
            gp, gc = (a, b) if gp is None else (gp + a, gc + b)
            states.append(st)
        pending.extend(states)
        last["states"] = states
        if reds:
            parts = [r.wait() for r in reds]
            gp, gc = parts[0][0].clone(), parts[0][1].clone()
            for x in parts[1:]:
                gp += x[0]
                gc += x[1]
        elif multi:
            gp, gc, _ = gdist.allreduce_vertex_grads(gp, gc)
        keep = 0 if final else len(states)
        while len(pending) > keep:
            engine.check_status(pending.pop(0))   # raises on overflow / non-finite
        return gp

    def timed(k, **kw):
        """K steps bracketed by barrier + synchronize; device ms (max over ranks)."""
        if multi:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(k):
            step(final=(i == k - 1), **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if multi:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for i in range(args.warmup):
        step(final=(i == args.warmup - 1))
    torch.cuda.synchronize()
    sampler = ClockSampler(local) if rank == 0 else None
    time.sleep(0.3 if sampler else 0)
    n0 = L.gmr_launch_count()
    wall0 = time.time()
    ms = timed(args.steps)
    wall1 = time.time()
    launches = (L.gmr_launch_count() - n0) // args.steps
    st_main = last["states"][0]
    E_step = sum(int(st.entries) for st in last["states"])   # tile entries of one step (all chunks)
    value = total_views * args.steps / (ms / 1e3)

    # per-stage times: the same K steps again with the library's stage
    # timers on (CUDA events on the launching stream around every stage);
    # kept out of the pass above, whose step time is the headline
    L.gmr_timing_enable(1)
    L.gmr_timing_read(None, None, 0, 1)
    for i in range(args.steps):
        step(final=(i == args.steps - 1))
    torch.cuda.synchronize()
    sms = (ctypes.c_double * 8)()
    scnt = (ctypes.c_int64 * 8)()
    L.gmr_timing_read(sms, scnt, 8, 1)
    L.gmr_timing_enable(0)

    # config 3 extras in the same run: the reference's exact tile lists
    # (GMR_FLAG_FULL_TILE_LISTS) and batch 1 (BASELINE configs[2])
    extras = {}
    if args.config == "c3" and not args.no_extras:
        for i in range(2):
            step(final=(i == 1), flags=lib.FLAG_FULL_TILE_LISTS)
        ms_full = timed(args.steps, flags=lib.FLAG_FULL_TILE_LISTS)
        extras["full_tile_lists"] = {
            "value": round(total_views * args.steps / (ms_full / 1e3), 2), "unit": "views/s",
            "ms_per_step": round(ms_full / args.steps, 4),
            "tile_entries_per_step": sum(int(st.entries) for st in last["states"]),
            "note": "GMR_FLAG_FULL_TILE_LISTS: every tile of each splat's 3-sigma rectangle, the reference's "
                    "_RasterPlan lists bit for bit (render.py:214-226); the headline drops tiles a splat's "
                    "alpha >= 1/255 ellipse cannot reach (identical images and gradients)"}
        for i in range(3):
            step(final=(i == 2), views=1)
        ms_b1 = timed(args.steps, views=1)
        extras["batch1"] = {"value": round(world * args.steps / (ms_b1 / 1e3), 2), "unit": "views/s",
                            "ms_per_step": round(ms_b1 / args.steps, 4),
                            "note": "config 3 batch 1: one view per GPU per step (BASELINE configs[2])"}

    # ---- end to end through the public torch API, host buffers -------------
    # Every step uploads its inputs (vertices, colours, upstream image grads)
    # from pinned host memory and reads its vertex/colour grads back.  The
    # copies run on their own streams, double-buffered, so step k+1's upload
    # and step k-1's download overlap step k's kernels (PCIe and the copy
    # engines are otherwise idle while the SMs render).
    pin = lambda t: t.cpu().pin_memory()
    h_pos, h_col, h_g, h_a = pin(pos), pin(col), pin(g_rgb), pin(g_a)
    o_gp = [torch.empty_like(h_pos).pin_memory() for _ in range(2)]
    o_gc = [torch.empty_like(h_col).pin_memory() for _ in range(2)]
    slots = [dict(p=torch.empty_like(pos), c=torch.empty_like(col), g=torch.empty_like(g_rgb),
                  a=torch.empty_like(g_a), up=torch.cuda.Event(), up_g=torch.cuda.Event(),
                  used=torch.cuda.Event(), down=torch.cuda.Event()) for _ in range(2)]
    main, up_s, down_s = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ctr = [0]

    def upload(s):
        with torch.cuda.stream(up_s):
            up_s.wait_event(s["used"])           # the step that last read this slot is done
            s["p"].copy_(h_pos, non_blocking=True)
            s["c"].copy_(h_col, non_blocking=True)
            s["up"].record(up_s)                 # the forward needs only the mesh ...
            s["g"].copy_(h_g, non_blocking=True)
            s["a"].copy_(h_a, non_blocking=True)
            s["up_g"].record(up_s)               # ... the backward the image grads

    def e2e_step(prefetch=True):
        k = ctr[0]
        ctr[0] += 1
        s = slots[k % 2]
        main.wait_event(s["up"])
        p = s["p"].detach().requires_grad_(True)
        c = s["c"].detach().requires_grad_(True)
        reds = []
        for c0 in range(0, B, chunk):
            c1 = min(B, c0 + chunk)
            rgb, alpha = gmr.render_views(p, c, faces, cams[c0:c1], W, H, BG)
            if prefetch and c0 == 0:
                upload(slots[(k + 1) % 2])        # next step's inputs, behind this forward
            main.wait_event(s["up_g"])
            if multi and B > chunk:               # per view group, reduced while the next group renders
                a, b = torch.autograd.grad([rgb, alpha], [p, c], [s["g"][c0:c1], s["a"][c0:c1]])
                reds.append(gdist.allreduce_vertex_grads(a, b, async_op=True))
            else:
                torch.autograd.backward([rgb, alpha], [s["g"][c0:c1], s["a"][c0:c1]])
        if reds:
            parts = [r.wait() for r in reds]
            gp, gc = parts[0][0].clone(), parts[0][1].clone()
            for x in parts[1:]:
                gp += x[0]
                gc += x[1]
        else:
            gp, gc = p.grad, c.grad
            if multi:
                gp, gc, _ = gdist.allreduce_vertex_grads(gp, gc)
        s["used"].record(main)
        with torch.cuda.stream(down_s):
            down_s.wait_event(s["used"])
            o_gp[k % 2].copy_(gp, non_blocking=True)
            o_gc[k % 2].copy_(gc, non_blocking=True)
            gp.record_stream(down_s)
            gc.record_stream(down_s)
            s["down"].record(down_s)

    upload(slots[0])
    for i in range(max(1, args.warmup)):
        e2e_step(prefetch=i < max(1, args.warmup) - 1)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    k_e2e = max(3, args.steps)
    ctr[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    up_s.wait_stream(main)
    upload(slots[0])                              # the first step's upload is timed too
    for i in range(k_e2e):
        e2e_step(prefetch=i < k_e2e - 1)
    main.wait_stream(down_s)                      # ... and the last step's read-back
    e1.record()
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if multi:
        t = torch.tensor([ms_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    h2d = (h_pos.numel() + h_col.numel() + h_g.numel() + h_a.numel()) * 4
    d2h = (o_gp[0].numel() + o_gc[0].numel()) * 4
    if sampler:
        sampler.mark(wall0, wall1)
    clocks = sampler.summary() if sampler else None

    if rank != 0:
        if multi:
            dist.destroy_process_group()
        return None

    # ---- rooflines of the dominant stage -----------------------------------
    peak, peak_src = load_peaks()
    names = lib.STAGES
    per_stage = {nm: sms[i] / args.steps for i, nm in enumerate(names) if scnt[i]}
    tds = bool(st_main.raster.flags & lib.FLAG_TILE_DEPTH_SORT)
    b8d = section8d_bytes(F, V, B, W, H, E_step, T)
    bimp = implementation_bytes(F, V, B, W, H, E_step, T * B, tds)
    stages = {}
    for grp, members in STAGE_GROUPS.items():
        t = sum(per_stage.get(m, 0.0) for m in members)
        if t <= 0:
            continue
        stages[grp] = {"ms_per_step": round(t, 4), "members": {m: round(per_stage[m], 4) for m in members
                                                              if m in per_stage},
                       "GBs_8d": round(b8d[grp] / (t / 1e3) / 1e9, 1),
                       "frac_8d": round(b8d[grp] / (t / 1e3) / 1e9 / peak, 4),
                       "GBs_implementation": round(bimp[grp] / (t / 1e3) / 1e9, 1)}
    dom = max(stages, key=lambda k: stages[k]["ms_per_step"])
    dms = stages[dom]["ms_per_step"] / ((B + chunk - 1) // chunk)   # per launch
    per_launch_8d = b8d[dom] / ((B + chunk - 1) // chunk)
    achieved = per_launch_8d / (dms / 1e3) / 1e9
    step_bytes = survey_bytes_per_view(F, V, E_step / B, T, W, H) * B
    step_gbs = step_bytes / (ms / args.steps / 1e3) / 1e9
    ctr_ = load_counters(args.config) or {}
    kc = ctr_.get(dom) or {}
    traffic = kc.get("dram_bytes")
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    issue = smem = None
    if kc.get("warp_instructions"):
        peak_issue = 148 * 4 * float(mhz) * 1e6
        ach = kc["warp_instructions"] / (dms / 1e3)
        issue = {"bound": "issue", "kernel": dom, "achieved": round(ach / 1e12, 4), "peak": round(peak_issue / 1e12, 4),
                 "unit": "T warp-instr/s", "frac": round(ach / peak_issue, 4),
                 "warp_instructions_per_launch": int(kc["warp_instructions"]),
                 "source": f"ncu smsp__inst_executed.sum, {ctr_.get('source', 'profiles/traffic_r02.json')}"}
    if kc.get("smem_wavefronts"):
        peak_wf = 148 * float(mhz) * 1e6
        ach = kc["smem_wavefronts"] / (dms / 1e3)
        smem = {"bound": "shared-memory pipe", "kernel": dom, "achieved": round(ach / 1e12, 4),
                "peak": round(peak_wf / 1e12, 4), "unit": "T wavefronts/s", "frac": round(ach / peak_wf, 4),
                "wavefronts_per_launch": int(kc["smem_wavefronts"]),
                "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"}

    # ---- CPU baseline (rank 0, N = 1): full unsampled views ---------------
    cpu = None
    if world == 1 and not args.no_cpu:
        from oracle.cpu_baseline import BandWorkers
        wk = BandWorkers(mesh.vertices, mesh.facets, mesh.colors, all_cams(cfg, 8), BG, bands=1)
        wall, per = wk.full_view()
        wk.close()
        cpu = {"value": round(wk.procs / wall, 5), "unit": "views/s", "cores": wk.procs, "kind": wk.impl,
               "sample": (f"{wk.procs} concurrent whole views (one process per host core, OPENBLAS_NUM_THREADS=1), "
                          f"{'the reference meshsplat from baseline/_ref' if wk.impl == 'reference' else 'the pinned numpy port oracle/gmr_oracle.py'}"
                          f": render_mesh(float32) + render_backward, unsampled; {float(np.mean(per)):.1f} s per view, "
                          f"{wall:.1f} s wall")}

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "views/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong" if cfg.get("total_views") else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (procedural mesh, seeded vertex colours, N(0,1) upstream image grads)",
        "config": static_config(cfg, args.config, world),
        "run": {"tile_entries_per_step": E_step, "views_per_call": chunk,
                "depth_order": "per-tile lists (GMR_FLAG_TILE_DEPTH_SORT)" if tds else "global item sort",
                "tile_lists": "unreachable tiles dropped (default)"},
        "e2e": {"value": round(total_views * k_e2e / (ms_e2e / 1e3), 2), "unit": "views/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "paper_2602_14493_b200.render_views + torch.autograd.backward; pinned host buffers, "
                       "uploads/read-backs double-buffered on copy streams"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "bytes_per_launch": int(per_launch_8d),
                     "model": "SURVEY 8(d) per-kernel compulsory bytes (K4: 24WH+8T+36E+32F per view)",
                     "peak_source": peak_src},
        "issue_roofline": issue,
        "smem_roofline": smem,
        "step_roofline": {"bytes_per_step": int(step_bytes), "achieved_GBs": round(step_gbs, 1),
                          "frac": round(step_gbs / peak, 4),
                          "model": "SURVEY 8d: 160F+60V+116E+24T+48WH per view"},
        "stages": stages,
        "stage_timing": "per-stage CUDA events on the launching stream, in a second pass of the same K steps",
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    line.update(extras)
    print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()
    return line


def run_fit(args, cfg):
    """Config 5: the whole 200-iteration loop (device render fwd+bwd per
    iteration, reference optimiser semantics); loss parity vs the reference
    trajectory recorded in tests/golden/fit_c5_200.npz."""
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import golden_cases as gc
    import paper_2602_14493_b200 as gmr
    from paper_2602_14493_b200 import fit as gfit
    case, g = gc.fit_case(), gc.load("fit_c5_200")
    init = gmr.TriangleMesh(case["init"]["vertices"], case["init"]["facets"], case["init"]["colors"])
    rgbs, masks = list(g["target_rgb"]), list(g["target_mask"])
    iters = 200
    cfg5 = gfit.FitConfig(iterations=iters, batch_size=1, seed=0, log_every=0, lr_positions=1e-2)
    for _ in range(max(1, args.warmup)):
        gfit.fit(init, case["cameras"], rgbs, masks, gfit.FitConfig(iterations=5, batch_size=1, seed=0,
                                                                  log_every=0, lr_positions=1e-2))
    torch.cuda.synchronize()
    walls, loops = [], []
    for _ in range(max(1, args.steps // 10)):
        res = gfit.fit(init, case["cameras"], rgbs, masks, cfg5)
        walls.append(res.wall_time)
        loops.append(res.loop_time)
    wall = float(np.median(walls))
    loop = float(np.median(loops))
    final = res.history[-1]["total"]
    ref_final = float(g["history"][-1, 0])
    line = {"metric": "config5 inverse-rendering loop: iterations/s (200 iterations, batch 1, 64x64, end to end)",
            "value": round(iters / wall, 2), "unit": "iterations/s", "n_gpus": 1, "steps": len(walls),
            "warmup": max(1, args.warmup), "ms_per_step": round(1e3 * wall / iters, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference toy task targets)",
            "config": {"workload": cfg["desc"]},
            "e2e": {"value": round(iters / wall, 2), "unit": "iterations/s",
                    "h2d_bytes_per_step": 642 * 6 * 4 + 64 * 64 * 4 * 8, "d2h_bytes_per_step": 642 * 6 * 8 + 16},
            "loop_only": {"ms_per_iteration": round(1e3 * loop / iters, 4),
                          "note": "the 200 iterations alone (dispatch to completion), without the per-call setup"},
            "loss_parity": {"final_total": round(final, 6), "reference_final_total": round(ref_final, 6),
                            "initial_total": round(res.history[0]["total"], 6), "reference_initial_total": 1.405564,
                            "reference_wall_s_build_container": round(float(g["wall_time"]), 2)}}
    print(json.dumps(line), flush=True)
    return line


def run_views(args, cfg):
    """batched forward-only dataset rendering
    (dataset.render_view_images: device render + fused 8-bit quantisation,
    images copied to pinned host memory).  One step = all 253 views."""
    import numpy as np
    import torch
    import paper_2602_14493_b200 as gmr
    from paper_2602_14493_b200 import dataset, lib
    L = lib.load()
    mesh = build_mesh(cfg)
    n, W = cfg["views"], cfg["res"]
    cams = gmr.hemisphere_cameras(n, 3.0, (W, W))
    dt = np.float32 if args.views_f32 else np.float64
    for _ in range(max(1, args.warmup)):
        dataset.render_view_images(mesh, cams, BG, dt)
    torch.cuda.synchronize()
    n0 = L.gmr_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(1, args.steps // 4)
    e0.record()
    for _ in range(steps):
        rgb8, a8 = dataset.render_view_images(mesh, cams, BG, dt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launches = (L.gmr_launch_count() - n0) // steps
    cpu = None
    if not args.no_cpu:
        from oracle import gmr_oracle as orc
        t0 = time.perf_counter()
        orc.render(mesh.vertices, mesh.facets, mesh.colors, cams[0], BG, True, dt)
        sec = time.perf_counter() - t0
        cpu = {"value": round(1.0 / sec, 4), "unit": "views/s", "cores": 1, "kind": "port",
               "sample": f"one view, oracle render (numpy restatement of render_mesh), {sec:.1f} s"}
    line = {"metric": "make_views forward-only views/s (8-bit images to host)", "value": round(n / (ms / 1e3), 1),
            "unit": "views/s", "n_gpus": 1, "steps": steps, "warmup": max(1, args.warmup),
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.views_f32 else "f64", "data": "synthetic (config-3 mesh)",
            "config": {"workload": cfg["desc"], "views": n, "resolution": [W, W]},
            "e2e": {"value": round(n / (ms / 1e3), 1), "unit": "views/s",
                    "h2d_bytes_per_step": int(mesh.vertices.size * 16 + mesh.facets.size * 4),
                    "d2h_bytes_per_step": int(rgb8.nbytes + a8.nbytes)},
            "gpu_launches": int(launches), "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    return line


def run_eval(args, cfg):
    """Chamfer + normal consistency (metrics.py:49-86) at
    100K samples per mesh.  One step = the full metric pair (4 nearest-sample
    query sets of 100K x 100K, exact float64), host sampling included."""
    import numpy as np
    import torch
    import paper_2602_14493_b200 as gmr
    from paper_2602_14493_b200 import lib, metrics
    L = lib.load()
    gt = build_mesh(cfg)
    rng = np.random.default_rng(0)
    pred = gmr.TriangleMesh(gt.vertices + 0.003 * rng.standard_normal(gt.vertices.shape), gt.facets)
    n = 100_000
    for _ in range(max(1, args.warmup)):
        metrics.chamfer_and_normal_consistency(pred, gt, n_samples=n, seed=0)
    torch.cuda.synchronize()
    steps = max(1, args.steps // 4)
    n0 = L.gmr_launch_count()
    t0 = time.perf_counter()
    for _ in range(steps):
        cd, nc = metrics.chamfer_and_normal_consistency(pred, gt, n_samples=n, seed=0)
    wall = (time.perf_counter() - t0) / steps
    launches = (L.gmr_launch_count() - n0) // steps
    # device-only: the four nearest-sample query sets on resident samples
    pa, na = metrics.sample_surface(pred, n, 0)
    pb, nb = metrics.sample_surface(gt, n, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import ctypes
    dev = torch.device("cuda", 0)
    tpa, tna, tpb, tnb = (torch.tensor(x, device=dev) for x in (pa, na, pb, nb))
    sz = ctypes.c_size_t()
    L.gmr_chamfer_scratch_size(n, n, ctypes.byref(sz))
    scr = torch.empty(sz.value, dtype=torch.uint8, device=dev)
    out = torch.empty(4, dtype=torch.float64, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    call = lambda: lib.check(L.gmr_chamfer_nc(tpa.data_ptr(), tna.data_ptr(), n, tpb.data_ptr(), tnb.data_ptr(), n,
                                              out.data_ptr(), scr.data_ptr(), sz.value, st))
    call()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        call()
    e1.record()
    torch.cuda.synchronize()
    pass_ms = e0.elapsed_time(e1) / 4
    pairs = 2.0 * n * n
    cpu = None
    if not args.no_cpu:
        from scipy.spatial import cKDTree
        t0 = time.perf_counter()
        for _ in range(2):
            d1, i1 = cKDTree(pb).query(pa, workers=-1)
            d2, i2 = cKDTree(pa).query(pb, workers=-1)
        sec = (time.perf_counter() - t0) / 2
        cpu = {"value": round(1.0 / (2 * sec), 3), "unit": "metric pairs/s", "cores": os.cpu_count(),
               "kind": "reference",
               "sample": f"the reference's own cKDTree queries (workers=-1) for one stream assignment, "
                         f"{sec:.3f} s, x2 for both assignments; sampling excluded"}
    line = {"metric": "chamfer_distance + normal_consistency pairs/s (100K samples, both stream assignments)",
            "value": round(1.0 / (2 * pass_ms / 1e3), 2), "unit": "metric pairs/s", "n_gpus": 1, "steps": steps,
            "warmup": max(1, args.warmup), "ms_per_step": round(2 * pass_ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-3 mesh + noise)",
            "config": {"workload": cfg["desc"], "n_samples": n, "cd": cd, "nc": nc},
            "e2e": {"value": round(1.0 / wall, 2), "unit": "metric pairs/s",
                    "h2d_bytes_per_step": int(8 * n * 3 * 4 * 2), "d2h_bytes_per_step": 64,
                    "note": "includes the reference-exact numpy sample stream on the host"},
            "roofline": {"bound": "fp64", "achieved": round(pairs / (pass_ms / 1e3) * 8 / 1e12, 2),
                         "unit": "TFLOP/s (8 fp64 ops per pair)", "peak": None, "frac": None, "traffic": None},
            "gpu_launches": int(launches), "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    return line


def run_reference(args, cfg):
    """Reference arm: the reference's own CPU render path (the real meshsplat
    from baseline/_ref when installed, else the pinned numpy port) on all
    host cores, unsampled -- see oracle/cpu_baseline.py.  A step: every
    worker renders the next band (1/bands of its view's tile rows) through
    the reference API; `bands` steps are P whole views.  A calibration pass
    of P whole views (same workers, concurrent) gives the band split's
    overhead, and `value` is the whole-view rate."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    import numpy as np
    from oracle.cpu_baseline import BandWorkers
    mesh = build_mesh(cfg)
    bands = args.ref_bands
    wk = BandWorkers(mesh.vertices, mesh.facets, mesh.colors, all_cams(cfg, 8), BG, bands=bands)
    for i in range(args.warmup):
        wk.step(i)
    wk.band_renders, wk.wall = 0, 0.0
    t0 = time.perf_counter()
    for i in range(args.steps):
        wk.step(args.warmup + i)
    wall = time.perf_counter() - t0
    band_rate = wk.views_per_s()
    full_wall, full_per = (wk.full_view() if not args.ref_no_full else (None, None))
    wk.close()
    value = wk.procs / full_wall if full_wall else band_rate
    ms_per_step = 1e3 * wall / args.steps
    sample = (f"{wk.procs} worker processes (one per host core, OPENBLAS_NUM_THREADS=1), "
              f"{'the reference meshsplat (baseline/_ref)' if wk.impl == 'reference' else 'the pinned numpy port'}"
              f" render_mesh(float32) + render_backward, unsampled; a step = every worker renders one of "
              f"{bands} tile-row bands of its view through a crop camera; value = {wk.procs} concurrent whole "
              f"views / their wall time ({full_wall:.1f} s)" if full_wall else "")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "views/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 1),
        "higher_is_better": True, "scaling": "strong" if cfg.get("total_views") else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (procedural mesh, seeded vertex colours, N(0,1) upstream image grads)",
        "config": static_config(cfg, args.config, world),
        "cpu_baseline": {"value": round(value, 5), "unit": "views/s", "cores": wk.procs, "kind": wk.impl,
                         "sample": sample},
        "band_steps": {"views_per_s": round(band_rate, 5), "wall_s": round(wall, 2), "bands_per_view": bands,
                       "overhead_vs_whole_views": round(value / band_rate, 3) if band_rate else None},
        "whole_view_s": round(float(np.mean(full_per)), 2) if full_per else None,
        "e2e": {"value": round(value, 5), "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="gmr", choices=["gmr", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-extras", action="store_true", help="config 3: skip the full-tile-list and batch-1 lines")
    ap.add_argument("--ref-bands", type=int, default=10, help="reference arm: tile-row bands per view")
    ap.add_argument("--ref-no-full", action="store_true", help="reference arm: skip the whole-view pass")
    ap.add_argument("--views-f32", action="store_true", help="--config views: render in float32")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.config == "c5":
        run_fit(args, cfg)
    elif args.config == "views":
        run_views(args, cfg)
    elif args.config == "eval":
        run_eval(args, cfg)
    else:
        run_gmr(args, cfg)


if __name__ == "__main__":
    main()
