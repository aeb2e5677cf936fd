"""Multi-GPU view sharding.

The reference sums per-view vertex gradients in a serial Python loop
(`losses.py:151-162`: grad_v += gv, grad_c += gc, each view scaled by w/n).
Views are independent given the mesh, so every rank renders a contiguous
shard of the batch on its own GPU, and the only exchange is one SUM
all-reduce of the packed [grad_pos | grad_col] (V x 6) buffer plus the
loss partial sums.  One process per GPU, `torch.distributed` with NCCL
over NVLink/NVSwitch (gloo works for CPU tests of this logic).

Single-rank vs R-rank results differ only by the summation order of the
all-reduce.  NCCL picks its algorithm (ring, tree, NVLS in-switch
reduction) per size and topology, so the default SUM is not guaranteed to
be bit-identical across runs or machines; `reproducible=True` all-gathers
the per-rank partials and sums them in rank order instead (SURVEY 8e's
bit-reproducible mode): the result then depends only on the world size.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Contiguous split of n views: rank r gets [r*n/R, (r+1)*n/R)."""
    return (rank * n) // world, ((rank + 1) * n) // world


class PendingReduce:
    """An all-reduce in flight on the backend's own stream (async_op=True):
    the caller's stream keeps rendering the next view group meanwhile.
    wait() makes the current stream wait for it and returns the result."""

    def __init__(self, work, result):
        self.work, self.result = work, result

    def wait(self):
        if self.work is not None:
            self.work.wait()
        return self.result


def allreduce_vertex_grads(g_pos: torch.Tensor, g_col: torch.Tensor, extra: torch.Tensor | None = None,
                           group=None, reproducible: bool = False, async_op: bool = False):
    """One packed SUM all-reduce of [grad_pos | grad_col (| extra scalars)].

    reproducible: all-gather the packed partials and add them in rank order
    (R x the buffer in memory and traffic; bit-identical for a given world
    size whatever algorithm NCCL would have chosen).
    async_op: return a PendingReduce instead of waiting (plain SUM only), so
    one view group's reduction overlaps the next group's kernels; the sum of
    the groups' reduced buffers equals the reduction of their sum up to
    floating-point summation order."""
    parts = [g_pos.reshape(-1), g_col.reshape(-1)]
    if extra is not None:
        parts.append(extra.reshape(-1).to(g_pos.dtype))
    buf = torch.cat(parts)
    n = g_pos.numel()

    def split(b):
        return b[:n].view_as(g_pos), b[n:2 * n].view_as(g_col), (b[2 * n:] if extra is not None else None)

    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if async_op:
        if reproducible:
            raise ValueError("async_op needs the plain SUM all-reduce (reproducible=False)")
        work = dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group, async_op=True) if multi else None
        return PendingReduce(work, split(buf))
    if multi:
        if reproducible:
            world = dist.get_world_size(group)
            gathered = torch.empty(world * buf.numel(), dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(gathered, buf, group=group)
            gathered = gathered.view(world, buf.numel())
            buf = gathered[0].clone()
            for r in range(1, world):
                buf += gathered[r]
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return split(buf)


def sharded_image_loss(local_fn: Callable, cameras: Sequence, target_rgb: Sequence, target_mask: Sequence,
                       num_vertices: int, w_color: float = 1.0, w_sil: float = 1.0, group=None,
                       device=None, reproducible: bool = False):
    """Image part of `total_loss` (losses.py:146-164) over views sharded
    across the process group.

    `local_fn(cams, rgbs, masks, scale_rgb, scale_alpha)` evaluates this
    rank's views and returns (sum of per-view colour losses, sum of per-view
    silhouette losses, grad_pos [V,3], grad_col [V,3]) with image grads
    pre-scaled by w/n (n = the GLOBAL view count) -- on the GPU that is
    `gpu_local_image_loss` below.  Returns
    (color, silhouette, grad_pos, grad_col) identical on every rank.
    """
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if device is None:
        # every rank must hand the collective a tensor on the backend's device,
        # including ranks whose shard is empty (more ranks than views)
        nccl = dist.is_available() and dist.is_initialized() and dist.get_backend(group) == "nccl"
        device = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    n = len(cameras)
    lo, hi = shard_range(n, rank, world)
    if hi > lo:
        cval, sval, gp, gc = local_fn(cameras[lo:hi], target_rgb[lo:hi], target_mask[lo:hi],
                                      w_color / n, w_sil / n)
        gp = torch.as_tensor(gp, dtype=torch.float64).to(device)
        gc = torch.as_tensor(gc, dtype=torch.float64).to(device)
        extra = torch.stack([torch.as_tensor(cval, dtype=torch.float64).to(device).reshape(()),
                             torch.as_tensor(sval, dtype=torch.float64).to(device).reshape(())])
    else:
        gp = torch.zeros((num_vertices, 3), dtype=torch.float64, device=device)
        gc = torch.zeros((num_vertices, 3), dtype=torch.float64, device=device)
        extra = torch.zeros(2, dtype=torch.float64, device=device)
    gp, gc, extra = allreduce_vertex_grads(gp, gc, extra, group, reproducible)
    ex = extra.cpu()   # the one host read: the two loss values
    return float(ex[0]) / n, float(ex[1]) / n, gp, gc


def gpu_local_image_loss(mesh, background=(0.0, 0.0, 0.0), rescale=True, dtype=np.float32):
    """The GPU `local_fn` for `sharded_image_loss`: this rank's views in one
    libgmr call per resolution, with the colour/silhouette losses fused into
    the blend epilogue (gmr_render_forward_loss, the paper_2602_14493_b200
    .api.total_loss path).  Losses and gradients stay on the device; the
    call's status is validated after the backward is enqueued."""
    from . import api, engine

    pos, col, faces = api._device_mesh(mesh, dtype)
    tdt = api._torch_dtype(dtype)
    dev = pos.device
    bg = np.asarray(background, np.float64)

    def local_fn(cams, rgbs, masks, scale_rgb, scale_alpha):
        gp_all = torch.zeros((pos.shape[0], 3), dtype=torch.float64, device=dev)
        gc_all = torch.zeros_like(gp_all)
        loss = torch.zeros(2, dtype=torch.float64, device=dev)
        groups = {}
        for i, c in enumerate(cams):
            groups.setdefault((c.width, c.height), []).append(i)
        for (w, h), idx in groups.items():
            t_rgb = torch.as_tensor(np.stack([np.asarray(rgbs[i], np.float64) for i in idx]), dtype=tdt).to(dev)
            t_m = torch.as_tensor(np.stack([np.asarray(masks[i], np.float64) for i in idx]), dtype=tdt).to(dev)
            for attempt in range(3):
                rgb, alpha, g_rgb, g_a, sums, st = engine.render_forward_loss(
                    pos, col, faces, [cams[i] for i in idx], w, h, bg, t_rgb, t_m, scale_rgb, scale_alpha,
                    rescale, check=False)
                gp, gc = engine.render_backward(st, pos, col, faces, rgb, g_rgb, g_a)
                try:
                    # waits for this forward's status copy only; the backward stays queued
                    engine.check_status(st)
                    break
                except engine.CapacityExceeded:
                    if attempt == 2:
                        raise
            loss[0] += sums[0] / (3.0 * w * h)
            loss[1] += sums[1] / (1.0 * w * h)
            gp_all += gp.double()
            gc_all += gc.double()
        return loss[0], loss[1], gp_all, gc_all

    return local_fn
