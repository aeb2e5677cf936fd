"""World-size-2 gloo tests of the view-sharding host logic.

The per-rank compute is injected: here the pinned CPU oracle renders each
rank's shard, so the test checks the sharding, the w/n scaling with the
GLOBAL view count and the packed all-reduce against the single-process
reference semantics (losses.py:151-164).  On the GPU the same function runs
with `dist.gpu_local_image_loss` (NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_cases as gc
from oracle import gmr_oracle as orc
from paper_2602_14493_b200 import dist as gdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_local_fn(case):
    def fn(cams, rgbs, masks, scale_rgb, scale_alpha):
        gv = np.zeros((len(case["vertices"]), 3))
        gcol = np.zeros_like(gv)
        cv = sv = 0.0
        for cam, rt, mt in zip(cams, rgbs, masks):
            rgb, alpha, ctx = orc.render(case["vertices"], case["facets"], case["colors"], cam,
                                         case["background"])
            c, g_rgb = orc.color_loss(rgb, rt)
            s, g_a = orc.silhouette_loss(alpha, mt)
            cv += c
            sv += s
            a, b = orc.render_grad(ctx, scale_rgb * g_rgb, scale_alpha * g_a)
            gv += a
            gcol += b
        return cv, sv, gv, gcol
    return fn


def _worker(rank, world, port, ncams, q, reproducible=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = gc.loss_case()
        cams = (case["cameras"] * 3)[:ncams]
        rgbs = (case["target_rgb"] * 3)[:ncams]
        masks = (case["target_mask"] * 3)[:ncams]
        c, s, gp, gcol = gdist.sharded_image_loss(oracle_local_fn(case), cams, rgbs, masks,
                                                  len(case["vertices"]), reproducible=reproducible)
        q.put((rank, c, s, gp.numpy(), gcol.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ncams", [3, 4, 1])
def test_two_rank_sharding_matches_single_process(ncams):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ncams, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = gc.loss_case()
    cams = (case["cameras"] * 2)[:ncams]
    rgbs = (case["target_rgb"] * 2)[:ncams]
    masks = (case["target_mask"] * 2)[:ncams]
    cv, sv, gv, gcol = orc.views_image_grad(case["vertices"], case["facets"], case["colors"], cams, rgbs,
                                            masks, background=case["background"])
    for _, c, s, gp, gcc in res:
        assert c == pytest.approx(cv, rel=1e-12) and s == pytest.approx(sv, rel=1e-12)
        np.testing.assert_allclose(gp, gv, rtol=0, atol=1e-12)
        np.testing.assert_allclose(gcc, gcol, rtol=0, atol=1e-12)
    # both ranks hold identical results (replicated optimiser input)
    np.testing.assert_array_equal(res[0][3], res[1][3])


def test_four_rank_reproducible_sum_in_rank_order():
    """World size 4 over 3 views (one rank holds an empty shard), the
    reproducible mode: every rank returns exactly the rank-order sum of the
    per-shard partials, and that sum matches the single-process result."""
    ncams, world = 3, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ncams, q, True)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = gc.loss_case()
    cams, rgbs, masks = case["cameras"][:ncams], case["target_rgb"][:ncams], case["target_mask"][:ncams]
    fn = oracle_local_fn(case)
    V = len(case["vertices"])
    exp_p, exp_c = np.zeros((V, 3)), np.zeros((V, 3))
    for r in range(world):
        lo, hi = gdist.shard_range(ncams, r, world)
        if hi > lo:
            _, _, a, b = fn(cams[lo:hi], rgbs[lo:hi], masks[lo:hi], 1.0 / ncams, 1.0 / ncams)
        else:
            a, b = np.zeros((V, 3)), np.zeros((V, 3))
        exp_p, exp_c = exp_p + a, exp_c + b
    cv, sv, gv, gcol = orc.views_image_grad(case["vertices"], case["facets"], case["colors"], cams, rgbs,
                                            masks, background=case["background"])
    for _, c, s, gp, gcc in res:
        np.testing.assert_array_equal(gp, exp_p)
        np.testing.assert_array_equal(gcc, exp_c)
        np.testing.assert_allclose(gp, gv, rtol=0, atol=1e-12)
        assert c == pytest.approx(cv, rel=1e-12) and s == pytest.approx(sv, rel=1e-12)


def test_eight_rank_sharding_matches_single_process():
    """World size 8 (R in {1, 2, 4, 8}) over 9 views: shards of
    one or two views, gradients and losses equal to the single-process
    reference semantics on every rank."""
    ncams, world = 9, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ncams, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = gc.loss_case()
    cams = (case["cameras"] * 3)[:ncams]
    rgbs = (case["target_rgb"] * 3)[:ncams]
    masks = (case["target_mask"] * 3)[:ncams]
    cv, sv, gv, gcol = orc.views_image_grad(case["vertices"], case["facets"], case["colors"], cams, rgbs,
                                            masks, background=case["background"])
    for _, c, s, gp, gcc in res:
        assert c == pytest.approx(cv, rel=1e-12) and s == pytest.approx(sv, rel=1e-12)
        np.testing.assert_allclose(gp, gv, rtol=0, atol=1e-12)
        np.testing.assert_allclose(gcc, gcol, rtol=0, atol=1e-12)
    for r in res[1:]:
        np.testing.assert_array_equal(res[0][3], r[3])


def test_shard_ranges_cover_views_once():
    for n in range(0, 17):
        for world in (1, 2, 3, 4, 8):
            spans = [gdist.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_allreduce_single_process_is_identity():
    gp, gcol = torch.randn(5, 3), torch.randn(5, 3)
    a, b, e = gdist.allreduce_vertex_grads(gp.clone(), gcol.clone(), torch.tensor([1.0, 2.0]))
    assert torch.equal(a, gp) and torch.equal(b, gcol) and e.tolist() == [1.0, 2.0]


def _async_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(100 + rank)
        groups = [(torch.randn(7, 3, generator=g, dtype=torch.float64),
                   torch.randn(7, 3, generator=g, dtype=torch.float64)) for _ in range(3)]
        # per view group, in flight together, summed after (bench.py's overlapped step)
        pend = [gdist.allreduce_vertex_grads(a, b, async_op=True) for a, b in groups]
        parts = [p.wait() for p in pend]
        gp = parts[0][0] + parts[1][0] + parts[2][0]
        gc_ = parts[0][1] + parts[1][1] + parts[2][1]
        # one reduction of the summed groups
        sp, sc, _ = gdist.allreduce_vertex_grads(sum(a for a, _ in groups), sum(b for _, b in groups))
        q.put((rank, gp.numpy(), gc_.numpy(), sp.numpy(), sc.numpy()))
    finally:
        dist.destroy_process_group()


def test_async_group_reductions_match_one_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_async_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, gp, gcol, sp, sc in res:
        np.testing.assert_allclose(gp, sp, rtol=0, atol=1e-12)
        np.testing.assert_allclose(gcol, sc, rtol=0, atol=1e-12)
    np.testing.assert_array_equal(res[0][1], res[1][1])   # identical on every rank
    with pytest.raises(ValueError):
        gdist.allreduce_vertex_grads(torch.zeros(2, 3), torch.zeros(2, 3), reproducible=True, async_op=True)
