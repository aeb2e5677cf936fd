"""The multi-GPU path on NCCL, on the one GPU a box has.

`tests/test_dist_cpu.py` checks the sharding logic at world size 2 and 4 on
gloo. Here the same functions run with the NCCL backend and the CUDA local
loss (`dist.gpu_local_image_loss`: fused-loss forward + backward through
libgmr) at world size 1, against the pinned oracle's single-process sums
(losses.py:151-164). The bench's torchrun launch form (the driver's N > 1
command line) is also run end to end with one rank."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import golden_cases as gc
from oracle import gmr_oracle as orc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    torch.cuda.set_device(0)
    store = dist.TCPStore("127.0.0.1", _free_port(), 1, is_master=True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        yield dist
    finally:
        dist.destroy_process_group()


def _oracle_sums(case, cams, rgbs, masks):
    n = len(cams)
    gv = np.zeros((len(case["vertices"]), 3))
    gcol = np.zeros_like(gv)
    cv = sv = 0.0
    for cam, rt, mt in zip(cams, rgbs, masks):
        rgb, alpha, ctx = orc.render(case["vertices"], case["facets"], case["colors"], cam, case["background"])
        c, g_rgb = orc.color_loss(rgb, rt)
        s, g_a = orc.silhouette_loss(alpha, mt)
        cv += c
        sv += s
        a, b = orc.render_grad(ctx, g_rgb / n, g_a / n)
        gv += a
        gcol += b
    return cv / n, sv / n, gv, gcol


@pytest.mark.parametrize("reproducible", [False, True])
def test_nccl_sharded_image_loss_matches_oracle(gmr, nccl_group, reproducible):
    import paper_2602_14493_b200 as g
    from paper_2602_14493_b200 import dist as gdist
    case = gc.loss_case()
    mesh = g.TriangleMesh(case["vertices"], case["facets"], case["colors"])
    cams, rgbs, masks = case["cameras"], case["target_rgb"], case["target_mask"]
    local = gdist.gpu_local_image_loss(mesh, background=case["background"], dtype=np.float64)
    c, s, gp, gcol = gdist.sharded_image_loss(local, cams, rgbs, masks, len(case["vertices"]),
                                              reproducible=reproducible)
    assert gp.is_cuda and gcol.is_cuda   # NCCL backend: results stay on the device
    rc, rs, rgv, rgc = _oracle_sums(case, cams, rgbs, masks)
    assert abs(c - rc) <= 1e-10 * max(1.0, abs(rc)) and abs(s - rs) <= 1e-10 * max(1.0, abs(rs))
    for ours, ref in ((gp.cpu().numpy(), rgv), (gcol.cpu().numpy(), rgc)):
        assert np.abs(ours - ref).max() <= 1e-8 * max(1.0, np.abs(ref).max())


def test_nccl_collectives_on_device(gmr, nccl_group):
    """The collectives the sharded path uses (SUM all-reduce, all-gather of
    the packed partials) run on this box's NCCL with device buffers."""
    import torch
    dist = nccl_group
    assert dist.get_backend() == "nccl"
    x = torch.arange(12, dtype=torch.float64, device="cuda")
    y = x.clone()
    dist.all_reduce(y, op=dist.ReduceOp.SUM)
    assert torch.equal(x, y)
    out = torch.empty(12, dtype=torch.float64, device="cuda")
    dist.all_gather_into_tensor(out, x)
    assert torch.equal(out, x)


def test_nccl_async_group_reduction(gmr, nccl_group):
    import torch
    from paper_2602_14493_b200 import dist as gdist
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = [torch.randn(1000, 3, generator=gen, device="cuda", dtype=torch.float64) for _ in range(4)]
    pend = [gdist.allreduce_vertex_grads(a[i], a[i + 1], async_op=True) for i in (0, 2)]
    outs = [p.wait() for p in pend]
    torch.testing.assert_close(outs[0][0] + outs[1][0], a[0] + a[2], rtol=0, atol=0)
    torch.testing.assert_close(outs[0][1] + outs[1][1], a[1] + a[3], rtol=0, atol=0)


def test_bench_under_torchrun_one_rank(gmr):
    """The driver's N > 1 launch form with one rank: NCCL init and the
    max-over-ranks timing run (GMR_BENCH_DIST=1); the vertex-gradient
    all-reduce is an identity at one rank and is skipped."""
    env = dict(os.environ, GMR_BENCH_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--config", "c1",
           "--steps", "3", "--warmup", "3", "--no-cpu", "--no-extras"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout.strip().splitlines()
    # the JSON line last; NCCL's INFO lines go to stderr (only its version banner reaches stdout)
    assert all(x.startswith("NCCL version") for x in out[:-1]), out[:5]
    line = json.loads(out[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert "NCCL all-reduce" in line["config"]["parallelism"]
