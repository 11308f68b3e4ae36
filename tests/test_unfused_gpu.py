"""The unfused NCCL baseline (paper_2604_19241_b200/unfused.py) is the bitwise
reference of the fused MegaKernels -- the reference's fused_vs_sequential contract
(precision.cpp:54-96, tests/test_precision.cpp:105-116: the fused combine equals the sequential
combine bit for bit): same routing, same inputs, every output of a fwd+bwd step identical, at EP=1,
at EP=2 / EP=4 on virtual ranks, and at EP=2 in two processes exchanging over torch.distributed.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_moe_gpu import Problem, from_u16, gather, run_layer, to_u16  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(prob, W):
    T = prob.world * prob.T // W
    epr = prob.E // W
    sel, gw = prob.sel.reshape(-1, prob.k), prob.gw.reshape(-1, prob.k)
    x, dy = prob.x.reshape(-1, prob.H), prob.dy.reshape(-1, prob.H)
    out = dict(xs=[], ids=[], gws=[], dys=[], w_ups=[], w_downs=[])
    for r in range(W):
        sl = slice(r * T, (r + 1) * T)
        out["ids"].append(torch.from_numpy(np.ascontiguousarray(sel[sl])).cuda())
        out["gws"].append(torch.from_numpy(np.ascontiguousarray(gw[sl])).cuda())
        out["xs"].append(from_u16(x[sl]))
        out["dys"].append(from_u16(dy[sl]))
        out["w_ups"].append(from_u16(prob.w_up[r * epr:(r + 1) * epr]))
        out["w_downs"].append(from_u16(prob.w_down[r * epr:(r + 1) * epr]))
    return T, out


def run_unfused(prob, W):
    from paper_2604_19241_b200.unfused import LocalComm, UnfusedEpMoE, unfused_step
    T, a = _inputs(prob, W)
    layers = [UnfusedEpMoE(prob.H, prob.F, prob.E, prob.k, T, rank=r, world=W) for r in range(W)]
    ys, gs = unfused_step(layers, LocalComm(), a["xs"], a["ids"], a["gws"], a["dys"], a["w_ups"], a["w_downs"])
    for L in layers:
        L.check()
    torch.cuda.synchronize()
    out = [dict(y=to_u16(ys[r]), dx=to_u16(gs[r]["dx"]), dgate=gs[r]["dgate"].cpu().numpy(),
                dw_up=to_u16(gs[r]["dw_up"]), dw_down=to_u16(gs[r]["dw_down"])) for r in range(W)]
    for L in layers:
        L.close()
    return out


@pytest.mark.parametrize("W,E,k,H,F,T", [(1, 8, 2, 512, 512, 384), (1, 16, 4, 256, 512, 300),
                                         (1, 32, 8, 1024, 256, 200), (2, 16, 4, 256, 256, 192),
                                         (4, 32, 8, 256, 256, 160)])
def test_fused_equals_unfused_bitwise(W, E, k, H, F, T):
    prob = Problem(W, E, k, H, F, T, seed=37)
    fused, _, _ = run_layer(prob)
    unf = run_unfused(prob, W)
    a, b = gather(fused[0]), gather(unf)
    for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
        assert (a[key] == b[key]).all(), f"W={W}: fused != unfused in {key}"


def test_fused_equals_unfused_mixtral_shape_reduced_tokens():
    """Full Mixtral dims (H 4096, F 14336, 8 experts, top-2), 2048 tokens: long-K tiles."""
    prob = Problem(1, 8, 2, 4096, 14336, 2048, seed=3)
    fused, _, _ = run_layer(prob)
    unf = run_unfused(prob, 1)
    a, b = gather(fused[0]), gather(unf)
    for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
        assert (a[key] == b[key]).all(), key


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_19241_b200.unfused import NcclComm, UnfusedEpMoE, unfused_step
        torch.cuda.set_device(0)
        prob = Problem(world, 16, 4, 256, 256, 192, seed=37)
        T, a = _inputs(prob, world)
        L = UnfusedEpMoE(prob.H, prob.F, prob.E, prob.k, T, rank=rank, world=world)
        ys, gs = unfused_step([L], NcclComm(staged=True), [a["xs"][rank]], [a["ids"][rank]], [a["gws"][rank]],
                              [a["dys"][rank]], [a["w_ups"][rank]], [a["w_downs"][rank]])
        L.check()
        q.put((rank, dict(y=to_u16(ys[0]), dx=to_u16(gs[0]["dx"]), dgate=gs[0]["dgate"].cpu().numpy(),
                          dw_up=to_u16(gs[0]["dw_up"]), dw_down=to_u16(gs[0]["dw_down"]))))
        dist.barrier()
        L.close()
    except Exception as e:  # fail the test at once instead of timing out on the queue
        q.put((rank, f"worker {rank} failed: {type(e).__name__}: {e}"))
        raise
    finally:
        dist.destroy_process_group()


def test_unfused_two_processes_equals_fused():
    """EP=2 with one process per rank and the collectives over torch.distributed (the bench's NCCL
    path; gloo with host staging here, because NCCL refuses two ranks on one GPU)."""
    import torch.multiprocessing as mp
    from tests.test_multiprocess import _free_port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert all(isinstance(v, dict) for v in res.values()), res
    prob = Problem(2, 16, 4, 256, 256, 192, seed=37)
    fused, _, _ = run_layer(prob)
    a, b = gather(fused[0]), gather([res[0], res[1]])
    for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
        assert (a[key] == b[key]).all(), key
