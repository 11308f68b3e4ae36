"""N > 1 paths with one process per rank.

* CPU (gloo, world 2 and 4): the bootstrap plumbing through the library's host API -- every rank
  derives its shard of the routing from the reference generator, the per-expert counts are
  all-gathered (Alg. 1 line 3, the exchange the device planner does over NVLink), and each
  rank's token map computed by libeplab_b200.so from (its own routing + the gathered counts)
  equals the reference's global map (oracle/_ref, else the C oracle); the EPLAB_IPC_HANDLE_BYTES
  record all-gather of EpMoE.connect_distributed.
* GPU (2 and 4 processes sharing cuda:0, each with 148/N SMs): CUDA-IPC symmetric buffers opened
  across processes, the four MegaKernels at EP=N, outputs bitwise equal to the EP=1 run; a rank
  whose symmetric layout differs is rejected by connect_ipc with error 2 on every rank.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ------------------------------------------------------------------ CPU / gloo
def _cpu_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import pyoracle as po
    from paper_2604_19241_b200.model import rank_token_map, sample_routing
    _init(rank, world, port)
    try:
        E, k, T = 16, 4, 300
        sel_all, _ = sample_routing(E, k, T, world, 5)  # every rank can regenerate its shard
        mine = sel_all[rank]
        counts = torch.from_numpy(np.bincount(mine, minlength=E).astype(np.int64))
        gathered = [torch.zeros(E, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, counts)  # Alg. 1 line 3 over gloo
        c_all = torch.stack(gathered).numpy()
        tr, le, off = rank_token_map(mine, c_all, rank, world, E, k)  # the library, this rank only
        ref = po.Reference() if po.has_reference() else po.Oracle()
        rtr, rle, roff, _, _ = ref.token_map(sel_all, E, k)
        ok = bool((off == roff[rank]).all() and (tr == rtr[rank]).all() and (le == rle[rank]).all())
        rec = bytes([rank]) * 128  # EPLAB_IPC_HANDLE_BYTES records, as connect_distributed exchanges
        hs = [None] * world
        dist.all_gather_object(hs, rec)
        ok = ok and hs == [bytes([r]) * 128 for r in range(world)]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_bootstrap_and_token_map(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


# ------------------------------------------------------------------ GPU / CUDA IPC
def _gpu_worker(rank, world, port, q, mismatch=False):
    import sys
    sys.path.insert(0, ROOT)
    from tests.test_moe_gpu import Problem, from_u16, to_u16
    from paper_2604_19241_b200 import moe as M
    _init(rank, world, port)
    try:
        torch.cuda.set_device(0)
        prob = Problem(world, 8, 2, 256, 256, 256, seed=11)
        T, k, H = prob.T, prob.k, prob.H
        epr = prob.E // world
        t_max = T + 64 if (mismatch and rank == world - 1) else T
        layer = M.EpMoE(prob.H, prob.F, prob.E, k, t_max, rank=rank, world=world, timeout_s=20.0)
        if mismatch:
            try:
                layer.connect_distributed()
                q.put((rank, "connected"))
            except M.EplabError as e:
                q.put((rank, (e.code, "layout differs" in str(e))))
            dist.barrier()
            layer.close()
            return
        layer.connect_distributed()
        layer.set_sm_budget(148 // world)
        ids = torch.from_numpy(prob.sel[rank].reshape(T, k).copy()).cuda()
        gw = torch.from_numpy(prob.gw[rank].reshape(T, k).copy()).cuda()
        wu = from_u16(prob.w_up[rank * epr:(rank + 1) * epr])
        wd = from_u16(prob.w_down[rank * epr:(rank + 1) * epr])
        y = layer.forward(from_u16(prob.x[rank]), ids, gw, wu, wd)
        g = layer.backward(from_u16(prob.dy[rank]), wu, wd)
        layer.check()
        q.put((rank, dict(y=to_u16(y), dx=to_u16(g["dx"]), dgate=g["dgate"].cpu().numpy(),
                          dw_up=to_u16(g["dw_up"]), dw_down=to_u16(g["dw_down"]))))
        dist.barrier()
        layer.close()
    finally:
        dist.destroy_process_group()


def _spawn(world, mismatch=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, mismatch)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_processes_ipc_match_single_process(world):
    from tests.test_moe_gpu import Problem, gather, run_layer
    res = _spawn(world)
    prob = Problem(world, 8, 2, 256, 256, 256, seed=11)
    ep1, _, _ = run_layer(prob, world=1)
    ref = gather(ep1[0])
    got = gather([res[r] for r in range(world)])
    for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
        assert (got[key] == ref[key]).all(), key


@pytest.mark.gpu
def test_ipc_layout_mismatch_rejected_on_every_rank():
    """The last rank was created with a different max_tokens: its symmetric region has another
    layout, so every rank's connect_ipc refuses it (error 2) instead of writing at wrong offsets."""
    res = _spawn(2, mismatch=True)
    assert res == {0: (2, True), 1: (2, True)}, res
