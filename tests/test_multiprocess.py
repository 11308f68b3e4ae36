"""N > 1 paths with one process per rank.

* CPU (gloo, world 2): the bootstrap plumbing -- every rank derives its shard of the routing
  from the reference generator, the per-expert counts are all-gathered, and each rank's token
  map built from (its own routing + the gathered counts) equals the global reference map; the
  64-byte handle all-gather used by EpMoE.connect_distributed.
* GPU (two processes sharing cuda:0, each with half the SMs): CUDA-IPC symmetric buffers opened
  across processes, the four MegaKernels at EP=2, outputs bitwise equal to the EP=1 run.
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
    _init(rank, world, port)
    try:
        E, k, T = 16, 4, 300
        orc = po.Oracle()
        sel_all, _ = orc.sample_routing(E, k, T, world, 5)  # every rank can regenerate its shard
        mine = sel_all[rank]
        counts = torch.from_numpy(np.bincount(mine, minlength=E).astype(np.int64))
        gathered = [torch.zeros(E, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, counts)  # Alg. 1 line 3 over gloo
        c_all = torch.stack(gathered).numpy()
        epr = E // world
        # this rank's final offsets from its own local sort + the gathered counts (Eq. 1)
        local = np.zeros(T * k, np.int64)
        seen = np.zeros(E, np.int64)
        for i, e in enumerate(mine):
            local[i] = seen[e]
            seen[e] += 1
        o_all = c_all[:rank].sum(axis=0)
        off = local + o_all[mine]
        tr, le, ref_off, _, _ = orc.token_map(sel_all, E, k)
        ok = bool((off == ref_off[rank]).all() and (mine // epr == tr[rank]).all())
        hs = [None] * world
        dist.all_gather_object(hs, bytes([rank]) * 64)  # EpMoE.connect_distributed's exchange
        ok = ok and hs == [bytes([r]) * 64 for r in range(world)]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_bootstrap_and_token_map_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


# ------------------------------------------------------------------ GPU / CUDA IPC
def _gpu_worker(rank, world, port, q):
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
        layer = M.EpMoE(prob.H, prob.F, prob.E, k, T, rank=rank, world=world, timeout_s=20.0)
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


@pytest.mark.gpu
def test_two_processes_ipc_match_single_process():
    from tests.test_moe_gpu import Problem, gather, run_layer
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    prob = Problem(2, 8, 2, 256, 256, 256, seed=11)
    ep1, _, _ = run_layer(prob, world=1)
    ref = gather(ep1[0])
    got = gather([res[0], res[1]])
    for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
        assert (got[key] == ref[key]).all(), key
