"""Hardened parity of the EP-MoE MegaKernels.

* a15, the combine fold, BIT-EXACT against the reference's own `accumulate` (precision.cpp:31-52,
  FpFormat::Binary32): the device's replica rows (the `rep` / `rep_dx` slots at the source, exported
  after the step) folded by the reference's fold -- acc = w_0 o_0, acc = acc + w_j o_j in k order,
  fp32 rounding of every product and sum -- then rounded once to bf16 (softfloat.cpp:27-33) equal
  the device's y bit for bit; dx likewise with unit weights. Checked with a numpy restatement on
  every element and with oracle/_ref's compiled `accumulate` on a sample.
* per-element tolerance vs the CPU oracle (tests/parity.py): >= 99 % of y / dx and >= 99.9 % of
  dW elements within 1 bf16 ulp of the oracle, relative L2 <= 1e-3 / 5e-4.
* adversarial routing at EP=8 (virtual ranks): every token on one rank's experts (seven empty
  ranks), one rank never routed to, n_tok % 128 != 0 -- each bitwise equal to EP=1 and within the
  tolerance of the oracle.
* the DeepSeek-V3 shape (H 7168, F 2048, 256 experts, top-8; the AllGather regime) at EP=8 on
  virtual ranks, relay on and off, bitwise equal to EP=1.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pyoracle as po  # noqa: E402
from tests.parity import assert_layer  # noqa: E402
from tests.test_moe_gpu import Problem, bf16_to_f32, gather, run_layer  # noqa: E402


def round_bf16(x):
    """softfloat.cpp:27-33 round_to_bf16 (RNE, NaN quieted) on float32 arrays -> float32."""
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    nan = np.isnan(x)
    r[nan] = ((x.astype(np.float32).view(np.uint32)[nan] | 0x00400000) & 0xFFFF0000)
    return r.view(np.float32)


def ref_fold_np(w, v):
    """precision.cpp:31-37 fold with FpFormat::Binary32, vectorised: w [n_tok, k], v [n_tok, k, H]
    (float32); numpy float32 ops round every product and sum (no contraction)."""
    acc = (w[:, 0:1] * v[:, 0, :]).astype(np.float32)
    for j in range(1, w.shape[1]):
        acc = (acc + (w[:, j:j + 1] * v[:, j, :]).astype(np.float32)).astype(np.float32)
    return acc


def _check_fold(prob, outs, world):
    T, k, H = prob.T * prob.world // world, prob.k, prob.H
    gw_all = prob.gw.reshape(-1, k)
    for r in range(world):
        o = outs[r]
        rep = bf16_to_f32(o["rep"]).reshape(T, k, H)
        rep_dx = bf16_to_f32(o["rep_dx"]).reshape(T, k, H)
        w = gw_all[r * T:(r + 1) * T].astype(np.float32)
        y_ref = round_bf16(ref_fold_np(w, rep))
        dx_ref = round_bf16(ref_fold_np(np.ones_like(w), rep_dx))
        y = bf16_to_f32(o["y"]).reshape(T, H)
        dx = bf16_to_f32(o["dx"]).reshape(T, H)
        assert (y.view(np.uint32) == y_ref.view(np.uint32)).all(), f"rank {r}: y != fold(rep)"
        assert (dx.view(np.uint32) == dx_ref.view(np.uint32)).all(), f"rank {r}: dx != fold(rep_dx)"
        if po.has_reference():  # the reference's compiled accumulate() on a sample of elements
            ref = po.Reference()
            rng = np.random.default_rng(r)
            for t, n in zip(rng.integers(0, T, 64), rng.integers(0, H, 64)):
                a = ref.round_to_bf16(ref.fold(np.ascontiguousarray(w[t]), np.ascontiguousarray(rep[t, :, n]), False))
                assert np.float32(a).view(np.uint32) == y[t, n].view(np.uint32), (r, t, n)
                b = ref.round_to_bf16(ref.fold(np.ones(k, np.float32), np.ascontiguousarray(rep_dx[t, :, n]), False))
                assert np.float32(b).view(np.uint32) == dx[t, n].view(np.uint32), (r, t, n)


@pytest.mark.parametrize("W,E,k,T,cfg", [(1, 8, 2, 300, None), (1, 32, 8, 200, None), (1, 16, 16, 130, None),
                                         (2, 16, 4, 192, (4, 2, 1, 74, 8)), (4, 32, 8, 96, (2, 2, 1, 37, 8))])
def test_combine_fold_bit_exact_vs_reference_accumulate(W, E, k, T, cfg):
    prob = Problem(W, E, k, 256, 256, T, seed=31)
    outs, _, _ = run_layer(prob, cfg=cfg, keep=("rep", "rep_dx"))
    _check_fold(prob, outs[0], W)


@pytest.mark.parametrize("W,E,k,H,F,T", [(1, 8, 2, 512, 512, 384), (1, 16, 4, 512, 512, 200),
                                         (1, 32, 8, 1024, 256, 256), (2, 16, 4, 256, 512, 192)])
def test_per_element_ulp_tolerance_vs_oracle(W, E, k, H, F, T):
    prob = Problem(W, E, k, H, F, T, seed=5)
    outs, _, _ = run_layer(prob)
    assert_layer(gather(outs[0]), prob.oracle())


def _adversarial(kind, W=8, E=32, k=4, T=333, seed=41):
    prob = Problem(W, E, k, 256, 256, T, seed=seed)
    rng = np.random.default_rng(seed)
    epr = E // W
    if kind == "one_hot_rank":  # every token of every rank on rank 0's experts: 7 ranks receive nothing
        sel = np.stack([rng.permutation(epr)[:k] for _ in range(W * T)]).astype(np.int32)
    elif kind == "empty_rank":  # nobody routes to rank W-1's experts
        allowed = np.arange(E - epr)
        sel = np.stack([rng.choice(allowed, k, replace=False) for _ in range(W * T)]).astype(np.int32)
    else:
        raise ValueError(kind)
    prob.sel = sel.reshape(W, T * k)
    return prob


@pytest.mark.parametrize("kind", ["one_hot_rank", "empty_rank"])
def test_adversarial_routing_ep8(kind):
    """n_tok = 333 per rank (not a multiple of 128) on 8 virtual ranks; relay on and off."""
    prob = _adversarial(kind)
    ep1, _, _ = run_layer(prob, world=1)
    ref1 = gather(ep1[0])
    for cfg in [(2, 0, 1, 18, 8), (1, 2, 1, 18, 8)]:
        ep8, _, _ = run_layer(prob, cfg=cfg)
        got = gather(ep8[0])
        for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
            assert (got[key] == ref1[key]).all(), f"{kind} {cfg}: EP=8 != EP=1 in {key}"
    assert_layer(ref1, prob.oracle())


@pytest.mark.parametrize("relay", [0, 2])
def test_dsv3_dims_ep8_virtual_ranks_bitwise_equal_ep1(relay):
    """DeepSeek-V3 layer dims (H 7168, F 2048, 256 experts, top-8: ~5.3 distinct ranks per token,
    the AllGather regime where the relay dedups) with 2048 tokens per rank on 8 virtual ranks
    equal EP=1 over the same 16K tokens bit for bit; relay off (AllToAll) and on (AllGather)."""
    from paper_2604_19241_b200 import moe as M
    from paper_2604_19241_b200.model import sample_routing
    H, F, E, k, T, W = 7168, 2048, 256, 8, 2048, 8
    sel, gw = sample_routing(E, k, T, W, 13)
    g = torch.Generator(device="cuda").manual_seed(17)
    x = torch.randn(W * T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(W * T, H, device="cuda", generator=g) * 0.5).bfloat16()
    w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    ids = torch.from_numpy(sel.reshape(W * T, k).copy()).cuda()
    gws = torch.from_numpy(gw.reshape(W * T, k).copy()).cuda()
    one = M.EpMoE(H, F, E, k, W * T, max_recv_rows=W * T * k)
    y1 = one.forward(x, ids, gws, w_up, w_down)
    g1 = one.backward(dy, w_up, w_down)
    one.check()
    torch.cuda.synchronize()
    one.close()
    epr = E // W
    ranks = [M.EpMoE(H, F, E, k, T, rank=r, world=W, max_recv_rows=T * k * 5 // 4, timeout_s=60.0)
             for r in range(W)]
    M.EpMoE.connect_local(ranks)
    for r in ranks:
        r.set_sm_budget(148 // W)
        r.set_tune_config((2, relay, 1, 148 // W, 8))
    streams = [torch.cuda.Stream() for _ in range(W)]
    torch.cuda.synchronize()
    ys, gs = [None] * W, [None] * W
    for ph in range(3):
        for r in range(W):
            sl = slice(r * T, (r + 1) * T)
            with torch.cuda.stream(streams[r]):
                if ph == 0:
                    ranks[r].plan(ids[sl], gws[sl], streams[r])
                elif ph == 1:
                    ranks[r].dispatch_group_gemm(x[sl], w_up[r * epr:(r + 1) * epr], streams[r])
                    ys[r] = ranks[r].group_gemm_combine(w_down[r * epr:(r + 1) * epr], stream=streams[r])
                else:
                    gs[r] = ranks[r].backward(dy[sl], w_up[r * epr:(r + 1) * epr], w_down[r * epr:(r + 1) * epr],
                                              stream=streams[r])
        if ph == 0:
            torch.cuda.synchronize()
    for r in range(W):
        ranks[r].check(streams[r])
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(ys), y1), "y"
    for key in ("dx", "dgate", "dw_up", "dw_down"):
        assert torch.equal(torch.cat([gg[key] for gg in gs]), g1[key]), key
    for r in ranks:
        r.close()
