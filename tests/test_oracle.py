"""Pins the CPU oracle (oracle/liborc.so) to the reference.

Three anchors, per SURVEY.md §8(c):
  1. the reference's own golden vectors / known-answer tests (proj/tests/*.cpp, cited per test);
  2. the reference compiled from its sources (oracle/_ref/libeplab_ref.so) on seeded inputs;
  3. the committed fixtures in tests/golden/ (generated from (2) by tests/golden/make_golden.py),
     which travel to machines where /root/reference is absent.
"""
import ctypes
import os

import numpy as np
import pytest

from oracle import pyoracle as po

ORC = po.Oracle()
REF = po.Reference() if po.has_reference() else None
needs_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built (reference not mounted)")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cluster1(world=8):  # test_perf_model.cpp:13-24
    return po.make_hw(132, 989e12, 3.35e12, 200e9, world)


def moe1(n_tok=32768):  # test_perf_model.cpp:26-36
    return po.make_shape(2048, 1408, 64, 6, n_tok, s_tok=4096)


def gather_stable_sort(sel, n_exp, topk):
    """support.hpp:32-52: concat (src,t,j), stable sort by expert, position in segment."""
    world = sel.shape[0]
    epr = n_exp // world
    copies = [(sel[r][i], r, i) for r in range(world) for i in range(sel.shape[1])]
    copies.sort(key=lambda c: c[0])  # Python sort is stable
    pos = [0] * n_exp
    out = {}
    for e, r, i in copies:
        out[(r, i)] = (e // epr, e % epr, pos[e])
        pos[e] += 1
    return out


# ------------------------------------------------------------------ routing (a2)
def test_routing_forced_selection():  # test_core.cpp:95-105
    sel, _ = ORC.sample_routing(2, 2, 64, 1, 42)
    for t in range(64):
        assert set(sel[0][2 * t:2 * t + 2]) == {0, 1}


def test_routing_purity_and_invariants():  # test_core.cpp:107-138
    a = ORC.sample_routing(32, 4, 128, 4, 7)
    b = ORC.sample_routing(32, 4, 128, 4, 7)
    c = ORC.sample_routing(32, 4, 128, 4, 8)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and not (a[0] == c[0]).all()
    for seed in range(200):
        sel, gw = ORC.sample_routing(16, 5, 17, 2, seed)
        s = sel.reshape(2, 17, 5)
        assert all(len(set(s[r, t])) == 5 for r in range(2) for t in range(17))
        assert ((sel >= 0) & (sel < 16)).all() and np.isfinite(gw).all()
    _, gw = ORC.sample_routing(16, 5, 17, 2, 3)
    assert np.allclose(gw.reshape(2, 17, 5).sum(-1), 1.0, atol=1e-5)


def test_routing_mean_distinct_ranks_without_replacement():  # test_core.cpp:151-175
    sel, _ = ORC.sample_routing(256, 8, 125000, 8, 7)
    ranks = sel.reshape(8, 125000, 8) // 32
    srt = np.sort(ranks, axis=-1)
    distinct = 1 + (np.diff(srt, axis=-1) != 0).sum(-1)
    mean = distinct.mean()
    assert abs(mean - 5.29465) / 5.29465 < 0.002


@needs_ref
@pytest.mark.parametrize("n_exp,topk,n_tok,world,seed", [(8, 2, 300, 2, 7), (128, 8, 257, 8, 0),
                                                         (256, 8, 64, 8, 1), (16, 16, 33, 4, 99)])
def test_routing_bit_exact_vs_reference(n_exp, topk, n_tok, world, seed):
    a = ORC.sample_routing(n_exp, topk, n_tok, world, seed)
    b = REF.sample_routing(n_exp, topk, n_tok, world, seed)
    assert (a[0] == b[0]).all()
    assert (a[1].view(np.uint32) == b[1].view(np.uint32)).all()


# ------------------------------------------------------------------ token map (a3-a5)
def test_token_map_spec_two_rank_example():  # test_token_map.cpp:97-107
    sel = np.array([[0, 1], [1, 0]], np.int32)
    tr, le, off, _, _ = ORC.token_map(sel, 2, 1)
    assert (tr[0][0], le[0][0], off[0][0]) == (0, 0, 0)
    assert (tr[1][1], le[1][1], off[1][1]) == (0, 0, 1)
    assert (tr[0][1], le[0][1], off[0][1]) == (1, 0, 0)
    assert (tr[1][0], le[1][0], off[1][0]) == (1, 0, 1)


def test_token_map_hand_local_sort():  # test_token_map.cpp:52-58
    tr, le, off, rt, sb = ORC.token_map(np.array([[1, 0]], np.int32), 2, 1)
    assert list(off[0]) == [0, 0] and list(rt) == [1, 1] and list(sb) == [0, 1]


def test_token_map_matches_gather_sort_oracle_100_seeds():  # test_token_map.cpp:119-124
    for seed in range(100):
        sel, _ = ORC.sample_routing(8, 2, 16, 4, seed)
        tr, le, off, _, _ = ORC.token_map(sel, 8, 2)
        exp = gather_stable_sort(sel, 8, 2)
        for (r, i), (d, e, o) in exp.items():
            assert (tr[r][i], le[r][i], off[r][i]) == (d, e, o)


def test_token_map_bijection():  # test_token_map.cpp:126-144
    sel, _ = ORC.sample_routing(16, 4, 16, 4, 11)
    tr, le, off, rt, _ = ORC.token_map(sel, 16, 4)
    keys = set(zip(tr.ravel(), le.ravel(), off.ravel()))
    assert len(keys) == tr.size
    for d, e, o in keys:
        assert 0 <= o < rt[d * 4 + e]


def test_token_map_rejects_bad_routing():  # types.cpp:74-94
    with pytest.raises(ValueError):
        ORC.token_map(np.array([[0, 0]], np.int32), 2, 2)  # duplicate expert
    with pytest.raises(ValueError):
        ORC.token_map(np.array([[5, 0]], np.int32), 2, 2)  # out of range


@needs_ref
@pytest.mark.parametrize("n_exp,topk,n_tok,world,seed", [(8, 2, 500, 2, 7), (128, 8, 300, 8, 1),
                                                         (256, 8, 200, 8, 0), (8, 2, 400, 1, 3),
                                                         (64, 6, 0, 4, 5)])
def test_token_map_and_schedule_bit_exact_vs_reference(n_exp, topk, n_tok, world, seed):
    sel, _ = ORC.sample_routing(n_exp, topk, n_tok, world, seed)
    a = ORC.token_map(sel, n_exp, topk)
    b = REF.token_map(sel, n_exp, topk)
    for x, y in zip(a, b):
        assert (x == y).all()
    epr = n_exp // world
    for r in range(world):
        s1 = ORC.send_schedule(a[0], a[1], a[2], topk, world, epr, r)
        s2 = REF.send_schedule(sel, n_exp, topk, r)
        for x, y in zip(s1, s2):
            assert (x == y).all()


def test_schedule_sorted_by_declared_key():  # test_token_map.cpp:188-206
    for seed in range(10):
        sel, _ = ORC.sample_routing(8, 3, 32, 4, seed)
        tr, le, off, _, _ = ORC.token_map(sel, 8, 3)
        for r in range(4):
            tok, slot, dr, de, do = ORC.send_schedule(tr, le, off, 3, 4, 2, r)
            keys = list(zip(de, dr, do))
            assert keys == sorted(keys) and len(set(keys)) == len(keys)
            assert len(set(zip(tok, slot))) == 96


# ------------------------------------------------------------------ traffic (a21)
def test_traffic_table1_numerators():  # test_traffic.cpp:49-67
    assert ORC.stirling2(8, 5) == 1050 and ORC.stirling2(8, 1) == 1 and ORC.stirling2(0, 0) == 1
    nums, pr, ex, sv = ORC.distinct_rank_distribution(8, 8)
    assert nums == [8, 7112, 324576, 2857680, 7056000, 5362560, 1128960, 40320]
    assert ex == pytest.approx(5.251128673553467, rel=1e-12)
    assert sv == pytest.approx(0.34360891580581665, rel=1e-12)
    assert pr[3] == pytest.approx(0.170, abs=0.005 * 0.170 + 1e-3)


def test_traffic_volumes():  # test_traffic.cpp:90-127
    t = ORC.volume_expected(4096, 8, 4096, 8)
    assert t.v_alltoall == 128 * 1024 * 1024 and t.v_allgather == 128 * 1024 * 1024
    assert t.v_megakernel_nvl / 2 ** 20 == pytest.approx(84.0, rel=0.01)
    t1 = ORC.volume_expected(100, 1, 64, 8)
    assert t1.v_megakernel_nvl == pytest.approx(t1.v_alltoall) and t1.v_megakernel_hbm == pytest.approx(0)
    tw = ORC.volume_expected(100, 4, 64, 1)
    assert tw.v_megakernel_nvl == 0 and tw.v_megakernel_hbm == tw.v_alltoall
    inc = ORC.volume_expected(1024, 8, 64, 8)
    rem = ORC.volume_expected(1024, 8, 64, 8, remote_only=True)
    assert rem.v_megakernel_nvl == pytest.approx(inc.v_megakernel_nvl * 7 / 8)


def test_traffic_exact_forced():  # test_traffic.cpp:110-141
    sel = np.tile(np.arange(8, dtype=np.int32), (8, 1))
    t = ORC.volume_exact(sel, 16, 8, 64)
    assert t.v_megakernel_nvl == pytest.approx(4 * 64) and t.v_megakernel_hbm == pytest.approx(4 * 64)
    sel2 = np.tile(np.array([0, 1], np.int32), (8, 1))
    t2 = ORC.volume_exact(sel2, 16, 2, 64)
    assert t2.v_megakernel_nvl == pytest.approx(64) and t2.v_megakernel_hbm == pytest.approx(64)


@needs_ref
def test_traffic_vs_reference():
    for world in (1, 2, 4, 8):
        for topk in (1, 2, 6, 8, 10):
            a = ORC.distinct_rank_distribution(world, topk)
            b = REF.distinct_rank_distribution(world, topk)
            assert a[0] == b[0] and (a[1] == b[1]).all() and a[2] == b[2] and a[3] == b[3]
            sh = po.make_shape(2048, 768, 128, topk, 4096)
            hw = po.make_hw(148, 1.7e15, 6.5e12, 9e11, world)
            for ro in (False, True):
                x, y = ORC.volume_expected(4096, topk, 4096, world, ro), REF.volume_expected(sh, hw, ro)
                assert (x.v_megakernel_nvl, x.v_megakernel_hbm) == (y.v_megakernel_nvl, y.v_megakernel_hbm)
    sel, _ = ORC.sample_routing(128, 8, 1000, 8, 7)
    sh = po.make_shape(2048, 768, 128, 8, 1000)
    hw = po.make_hw(148, 1.7e15, 6.5e12, 9e11, 8)
    for ro in (False, True):
        x, y = ORC.volume_exact(sel, 128, 8, 4096, ro), REF.volume_exact(sel, sh, hw, ro)
        assert (x.v_megakernel_nvl, x.v_megakernel_hbm) == (y.v_megakernel_nvl, y.v_megakernel_hbm)


# ------------------------------------------------------------------ perf model (a18)
def test_perf_model_frozen_vector():  # test_perf_model.cpp:111-137
    h, s = cluster1(), moe1()
    t = ORC.volume_expected(32768, 6, 4096, 8)
    assert t.v_megakernel_nvl == pytest.approx(591851520.0, rel=1e-12)
    b = ORC.predict_latency(s, h, po.Cfg(12, 5, 20, 33, 32), t)
    assert b.t_up == pytest.approx(3.185631967644085e-05, rel=1e-12)
    assert b.t_down == pytest.approx(2.2526219777553088e-05, rel=1e-12)
    assert (b.n_tiles_up, b.n_tiles_down) == (16896, 12288)
    assert b.l_swiglu == pytest.approx(0.000661072391641791, rel=1e-12)
    assert b.l_disp == pytest.approx(0.008299147936477612, rel=1e-12)
    assert b.l_up == pytest.approx(0.00449174107437816, rel=1e-12)
    assert b.l_s1 == pytest.approx(0.008331004256154052, rel=1e-12)
    assert b.l_comb == pytest.approx(0.00473481216, rel=1e-12)
    assert b.t_red == pytest.approx(0.007692478739104477, rel=1e-12)
    assert b.l_down == pytest.approx(0.0024778841755308395, rel=1e-12)
    assert b.w_gap == pytest.approx(0.25277593426054595, rel=1e-12)
    assert b.w_rem == 0.0
    assert b.l_total == pytest.approx(0.013726888807795844, rel=1e-12)


def test_perf_model_branches():  # test_perf_model.cpp:139-175
    h, s = cluster1(), moe1()
    t = ORC.volume_expected(32768, 6, 4096, 8)
    b = ORC.predict_latency(s, h, po.Cfg(4, 1, 20, 1, 32), t)
    assert b.l_disp >= b.l_up and b.l_s1 == pytest.approx(b.l_disp + b.t_up, rel=1e-15)
    p = ORC.predict_latency(s, h, po.Cfg(64, 5, 20, 33, 32), t)
    r = ORC.predict_latency(s, h, po.Cfg(64, 5, 20, 33, 32), t, redistributed=True)
    assert p.l_s1 == pytest.approx(p.l_disp + (p.l_up - p.l_disp) * 132 / 68)
    assert r.l_s1 == pytest.approx(r.l_disp + (r.l_up - r.l_disp) * 68 / 132)


@needs_ref
def test_perf_model_vs_reference_random_configs():
    rng = np.random.default_rng(0)
    for _ in range(300):
        world = int(rng.choice([1, 2, 4, 8]))
        s = po.make_shape(int(rng.choice([1024, 2048, 4096, 7168])), int(rng.choice([768, 2048, 14336])),
                          int(rng.choice([8, 64, 128, 256])), int(rng.choice([1, 2, 8])),
                          int(rng.integers(1, 70000)))
        h = po.make_hw(148, 1695.7e12, 6468.9e9, 900e9, world)
        t = ORC.volume_expected(s.n_tok, s.topk, s.s_tok, world)
        c = po.Cfg(int(rng.integers(1, 30)) * 4, 1 + 4 * int(rng.integers(0, 5)), int(rng.integers(1, 36)) * 4,
                   int(rng.integers(1, 149)), int(rng.choice([8, 16, 32])))
        if c.n_disp + c.n_relay >= 148 or c.n_comb >= 148:
            continue
        for red in (False, True):
            a = ORC.predict_latency(s, h, c, t, red)
            b = REF.predict_latency(s, h, c, t, red)
            for f, _ in po.Breakdown._fields_:
                assert getattr(a, f) == getattr(b, f), f


# ------------------------------------------------------------------ tuner (a19)
def test_tuner_space_sizes():  # test_tuner.cpp:36-42 ; SURVEY.md §8(a) a19
    assert ORC.space_sizes(132)[0] == 209088
    raw, en, fe = ORC.space_sizes(148)
    assert raw == 332667 and fe == 277992


@needs_ref
def test_tuner_space_and_search_vs_reference():
    for n_sm in (8, 32, 78, 132, 148):
        assert ORC.space_sizes(n_sm) == REF.space_sizes(n_sm)
    h, s = cluster1(), moe1()
    t = ORC.volume_expected(32768, 6, 4096, 8)
    a = ORC.search(s, h, t)
    b = REF.search(s, h, t, workers=4)
    assert a[0].tup() == b[0].tup() and a[1] == b[1] and a[2] == b[2]


# ------------------------------------------------------------------ numerics (a15)
def test_bf16_rne():  # test_precision.cpp:42-51
    assert ORC.round_to_bf16(257.0) == 256.0 and ORC.round_to_bf16(1.0) == 1.0
    assert np.isnan(ORC.round_to_bf16(float("nan")))
    assert np.signbit(ORC.round_to_bf16(-0.0))


def test_fold_order_sensitivity():  # test_precision.cpp:78-107
    one = [1.0, 1.0, 1.0]
    assert ORC.fold(one, [256.0, 1.0, -256.0], True) == 0.0
    assert ORC.fold(one, [256.0, -256.0, 1.0], True) == 1.0
    assert ORC.fold(one, [1.0, 2.0, 4.0], False) == 7.0
    assert ORC.fold([0.5], [257.0], True) == ORC.round_to_bf16(0.5 * 257.0)


@needs_ref
def test_fold_vs_reference():
    rng = np.random.default_rng(3)
    for _ in range(2000):
        n = int(rng.integers(1, 17))
        w = rng.random(n).astype(np.float32)
        v = (rng.standard_normal(n) * 2.0 ** rng.integers(-4, 8, n)).astype(np.float32)
        for b in (0, 1):
            x, y = ORC.fold(w, v, b), REF.fold(w, v, b)
            assert np.float32(x).view(np.uint32) == np.float32(y).view(np.uint32)


# ------------------------------------------------------------------ committed fixtures
def test_golden_fixtures():
    path = os.path.join(GOLDEN, "reference_vectors.npz")
    if not os.path.exists(path):
        pytest.skip("no fixtures committed")
    g = np.load(path)
    sel, gw = ORC.sample_routing(int(g["n_exp"]), int(g["topk"]), int(g["n_tok"]), int(g["world"]),
                                 int(g["seed"]))
    assert (sel == g["sel"]).all() and (gw.view(np.uint32) == g["gw"].view(np.uint32)).all()
    tr, le, off, rt, sb = ORC.token_map(sel, int(g["n_exp"]), int(g["topk"]))
    assert (tr == g["target_rank"]).all() and (le == g["local_expert"]).all()
    assert (off == g["offset"]).all() and (rt == g["recv_totals"]).all() and (sb == g["seg_base"]).all()
    world, epr = int(g["world"]), int(g["n_exp"]) // int(g["world"])
    for r in range(world):
        s = ORC.send_schedule(tr, le, off, int(g["topk"]), world, epr, r)
        assert (s[0] == g[f"sched{r}_token"]).all() and (s[1] == g[f"sched{r}_slot"]).all()


# ------------------------------------------------------------------ router (§8 f1)
def _np_router(lg, k, renorm):
    """Independent float64 restatement: stable top-k (descending, ties -> lower index) + softmax."""
    lg = lg.astype(np.float64)
    T, E = lg.shape
    order = np.lexsort((np.broadcast_to(np.arange(E), lg.shape), -lg), axis=1)[:, :k]
    sel = np.take_along_axis(lg, order, 1)
    m = lg.max(1, keepdims=True)
    num = np.exp(sel - m)
    den = num.sum(1, keepdims=True) if renorm else np.exp(lg - m).sum(1, keepdims=True)
    return order.astype(np.int32), num / den


def _np_weights(lg, ids, renorm):
    m = lg.max()
    num = np.exp(lg[ids] - m)
    return num / (num.sum() if renorm else np.exp(lg - m).sum())


def test_router_exp_portable_accuracy():
    o = po.Oracle()
    o.lib.orc_exp_portable.restype = ctypes.c_float
    o.lib.orc_exp_portable.argtypes = [ctypes.c_float]
    xs = np.concatenate([np.linspace(-86.9, 0.0, 4001), -np.logspace(-8, 1.9, 500)]).astype(np.float32)
    got = np.array([o.lib.orc_exp_portable(float(x)) for x in xs], np.float64)
    ref = np.exp(xs.astype(np.float64))
    assert (np.abs(got - ref) / ref).max() < 3e-7  # about 2.5 ulp
    assert o.lib.orc_exp_portable(0.0) == 1.0 and o.lib.orc_exp_portable(-100.0) == 0.0


@pytest.mark.parametrize("E,k,renorm", [(8, 2, True), (64, 8, True), (256, 8, False), (1000, 16, True),
                                        (7, 7, False), (33, 1, True)])
def test_router_oracle_vs_float64(E, k, renorm):
    rng = np.random.default_rng(E * 31 + k)
    lg = (rng.standard_normal((97, E)) * 3).astype(np.float32)
    lg[5] = np.round(lg[5])          # many ties
    lg[6] = 0.0                      # all equal: ids 0..k-1
    ids, gw = po.Oracle().router_topk(lg, k, renorm)
    rid, rgw = _np_router(lg, k, renorm)
    assert (ids == rid).all()
    assert (ids[6] == np.arange(k)).all()
    assert np.abs(gw - rgw).max() <= 1e-6
    if renorm:
        assert np.abs(gw.astype(np.float64).sum(1) - 1).max() < 1e-5


@pytest.mark.parametrize("renorm", [True, False])
def test_router_bwd_oracle_vs_finite_differences(renorm):
    rng = np.random.default_rng(5)
    T, E, k = 6, 40, 4
    lg = (rng.standard_normal((T, E)) * 2).astype(np.float32)
    ids, gw = po.Oracle().router_topk(lg, k, renorm)
    dg = rng.standard_normal((T, k)).astype(np.float32)
    dl = po.Oracle().router_topk_bwd(lg, ids, gw, dg, renorm)
    h = 1e-6
    for t in range(T):
        l64 = lg[t].astype(np.float64)
        num = np.zeros(E)
        for i in range(E):  # selection fixed (as in autograd through top-k)
            a, b = l64.copy(), l64.copy()
            a[i] += h
            b[i] -= h
            num[i] = (dg[t] @ _np_weights(a, ids[t], renorm) - dg[t] @ _np_weights(b, ids[t], renorm)) / (2 * h)
        assert np.abs(dl[t] - num).max() < 1e-5, (t, np.abs(dl[t] - num).max())
    if renorm:  # experts outside the selection get exactly zero
        mask = np.ones((T, E), bool)
        np.put_along_axis(mask, ids.astype(np.int64), False, 1)
        assert (dl[mask] == 0).all()


def test_router_validation():
    with pytest.raises(ValueError):
        po.Oracle().router_topk(np.zeros((2, 4), np.float32), 5)


def _torch_layer_grads(E, k, H, F, sel, gw, x, w_up, w_down, dy):
    """The layer math written as a plain torch fp32
    autograd graph on the same bf16 inputs: y_t = sum_j w_tj * W_down[e] silu(g) u with
    [g; u] = W_up[e] x_t; loss = <y, dy>."""
    import torch
    f = lambda a: torch.from_numpy((a.astype(np.uint32) << 16).view(np.float32))  # noqa: E731
    X, Wu, Wd, DY = f(x).requires_grad_(), f(w_up).requires_grad_(), f(w_down).requires_grad_(), f(dy)
    G = torch.from_numpy(gw.reshape(-1, k).astype(np.float32)).requires_grad_()
    S = torch.from_numpy(sel.reshape(-1, k).astype(np.int64))
    T = X.shape[0]
    y = torch.zeros(T, H)
    for j in range(k):
        gu = torch.einsum("th,tnh->tn", X, Wu[S[:, j]])
        h = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
        o = torch.einsum("tf,thf->th", h, Wd[S[:, j]])
        y = y + G[:, j:j + 1] * o
    (y * DY).sum().backward()
    return y.detach().numpy(), X.grad.numpy(), G.grad.numpy(), Wu.grad.numpy(), Wd.grad.numpy()


@pytest.mark.parametrize("E,k,H,F,T", [(4, 2, 64, 32, 24), (8, 4, 32, 64, 16)])
def test_oracle_layer_fwd_bwd_pinned_by_torch_autograd(E, k, H, F, T):
    """The oracle's forward AND backward formulas (orc_moe_layer: SwiGLU backward, gate gradient
    <dY, o>, dW_up = dGU^T X, dW_down = dY^T HW, the k-ordered dx) agree with torch.autograd of the
    layer in fp32: the two differ only by the oracle's bf16 rounding of its intermediates (gu, h,
    o, dGU, HW, dX), so the relative L2 error is a few bf16 ulps. A wrong derivative (e.g. a
    missing gate weight or a swapped g/u) is off by O(1)."""
    pytest.importorskip("torch")
    orc = po.Oracle()
    sel, gw = orc.sample_routing(E, k, T, 1, 3)
    x = orc.fill_normal_bf16(T * H, 4).reshape(1, T, H)
    dy = orc.fill_normal_bf16(T * H, 5, 0.5).reshape(1, T, H)
    w_up = orc.fill_normal_bf16(E * 2 * F * H, 6, H ** -0.5).reshape(E, 2 * F, H)
    w_down = orc.fill_normal_bf16(E * H * F, 7, F ** -0.5).reshape(E, H, F)
    ref = orc.moe_layer(1, E, k, H, F, sel, gw, x, w_up, w_down, dy)
    ty, tdx, tdg, tdwu, tdwd = _torch_layer_grads(E, k, H, F, sel, gw, x[0], w_up, w_down, dy[0])
    bf = lambda a: (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    for name, got, want in (("y", bf(ref["y"][0]), ty), ("dx", bf(ref["dx"][0]), tdx),
                            ("dgate", ref["dgate"].reshape(T, k).astype(np.float64), tdg),
                            ("dw_up", bf(ref["dw_up"]), tdwu), ("dw_down", bf(ref["dw_down"]), tdwd)):
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 8e-3, f"{name}: rel L2 {rel:.3g}"


def test_cpu_port_matches_c_oracle():
    """oracle/cpu_port.py (the bench's CPU arm: the same layer contract on CPU BLAS) agrees with the
    C oracle (the checker) within the per-element bounds of tests/parity.py -- only the fp32
    summation order inside the GEMMs differs."""
    pytest.importorskip("torch")
    import torch
    from oracle import cpu_port
    from tests.parity import assert_layer
    E, k, H, F, T = 8, 2, 128, 64, 96
    orc = po.Oracle()
    sel, gw = orc.sample_routing(E, k, T, 1, 9)
    x = orc.fill_normal_bf16(T * H, 1).reshape(1, T, H)
    dy = orc.fill_normal_bf16(T * H, 2, 0.5).reshape(1, T, H)
    w_up = orc.fill_normal_bf16(E * 2 * F * H, 3, H ** -0.5).reshape(E, 2 * F, H)
    w_down = orc.fill_normal_bf16(E * H * F, 4, F ** -0.5).reshape(E, H, F)
    ref = orc.moe_layer(1, E, k, H, F, sel, gw, x, w_up, w_down, dy)
    f = lambda a: torch.from_numpy((a.astype(np.uint32) << 16).view(np.float32))  # noqa: E731
    y, dx, dg, dwu, dwd = cpu_port.moe_layer(sel[0], gw[0], f(x[0]), f(w_up), f(w_down), f(dy[0]), E, k)
    u16 = lambda t: (t.numpy().view(np.uint32) >> 16).astype(np.uint16)  # noqa: E731
    assert_layer(dict(y=u16(y), dx=u16(dx), dgate=dg.numpy(), dw_up=u16(dwu), dw_down=u16(dwd)),
                 {kk: (v[0] if kk in ("y", "dx", "dgate") else v) for kk, v in ref.items()})
