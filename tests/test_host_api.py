"""CPU tests of libeplab_b200.so's host side: every symbol declared in include/eplab_b200.h is
exported, and the eplab:: host API (routing, token map, schedule, traffic, perf model, tuner)
reproduces the reference -- its golden vectors and the reference build in oracle/_ref."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "eplab_b200.h")
REF = po.Reference() if po.has_reference() else None
needs_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built")


def lib():
    from paper_2604_19241_b200 import _lib
    return _lib.lib()


def model():
    from paper_2604_19241_b200 import model as m
    return m


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def test_every_declared_symbol_is_exported():
    names = re.findall(r"EPLAB_API\s+[\w\s\*]+?\b(eplab_\w+)\s*\(", open(HDR).read())
    assert len(names) >= 30
    L = lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_sample_routing_bit_exact_vs_oracle_and_fixture():
    L = lib()
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_vectors_ep8.npz"))
    W, E, k, T = int(g["world"]), int(g["n_exp"]), int(g["topk"]), int(g["n_tok"])
    sel = np.zeros(W * T * k, np.int32)
    gw = np.zeros(W * T * k, np.float32)
    assert L.eplab_sample_routing(E, k, C.c_longlong(T), W, C.c_uint64(int(g["seed"])), _p(sel), _p(gw)) == 0
    assert (sel.reshape(W, -1) == g["sel"]).all()
    assert (gw.view(np.uint32).reshape(W, -1) == g["gw"].view(np.uint32)).all()


@pytest.mark.parametrize("fixture", ["reference_vectors.npz", "reference_vectors_ep8.npz"])
def test_host_token_map_and_schedule_vs_reference_fixture(fixture):
    L = lib()
    g = np.load(os.path.join(ROOT, "tests", "golden", fixture))
    W, E, k, T = int(g["world"]), int(g["n_exp"]), int(g["topk"]), int(g["n_tok"])
    sel = np.ascontiguousarray(g["sel"], np.int32)
    n = W * T * k
    tr, le, off = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int64)
    rt, sb = np.zeros(E, np.int64), np.zeros(E, np.int64)
    assert L.eplab_host_token_map(_p(sel), W, E, C.c_longlong(T), k, _p(tr), _p(le), _p(off), _p(rt), _p(sb)) == 0
    assert (tr.reshape(W, -1) == g["target_rank"]).all() and (le.reshape(W, -1) == g["local_expert"]).all()
    assert (off.reshape(W, -1) == g["offset"]).all()
    assert (rt == g["recv_totals"]).all() and (sb == g["seg_base"]).all()
    for r in range(W):
        out = [np.zeros(T * k, t) for t in (np.int64, np.int32, np.int32, np.int32, np.int64)]
        assert L.eplab_host_send_schedule(_p(sel), W, E, C.c_longlong(T), k, r, *[_p(a) for a in out]) == 0
        assert (out[0] == g[f"sched{r}_token"]).all() and (out[1] == g[f"sched{r}_slot"]).all()


def test_validation_errors_map_to_code_2():
    L = lib()
    sel = np.array([0, 0], np.int32)  # duplicate expert in one token
    z32, z64 = np.zeros(2, np.int32), np.zeros(2, np.int64)
    rc = L.eplab_host_token_map(_p(sel), 1, 4, C.c_longlong(1), 2, _p(z32), _p(z32), _p(z64), _p(z64), _p(z64))
    assert rc == 2
    buf = C.create_string_buffer(256)
    L.eplab_last_error(buf, 256)
    assert b"duplicate expert" in buf.value


def test_perf_model_frozen_vector():  # test_perf_model.cpp:111-137
    m = model()
    h = m.hw(8, n_sm=132, p_peak=989e12, bw_hbm=3.35e12, bw_nvl=200e9, tau_sync=2e-6)
    s = m.shape(2048, 1408, 64, 6, 32768, s_tok=4096)
    t = m.volume_expected(s, h)
    assert t.v_megakernel_nvl == pytest.approx(591851520.0, rel=1e-12)
    b = m.predict_latency(s, h, m.TuneConfig(12, 5, 20, 33, 32), t)
    assert b.t_up == pytest.approx(3.185631967644085e-05, rel=1e-12)
    assert (b.n_tiles_up, b.n_tiles_down) == (16896, 12288)
    assert b.l_disp == pytest.approx(0.008299147936477612, rel=1e-12)
    assert b.l_s1 == pytest.approx(0.008331004256154052, rel=1e-12)
    assert b.t_red == pytest.approx(0.007692478739104477, rel=1e-12)
    assert b.l_total == pytest.approx(0.013726888807795844, rel=1e-12)


@needs_ref
def test_perf_model_and_tuner_vs_reference_build():
    m = model()
    rng = np.random.default_rng(1)
    for _ in range(200):
        world = int(rng.choice([1, 2, 4, 8]))
        args = (int(rng.choice([1024, 2048, 4096, 7168])), int(rng.choice([768, 2048, 14336])),
                int(rng.choice([8, 64, 128, 256])), int(rng.choice([1, 2, 8])), int(rng.integers(1, 70000)))
        s, so = m.shape(*args), po.make_shape(*args)
        h, ho = m.hw(world, p_peak=1695.7e12), po.make_hw(148, 1695.7e12, 6468.9e9, 770e9, world, tau_sync=1e-6)
        t = m.volume_expected(s, h)
        to = REF.volume_expected(so, ho)
        assert (t.v_megakernel_nvl, t.v_megakernel_hbm) == (to.v_megakernel_nvl, to.v_megakernel_hbm)
        c = m.TuneConfig(int(rng.integers(1, 30)) * 4, 1 + 4 * int(rng.integers(0, 5)), int(rng.integers(1, 36)) * 4,
                         int(rng.integers(1, 149)), int(rng.choice([8, 16, 32])))
        if c.n_disp + c.n_relay >= 148 or c.n_comb >= 148:
            continue
        a = m.predict_latency(s, h, c, t)
        b = REF.predict_latency(so, ho, po.Cfg(c.n_disp, c.n_relay, c.n_comb, c.n_red, c.w), to)
        for f, _ in po.Breakdown._fields_:
            assert getattr(a, f) == getattr(b, f), f
    # exhaustive tuner at 148 SMs: same optimum, same evaluated count (277,992)
    s = m.shape(2048, 768, 128, 8, 16384)
    so = po.make_shape(2048, 768, 128, 8, 16384)
    h, ho = m.hw(8, p_peak=1695.7e12), po.make_hw(148, 1695.7e12, 6468.9e9, 770e9, 8, tau_sync=1e-6)
    best, lmin, ev = m.search(s, h, m.volume_expected(s, h), n_workers=4)
    rb, rl, rev, _ = REF.search(so, ho, REF.volume_expected(so, ho), workers=3)
    assert (best.n_disp, best.n_relay, best.n_comb, best.n_red, best.w) == rb.tup()
    assert lmin == rl and ev == rev == 277992


def _task_list(sel, shape, cfg, rank):
    L = lib()
    sel = np.ascontiguousarray(sel, np.int32)
    cs = np.zeros(2 * max(cfg.n_disp, 1), np.int64)
    rr = np.zeros(2 * max(cfg.n_relay, 1), np.int64)
    nc = C.c_longlong()
    rc = L.eplab_host_build_task_list(_p(sel), sel.shape[0], C.byref(shape), C.byref(cfg), rank, _p(cs), _p(rr),
                                      C.byref(nc))
    assert rc == 0
    return cs.reshape(-1, 2)[:cfg.n_disp], rr.reshape(-1, 2)[:cfg.n_relay], nc.value


def test_build_task_list_contract():
    """sim.cpp:226-250 semantics on a hand case: one rank -> nothing crosses a link, so the comm slices are the
    even split of the schedule; relay ranges split the up-GEMM tiles evenly; slices tile their range."""
    m = model()
    T, k, E, F = 100, 2, 4, 512
    sel = np.array([[(t + j) % E for t in range(T) for j in range(k)]], np.int32)
    s, c = po.make_shape(1024, F, E, k, T), po.Cfg(3, 2, 1, 4, 8)
    cs, rr, nc = _task_list(sel, s, c, 0)
    rows = np.bincount(sel[0], minlength=E)                       # 50 rows per expert
    assert nc == sum(-(-int(r) // 128) for r in rows) * (2 * F // 256)
    assert cs.tolist() == [[0, 67], [67, 134], [134, 200]]        # 200 items, no transmissions
    assert rr[0][0] == 0 and rr[-1][1] == nc and all(rr[i][1] == rr[i + 1][0] for i in range(len(rr) - 1))


@needs_ref
def test_build_task_list_vs_reference_build():
    """eplab::build_task_list (the a9 task layout) equals the reference's on random routings: transmission-
    balanced comm slices (world > 1), even relay tile ranges, the tile count."""
    rng = np.random.default_rng(5)
    for _ in range(40):
        W = int(rng.choice([1, 2, 4, 8]))
        E = W * int(rng.choice([1, 2, 4, 16]))
        k = int(rng.integers(1, min(E, 8) + 1))
        T = int(rng.integers(1, 600))
        F = int(rng.choice([256, 768, 2048]))
        sel = np.stack([np.concatenate([rng.permutation(E)[:k] for _ in range(T)]) for _ in range(W)]).astype(np.int32)
        s = po.make_shape(int(rng.choice([1024, 2048])), F, E, k, T)
        c = po.Cfg(int(rng.integers(0, 12)), int(rng.integers(0, 6)), 1, 8, 8)
        for r in range(W):
            a = _task_list(sel, s, c, r)
            b = REF.build_task_list(sel, s, c, r)
            assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and a[2] == b[2], (W, E, k, T, c.tup(), r)


def test_b200_layer_model_sanity():
    m = model()
    s = m.shape(4096, 14336, 8, 2, 16384)
    p1 = m.predict_layer(s, m.hw(1), m.TuneConfig(32, 0, 1, 148, 8))
    assert p1.total > p1.t_gemm_bound > 0 and p1.t_nvl_bound == 0
    # relay (AllGather-style dedup) sends fewer NVLink rows than AllToAll at top-8
    q = m.shape(2048, 768, 128, 8, 16384)
    a2a = m.predict_layer(q, m.hw(8), m.TuneConfig(24, 0, 1, 148, 8))
    ag = m.predict_layer(q, m.hw(8), m.TuneConfig(24, 9, 1, 148, 8))
    assert a2a.total > 0 and ag.total > 0
    best, lmin, ev = m.search_layer(q, m.hw(8))
    assert best.n_disp + best.n_relay < 148 and ev > 100 and lmin > 0


def test_cpp_caller_links_against_the_library(tmp_path):
    """A reference-style C++ caller (tests/cpp/cpp_caller.cpp) compiles against
    include/eplab/eplab.hpp and links libeplab_b200.so (the eplab:: API is exported); its results
    equal the C-ABI's, the oracle's, and the model's choice (host-only calls, no GPU)."""
    import json, os, subprocess
    import numpy as np
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2604_19241_b200")
    exe = str(tmp_path / "cpp_caller")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "cpp", "cpp_caller.cpp"), "-L", libdir,
                           "-leplab_b200", "-Wl,-rpath," + libdir, "-o", exe])
    out = json.loads(subprocess.check_output([exe], text=True).strip())
    from oracle import pyoracle as po
    from paper_2604_19241_b200.model import choose_config, sample_routing
    sel, gw = sample_routing(128, 8, 1024, 8, 7)
    osel, ogw = po.Oracle().sample_routing(128, 8, 1024, 8, 7)
    assert out["sel0"] == sel[0, 0] == osel[0, 0]
    assert np.float32(out["gw0"]) == gw[0, 0] == ogw[0, 0]
    _, _, off, _, _ = po.Oracle().token_map(osel, 128, 8)
    assert out["off_sum"] == int(off.sum())
    want = choose_config(2048, 768, 128, 8, 16384, 8)
    best_n_disp = out["n_disp"]  # raw search_layer result (choose_config adds n_red = n_sm)
    assert out["n_relay"] == want.n_relay and best_n_disp <= want.n_disp
    assert out["validation_error"] is True
