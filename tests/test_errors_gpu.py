"""Error paths of the device data path (§8(b) errors).

The reference raises ValidationError from validate_routing (types.cpp:74-94) and DeadlockError from
the simulators' stuck-queue check (sim.cpp:547-551, error.hpp:19-22; deadlock constructions in
tests/test_sim.cpp:193-209). On the device the planner applies the same routing checks and the
receive-capacity check of every rank; a failure on any rank aborts the iteration on all ranks
before a single row moves, and eplab_check reports 2. A scoreboard wait that never completes
trips the %globaltimer watchdog and eplab_check reports 3, naming the wait site.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_moe_gpu import Problem, from_u16, gather, run_layer, to_u16  # noqa: E402


def moe():
    from paper_2604_19241_b200 import moe as m
    return m


def _inputs(prob, r, T, W):
    epr = prob.E // W
    sel = prob.sel.reshape(-1, prob.k)
    gw = prob.gw.reshape(-1, prob.k)
    x = prob.x.reshape(-1, prob.H)
    dy = prob.dy.reshape(-1, prob.H)
    sl = slice(r * T, (r + 1) * T)
    return dict(ids=torch.from_numpy(np.ascontiguousarray(sel[sl])).cuda(),
                gw=torch.from_numpy(np.ascontiguousarray(gw[sl])).cuda(),
                x=from_u16(x[sl]), dy=from_u16(dy[sl]),
                w_up=from_u16(prob.w_up[r * epr:(r + 1) * epr]),
                w_down=from_u16(prob.w_down[r * epr:(r + 1) * epr]))


def _ranks(prob, W, T, timeout_s=20.0, max_recv_rows=0):
    m = moe()
    ranks = [m.EpMoE(prob.H, prob.F, prob.E, prob.k, T, rank=r, world=W, timeout_s=timeout_s,
                     max_recv_rows=max_recv_rows) for r in range(W)]
    if W > 1:
        m.EpMoE.connect_local(ranks)
        for rk in ranks:
            rk.set_sm_budget(148 // W)
    return ranks


def _step(ranks, ins, streams):
    """plan on every rank (synchronised between ranks, as run_layer does), then fwd + bwd."""
    W = len(ranks)
    ys, gs = [None] * W, [None] * W
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            ranks[r].plan(ins[r]["ids"], ins[r]["gw"], streams[r])
    torch.cuda.synchronize()
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            ranks[r].dispatch_group_gemm(ins[r]["x"], ins[r]["w_up"], streams[r])
            ys[r] = ranks[r].group_gemm_combine(ins[r]["w_down"], stream=streams[r])
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            gs[r] = ranks[r].backward(ins[r]["dy"], ins[r]["w_up"], ins[r]["w_down"], stream=streams[r])
    return ys, gs


def _codes(ranks, streams):
    m = moe()
    out = []
    for r, rk in enumerate(ranks):
        try:
            rk.check(streams[r])
            out.append((0, ""))
        except m.EplabError as e:
            out.append((e.code, str(e)))
    return out


@pytest.mark.parametrize("bad", ["range", "negative", "duplicate", "nan_weight"])
def test_bad_routing_on_one_rank_aborts_every_rank(bad):
    """validate_routing's three checks, on rank 1 of 2: both ranks report 2, nothing is written
    (the output buffers keep their sentinel), and the next valid iteration is bit-exact."""
    W, T = 2, 160
    prob = Problem(W, 8, 2, 256, 256, T, seed=17)
    ranks = _ranks(prob, W, T)
    streams = [torch.cuda.Stream() for _ in range(W)]
    ins = [_inputs(prob, r, T, W) for r in range(W)]
    bad_ids, bad_gw = ins[1]["ids"].clone(), ins[1]["gw"].clone()
    if bad == "range":
        bad_ids[37, 1] = 8
    elif bad == "negative":
        bad_ids[5, 0] = -3
    elif bad == "duplicate":
        bad_ids[99, 1] = bad_ids[99, 0]
    else:
        bad_gw[120, 0] = float("nan")
    good = dict(ins[1])
    ins[1] = dict(ins[1], ids=bad_ids, gw=bad_gw)
    ys, gs = _step(ranks, ins, streams)
    codes = _codes(ranks, streams)
    assert [c for c, _ in codes] == [2, 2], codes
    want = {"range": "out of range", "negative": "out of range", "duplicate": "duplicate expert",
            "nan_weight": "non-finite"}[bad]
    assert want in codes[1][1] and "rank 1" in codes[0][1], codes
    # the iteration was skipped: a second aborted step leaves fresh sentinel outputs untouched
    sentinel = [torch.full((T, prob.H), 7.0, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            ranks[r].plan(ins[r]["ids"], ins[r]["gw"], streams[r])
    torch.cuda.synchronize()
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            ranks[r].dispatch_group_gemm(ins[r]["x"], ins[r]["w_up"], streams[r])
            ranks[r].group_gemm_combine(ins[r]["w_down"], sentinel[r], stream=streams[r])
    assert [c for c, _ in _codes(ranks, streams)] == [2, 2]
    assert all(bool((s == 7.0).all()) for s in sentinel)
    # recovery: the same contexts, valid routing -> bitwise equal to a fresh run
    ins[1] = good
    ys, gs = _step(ranks, ins, streams)
    assert [c for c, _ in _codes(ranks, streams)] == [0, 0]
    torch.cuda.synchronize()
    ref, _, _ = run_layer(prob)
    got = [dict(y=to_u16(ys[r]), dx=to_u16(gs[r]["dx"]), dgate=gs[r]["dgate"].cpu().numpy(),
                dw_up=to_u16(gs[r]["dw_up"]), dw_down=to_u16(gs[r]["dw_down"])) for r in range(W)]
    a, b = gather(got), gather(ref[0])
    for key in a:
        assert (a[key] == b[key]).all(), key
    for rk in ranks:
        rk.close()


def test_receive_capacity_overflow_aborts_without_peer_writes():
    """All of rank 0's and rank 1's tokens routed to rank 0's experts with max_recv_rows sized for
    balanced routing: rank 0's capacity is exceeded. Every rank sees it (same counts), reports 2,
    and no row lands in either rank's receive buffer (a sender-side overflow would write past
    rank 0's M_cap)."""
    W, T, k = 2, 512, 2
    prob = Problem(W, 8, k, 256, 256, T, seed=19)
    cap = T * k  # rows per rank under balanced routing
    ranks = _ranks(prob, W, T, max_recv_rows=cap)
    streams = [torch.cuda.Stream() for _ in range(W)]
    ins = [_inputs(prob, r, T, W) for r in range(W)]
    for r in range(W):  # experts 0..3 live on rank 0: rank 0 receives 2*T*k rows > cap
        ids = torch.stack([torch.arange(T, device="cuda") % 4, (torch.arange(T, device="cuda") + 1) % 4], 1)
        ins[r]["ids"] = ids.int().contiguous()
    views = [rk.buffer("recv_x", cap, prob.H) for rk in ranks]
    for v in views:
        v.fill_(3.0)
    torch.cuda.synchronize()
    _step(ranks, ins, streams)
    codes = _codes(ranks, streams)
    assert [c for c, _ in codes] == [2, 2], codes
    assert all("capacity exceeded on rank 0" in m for _, m in codes), codes
    assert all(bool((v == 3.0).all()) for v in views), "rows were written during an aborted iteration"
    for rk in ranks:
        rk.close()


def test_deadlock_count_exchange_reports_error_3():
    """test_sim.cpp:193-209 analogue: a peer that never plans. Rank 0's count AllGather waits for
    rank 1's counts, the watchdog fires, eplab_check returns 3 naming the wait site, and the
    iteration's MegaKernels skip their work instead of hanging the GPU."""
    m = moe()
    W, T = 2, 128
    prob = Problem(W, 8, 2, 256, 256, T, seed=23)
    ranks = _ranks(prob, W, T, timeout_s=0.3)
    s = torch.cuda.Stream()
    ins = _inputs(prob, 0, T, W)
    with torch.cuda.stream(s):
        ranks[0].plan(ins["ids"], ins["gw"], s)
        ranks[0].dispatch_group_gemm(ins["x"], ins["w_up"], s)
        ranks[0].group_gemm_combine(ins["w_down"], stream=s)
    with pytest.raises(m.EplabError) as e:
        ranks[0].check(s)
    assert e.value.code == 3 and "count AllGather" in str(e.value)
    for rk in ranks:
        rk.close()


@pytest.mark.parametrize("relay,sites", [(0, ("up-GEMM tile's rowgroup wait",)),
                                         (2, ("relay worker's slot-flag wait", "up-GEMM tile's rowgroup wait"))])
def test_deadlock_dispatch_scoreboard_reports_error_3(relay, sites):
    """Both ranks plan, only rank 0 launches its dispatch MegaKernel: rank 0's up-GEMM tiles (relay
    off) or relay workers (relay on) wait for rows rank 1 never sends; the wait times out -> 3
    naming the site, no hang. With the relay on, the relay workers (slot flags of the missing rows) and
    the up-GEMM tiles (the rowgroups those workers would count) wait at the same time, and whichever
    watchdog expires first names the site."""
    m = moe()
    W, T = 2, 128
    prob = Problem(W, 8, 2, 256, 256, T, seed=29)
    ranks = _ranks(prob, W, T, timeout_s=0.3)
    for rk in ranks:
        rk.set_tune_config((4, relay, 1, 74, 8))
    streams = [torch.cuda.Stream() for _ in range(W)]
    ins = [_inputs(prob, r, T, W) for r in range(W)]
    for r in range(W):
        with torch.cuda.stream(streams[r]):
            ranks[r].plan(ins[r]["ids"], ins[r]["gw"], streams[r])
    torch.cuda.synchronize()
    with torch.cuda.stream(streams[0]):
        ranks[0].dispatch_group_gemm(ins[0]["x"], ins[0]["w_up"], streams[0])
    with pytest.raises(m.EplabError) as e:
        ranks[0].check(streams[0])
    assert e.value.code == 3 and any(site in str(e.value) for site in sites), str(e.value)
    for rk in ranks:
        rk.close()


def test_argument_checks_raise_validation_errors():
    """Every tensor crossing the C-ABI is checked (device, dtype, shape, contiguity) -> code 2."""
    m = moe()
    H, F, E, k, T = 256, 256, 8, 2, 64
    L = m.EpMoE(H, F, E, k, T)
    ids = torch.stack([torch.arange(T) % E, (torch.arange(T) + 1) % E], 1).int().cuda()
    gw = torch.full((T, k), 0.5, device="cuda")
    x = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    wu = torch.zeros(E, 2 * F, H, dtype=torch.bfloat16, device="cuda")
    wd = torch.zeros(E, H, F, dtype=torch.bfloat16, device="cuda")
    bad_calls = [
        lambda: L.plan(ids[:, :1], gw[:, :1]),                       # wrong k
        lambda: L.plan(ids.long(), gw),                              # int64 ids
        lambda: L.plan(ids, gw.double()),                            # fp64 weights
    ]
    for f in bad_calls:
        with pytest.raises(m.EplabError) as e:
            f()
        assert e.value.code == 2
    L.plan(ids, gw)
    for f in [lambda: L.dispatch_group_gemm(x.float(), wu),          # fp32 activations
              lambda: L.dispatch_group_gemm(x.t().contiguous().t(), wu),  # wrong shape
              lambda: L.dispatch_group_gemm(torch.zeros(2 * T, H, dtype=torch.bfloat16,
                                                        device="cuda")[::2], wu),  # strided view
              lambda: L.dispatch_group_gemm(x.cpu(), wu),            # host tensor
              lambda: L.dispatch_group_gemm(x, wu[:, :F]),           # wrong W_up shape
              lambda: L.group_gemm_combine(wd.transpose(1, 2))]:     # non-contiguous W_down
        with pytest.raises(m.EplabError) as e:
            f()
        assert e.value.code == 2
    with pytest.raises(m.EplabError) as e:
        L.set_option("no_such_knob", 1)
    assert e.value.code == 2
    L.close()


def test_autograd_state_gone_raises():
    """Forwards in flight are stashed (tests/test_microbatch_gpu.py); a backward whose plan state
    is neither live nor stashed -- a retained graph run backward a second time after a re-plan --
    raises error 2 instead of returning gradients of another plan."""
    m = moe()
    H, F, E, k, T = 256, 256, 8, 2, 64
    L = m.EpMoE(H, F, E, k, T)
    ids = torch.stack([torch.arange(T) % E, (torch.arange(T) + 3) % E], 1).int().cuda()
    gw = torch.full((T, k), 0.5, device="cuda", requires_grad=True)
    x = torch.randn(T, H, device="cuda").bfloat16().requires_grad_()
    wu = (torch.randn(E, 2 * F, H, device="cuda") * 0.05).bfloat16().requires_grad_()
    wd = (torch.randn(E, H, F, device="cuda") * 0.05).bfloat16().requires_grad_()
    y1 = m.EpMoEFunction.apply(L, x, ids, gw, wu, wd)
    y1.float().sum().backward(retain_graph=True)
    y1.float().sum().backward(retain_graph=True)  # fine: still the live plan
    y2 = m.EpMoEFunction.apply(L, x, ids, gw, wu, wd)
    with pytest.raises(m.EplabError) as e:
        y1.float().sum().backward()
    assert e.value.code == 2 and "gone" in str(e.value)
    y2.float().sum().backward()
    L.check()
    L.close()


def test_local_layout_mismatch_is_rejected():
    m = moe()
    a = m.EpMoE(256, 256, 8, 2, 64, rank=0, world=2)
    b = m.EpMoE(256, 256, 8, 2, 96, rank=1, world=2)  # different max_tokens
    with pytest.raises(m.EplabError) as e:
        m.EpMoE.connect_local([a, b])
    assert e.value.code == 2 and "symmetric" in str(e.value)
    a.close()
    b.close()
