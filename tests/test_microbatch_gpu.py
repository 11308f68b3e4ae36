"""Several forwards in flight on one context (VERDICT r1 "autograd safety": pipelined micro-batches,
layers sharing a context, activation recomputation).

A context holds one iteration's state; a later plan stashes it when an autograd backward still
needs it (EpMoE._evict -> eplab_stash_save, sized to the actual receive rows, not the worst-case
capacity) and that backward restores it (eplab_stash_restore). Every micro-batch's y, dx, dgate,
dW_up and dW_down must be BITWISE equal to the same micro-batch run alone (plan -> fwd -> bwd), in
every backward order: FIFO, LIFO and 1F1B. At EP = 2 (virtual ranks) the explicit stash / restore
API is driven the same way on both ranks.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_moe_gpu import Problem, from_u16, to_u16  # noqa: E402


def moe():
    from paper_2604_19241_b200 import moe as m
    return m


H, F, E, K, T = 256, 512, 8, 2, 384
ORDERS = {
    "fifo": ["F0", "F1", "F2", "B0", "B1", "B2"],
    "lifo": ["F0", "F1", "F2", "B2", "B1", "B0"],
    "1f1b": ["F0", "F1", "B0", "F2", "B1", "B2"],
}


def _micro(i, world=1):
    p = Problem(world, E, K, H, F, T, seed=11 + 5 * i)
    return p


def _leaf_inputs(p, r=0, W=1):
    epr = E // W
    return dict(ids=torch.from_numpy(np.ascontiguousarray(p.sel[r].reshape(T, K))).cuda(),
                gw=torch.from_numpy(np.ascontiguousarray(p.gw[r].reshape(T, K))).cuda(),
                x=from_u16(p.x[r]), dy=from_u16(p.dy[r]),
                w_up=from_u16(p.w_up[r * epr:(r + 1) * epr]), w_down=from_u16(p.w_down[r * epr:(r + 1) * epr]))


def _autograd_fwd(m, L, a):
    leaves = dict(x=a["x"].clone().requires_grad_(), gw=a["gw"].clone().requires_grad_(),
                  w_up=a["w_up"].clone().requires_grad_(), w_down=a["w_down"].clone().requires_grad_())
    y = m.EpMoEFunction.apply(L, leaves["x"], a["ids"], leaves["gw"], leaves["w_up"], leaves["w_down"])
    return y, leaves


def _grads(y, leaves):
    return dict(y=to_u16(y), dx=to_u16(leaves["x"].grad), dgate=leaves["gw"].grad.cpu().numpy(),
                dw_up=to_u16(leaves["w_up"].grad), dw_down=to_u16(leaves["w_down"].grad))


def _assert_same(got, ref, what):
    for key in ref:
        assert np.array_equal(got[key], ref[key]), f"{what}: {key} differs from the micro-batch run alone"


@pytest.mark.parametrize("order", sorted(ORDERS))
def test_autograd_microbatches_bitwise(order):
    m = moe()
    L = m.EpMoE(H, F, E, K, T)
    ins = [_leaf_inputs(_micro(i)) for i in range(3)]
    alone = []
    for a in ins:  # each micro-batch alone: plan -> fwd -> bwd
        y, lv = _autograd_fwd(m, L, a)
        y.backward(a["dy"])
        alone.append(_grads(y, lv))
    assert not L._stashes and not L._pending
    live = {}
    for op in ORDERS[order]:
        i = int(op[1])
        if op[0] == "F":
            live[i] = _autograd_fwd(m, L, ins[i])
        else:
            y, lv = live.pop(i)
            y.backward(ins[i]["dy"])
            _assert_same(_grads(y, lv), alone[i], f"{order} micro-batch {i}")
    assert not L._stashes and not L._pending
    L.check()
    L.close()


def test_freed_graph_drops_its_stash():
    """A forward whose graph is freed without a backward (evaluation under grad mode) must not
    keep its stash alive."""
    m = moe()
    L = m.EpMoE(H, F, E, K, T)
    a = _leaf_inputs(_micro(0))
    y0, _ = _autograd_fwd(m, L, a)
    y1, lv1 = _autograd_fwd(m, L, a)  # stashes micro-batch 0
    assert len(L._stashes) == 1 and L._stashes[min(L._stashes)].nbytes > 0
    del y0
    y2, lv2 = _autograd_fwd(m, L, a)  # stashes 1; 0's graph is gone -> its stash is dropped
    assert sorted(L._stashes) == [L.plan_epoch - 1]
    y2.backward(a["dy"])
    y1.backward(a["dy"])
    assert np.array_equal(to_u16(lv1["x"].grad), to_u16(lv2["x"].grad))
    assert not L._stashes
    L.close()


def test_stash_size_tracks_receive_rows():
    """The stash is sized to the iteration's receive rows, not the context's capacity."""
    m = moe()
    L = m.EpMoE(H, F, E, K, 4 * T)
    a = _leaf_inputs(_micro(0))
    L.plan(a["ids"], a["gw"])
    L.dispatch_group_gemm(a["x"], a["w_up"])
    small = L.stash().nbytes
    big_ids = torch.cat([a["ids"]] * 4)
    L.plan(big_ids, torch.cat([a["gw"]] * 4))
    L.dispatch_group_gemm(torch.cat([a["x"]] * 4), a["w_up"])
    big = L.stash().nbytes
    assert 3 * small < big < 5 * small
    L.close()


def test_restore_into_other_shape_rejected():
    m = moe()
    L = m.EpMoE(H, F, E, K, T)
    L2 = m.EpMoE(H, 2 * F, E, K, T)
    a = _leaf_inputs(_micro(0))
    L.plan(a["ids"], a["gw"])
    st = L.stash()
    with pytest.raises(m.EplabError) as e:
        L2.restore(st)
    assert e.value.code == 2
    L.close()
    L2.close()


@pytest.mark.parametrize("order", ["lifo", "1f1b"])
@pytest.mark.parametrize("relay", [0, 1])
def test_virtual_ep2_stash_restore_bitwise(order, relay):
    """EP = 2 on virtual ranks: both ranks stash before a later plan and restore before the
    backward, in the same order; results equal each micro-batch run alone, bitwise."""
    m = moe()
    W = 2
    cfg = m.TuneConfig(4, relay, 1, 148 // W, 8)
    ranks = [m.EpMoE(H, F, E, K, T, rank=r, world=W, timeout_s=20.0) for r in range(W)]
    m.EpMoE.connect_local(ranks)
    for rk in ranks:
        rk.set_sm_budget(148 // W)
        rk.set_tune_config(cfg)
    streams = [torch.cuda.Stream() for _ in range(W)]
    probs = [_micro(i, W) for i in range(3)]
    ins = [[_leaf_inputs(p, r, W) for r in range(W)] for p in probs]

    def fwd(i):
        ys = []
        for r in range(W):
            with torch.cuda.stream(streams[r]):
                ranks[r].plan(ins[i][r]["ids"], ins[i][r]["gw"], streams[r])
        torch.cuda.synchronize()
        for r in range(W):
            with torch.cuda.stream(streams[r]):
                ranks[r].dispatch_group_gemm(ins[i][r]["x"], ins[i][r]["w_up"], streams[r])
                ys.append(ranks[r].group_gemm_combine(ins[i][r]["w_down"], stream=streams[r]))
        torch.cuda.synchronize()
        return ys

    def bwd(i):
        gs = []
        for r in range(W):
            with torch.cuda.stream(streams[r]):
                a = ins[i][r]
                gs.append(ranks[r].backward(a["dy"], a["w_up"], a["w_down"], stream=streams[r]))
        torch.cuda.synchronize()
        return gs

    def outs(ys, gs):
        return [dict(y=to_u16(ys[r]), dx=to_u16(gs[r]["dx"]), dgate=gs[r]["dgate"].cpu().numpy(),
                     dw_up=to_u16(gs[r]["dw_up"]), dw_down=to_u16(gs[r]["dw_down"])) for r in range(W)]

    alone = [outs(fwd(i), bwd(i)) for i in range(3)]
    stashes, ys, live = {}, {}, None
    for op in ORDERS[order]:
        i = int(op[1])
        if live is not None and live not in stashes:
            torch.cuda.synchronize()
            stashes[live] = [rk.stash(streams[r]) for r, rk in enumerate(ranks)]
        if op[0] == "F":
            ys[i] = fwd(i)
            live = i
        else:
            if live != i:
                for r, rk in enumerate(ranks):
                    with torch.cuda.stream(streams[r]):
                        rk.restore(stashes[i][r], streams[r])
                live = i
            got = outs(ys.pop(i), bwd(i))
            stashes.pop(i, None)
            live = None  # consumed
            for r in range(W):
                for key in got[r]:
                    assert np.array_equal(got[r][key], alone[i][r][key]), \
                        f"{order} relay={relay} micro-batch {i} rank {r}: {key}"
    for r, rk in enumerate(ranks):
        rk.check(streams[r])
        rk.close()
