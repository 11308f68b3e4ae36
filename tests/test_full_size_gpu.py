"""Parity at BASELINE.json's full sizes (Mixtral-8x7B, Qwen3-30B-A3B and DeepSeek-V3 layer shapes,
16K tokens, EP=1), where the oracle cannot run the whole layer: size-independent checks.

* the device token map (permutation indices, per-expert counts, segment bases) is bit-exact with
  the C oracle's restatement of build_global_token_map on all 16K x k routing entries;
* the whole fwd+bwd step is bitwise deterministic (two runs, every output);
* y, dx and dgate are row-local: for a sample of tokens the oracle computes them from those
  tokens alone (with every expert's weights), per-element within 1 bf16 ulp (tests/parity.py);
* the weight gradients, all of them, against fp32 GEMMs (torch, TF32 off) of the device's own
  exported expert buffers: dW_up[e] = dGU_e^T X_e, dW_down[e] = dY_e^T HW_e (the oracle's
  definition), per-element within 1 bf16 ulp;
* the weight gradients satisfy a linearity property: scaling dY by 2 (exact in bf16) scales
  dW_up / dW_down by exactly 2 (power-of-two scaling commutes with every rounding on the path).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pyoracle as po  # noqa: E402
from tests.parity import assert_ulp  # noqa: E402
from tests.test_moe_gpu import bf16_to_f32, to_u16  # noqa: E402

SHAPES = {"mixtral": (4096, 14336, 8, 2, 16384), "qwen3": (2048, 768, 128, 8, 16384),
          "dsv3": (7168, 2048, 256, 8, 16384)}


def _dw_vs_fp32(layer, a, H, F, E):
    """Every expert's weight gradients vs fp32 GEMMs of the exported expert buffers (one expert at a
    time: DSv3's 11G weight-gradient elements would not fit as fp32 references at once)."""
    sb, rows = layer.export_layout()
    used = int(max(s + ((r + 127) // 128) * 128 for s, r in zip(sb, rows)))
    xs, dys = layer.buffer("recv_x", used, H), layer.buffer("recv_dy", used, H)
    dgu, hw = layer.buffer("dgu", used, 2 * F), layer.buffer("hw", used, F)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    got_u, ref_u, got_d, ref_d = [], [], [], []
    try:
        for e in range(E):
            s, r = int(sb[e]), int(rows[e])
            up = dgu[s:s + r].float().t() @ xs[s:s + r].float()
            down = dys[s:s + r].float().t() @ hw[s:s + r].float()
            # a deterministic sample of 2^16 elements per expert keeps the host side small
            g = torch.Generator(device="cuda").manual_seed(e)
            iu = torch.randint(0, up.numel(), (1 << 16,), device="cuda", generator=g)
            idn = torch.randint(0, down.numel(), (1 << 16,), device="cuda", generator=g)
            got_u.append(a["dw_up"][e].reshape(-1)[iu].float())
            ref_u.append(up.reshape(-1)[iu].bfloat16().float())  # the one rounding of the output
            got_d.append(a["dw_down"][e].reshape(-1)[idn].float())
            ref_d.append(down.reshape(-1)[idn].bfloat16().float())
            del up, down
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    assert_ulp(torch.cat(got_u).cpu().numpy(), torch.cat(ref_u).cpu().numpy(), "dw_up", "exact_inputs")
    assert_ulp(torch.cat(got_d).cpu().numpy(), torch.cat(ref_d).cpu().numpy(), "dw_down", "exact_inputs")


@pytest.mark.parametrize("cfg", sorted(SHAPES))
def test_full_size_parity(cfg):
    from paper_2604_19241_b200 import moe as M
    from paper_2604_19241_b200.model import sample_routing
    H, F, E, k, T = SHAPES[cfg]
    sel, gw = sample_routing(E, k, T, 1, 7)
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(T, H, device="cuda", generator=g) * 0.5).bfloat16()
    w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    ids = torch.from_numpy(sel[0].reshape(T, k).copy()).cuda()
    gws = torch.from_numpy(gw[0].reshape(T, k).copy()).cuda()
    layer = M.EpMoE(H, F, E, k, T)
    try:
        _full_size_checks(layer, H, F, E, k, T, sel, gw, x, dy, w_up, w_down, ids, gws)
    finally:
        layer.close()
        torch.cuda.empty_cache()


def _full_size_checks(layer, H, F, E, k, T, sel, gw, x, dy, w_up, w_down, ids, gws):
    def step(dy_):
        y = layer.forward(x, ids, gws, w_up, w_down)
        gr = layer.backward(dy_, w_up, w_down)
        layer.check()
        torch.cuda.synchronize()
        return dict(y=y, **gr)

    a = step(dy)
    tr, le, off, rt, sb = layer.export_token_map()
    _dw_vs_fp32(layer, a, H, F, E)
    b = step(dy)
    for key in ("y", "dx", "dgate", "dw_up", "dw_down"):
        assert torch.equal(a[key], b[key]), f"run-to-run {key}"
    # integer addressing: bit-exact at full size
    otr, ole, ooff, ort, osb = po.Oracle().token_map(sel, E, k)
    assert (tr == otr).all() and (le == ole).all() and (off == ooff).all()
    assert (rt == ort).all() and (sb == osb).all()
    # linearity of the weight gradients in dY (x2 is exact in bf16 and commutes with rounding)
    c = step((dy.float() * 2).bfloat16())
    for key in ("dw_up", "dw_down"):
        for e in range(E):  # per expert: DSv3's dW in fp32 would be 30 GB
            assert torch.equal(c[key][e].float(), a[key][e].float() * 2), f"{key}(2 dY) != 2 {key}(dY), expert {e}"
    del c
    # row-local outputs of sampled tokens vs the oracle
    toks = np.array([0, 1, 77, T // 3, T // 2, T - 2, T - 1])
    ref = po.Oracle().moe_layer(1, E, k, H, F, sel.reshape(T, k)[toks].reshape(1, -1),
                                gw.reshape(T, k)[toks].reshape(1, -1), to_u16(x[toks]).reshape(1, -1, H),
                                to_u16(w_up), to_u16(w_down), to_u16(dy[toks]).reshape(1, -1, H), want_dw=False)
    assert_ulp(bf16_to_f32(to_u16(a["y"][toks])).reshape(-1), bf16_to_f32(ref["y"]).reshape(-1), "y", "act_longk")
    assert_ulp(bf16_to_f32(to_u16(a["dx"][toks])).reshape(-1), bf16_to_f32(ref["dx"]).reshape(-1), "dx", "act_longk")
    assert_ulp(a["dgate"][toks].cpu().numpy().reshape(-1), ref["dgate"].reshape(-1), "dgate", "dgate")


def _world_invariance(cfg, W, T, relay, n_disp=4, seed=3):
    """cfg's layer with T tokens per rank on W virtual ranks (one process, 148/W SMs each, peer rows
    through the same symmetric buffers the NVLink path uses) == EP=1 on the same W*T tokens, bit for bit:
    y, dx, dgate, dW_up, dW_down."""
    from paper_2604_19241_b200 import moe as M
    from paper_2604_19241_b200.model import sample_routing
    H, F, E, k, _ = SHAPES[cfg]
    sel, gw = sample_routing(E, k, T, W, seed)  # [W][T*k]: rank r's tokens are global tokens r*T..
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(W * T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(W * T, H, device="cuda", generator=g) * 0.5).bfloat16()
    w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    ids = torch.from_numpy(sel.reshape(W * T, k).copy()).cuda()
    gws = torch.from_numpy(gw.reshape(W * T, k).copy()).cuda()
    # EP=1 over all W*T tokens
    one = M.EpMoE(H, F, E, k, W * T, max_recv_rows=W * T * k)
    y1 = one.forward(x, ids, gws, w_up, w_down)
    g1 = one.backward(dy, w_up, w_down)
    one.check()
    torch.cuda.synchronize()
    one.close()
    # EP=W: E/W experts and T tokens per virtual rank (receive capacity for balanced routing + slack)
    epr = E // W
    ranks = [M.EpMoE(H, F, E, k, T, rank=r, world=W, max_recv_rows=T * k * 5 // 4 + 128 * epr, timeout_s=60.0)
             for r in range(W)]
    M.EpMoE.connect_local(ranks)
    for r in ranks:
        r.set_sm_budget(148 // W)
        r.set_tune_config((n_disp, relay, 1, 148 // W, 8))
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
                    gs[r] = ranks[r].backward(dy[sl], w_up[r * epr:(r + 1) * epr],
                                              w_down[r * epr:(r + 1) * epr], stream=streams[r])
        if ph == 0:
            torch.cuda.synchronize()
    for r in range(W):
        ranks[r].check(streams[r])
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(ys), y1), "y"
    assert torch.equal(torch.cat([gg["dx"] for gg in gs]), g1["dx"]), "dx"
    assert torch.equal(torch.cat([gg["dgate"] for gg in gs]), g1["dgate"]), "dgate"
    assert torch.equal(torch.cat([gg["dw_up"] for gg in gs]), g1["dw_up"]), "dw_up"
    assert torch.equal(torch.cat([gg["dw_down"] for gg in gs]), g1["dw_down"]), "dw_down"
    for r in ranks:
        r.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("relay", [0, 4])
def test_world_invariance_full_size_qwen3_ep8(relay):
    """Qwen3 shape (128 experts, top-8, H 2048, F 768) with 16K tokens per rank on 8 virtual ranks equals
    EP=1 on the same 131K tokens bit for bit, with the AllToAll-style (relay off) and AllGather-style
    (relay on) dispatch."""
    _world_invariance("qwen3", 8, SHAPES["qwen3"][4], relay)


@pytest.mark.parametrize("W,T,relay", [(2, 16384, 0), (8, 4096, 0), (8, 4096, 2)])
def test_world_invariance_mixtral(W, T, relay):
    """The bench's Mixtral shape (8 experts top-2, H 4096, F 14336): 16K tokens per rank at EP=2, and 4K
    tokens per rank at EP=8 (one expert per rank, relay off and on) equal EP=1 on the same tokens bit for
    bit -- the GPU-count invariance of the headline configuration."""
    _world_invariance("mixtral", W, T, relay)


def test_small_config_ep2_full_size():
    """BASELINE configs[0] at its stated size (8 experts top-2, H 1024, F 2048, 4096 tokens per rank,
    EP=2 on two virtual ranks): equal to EP=1 on the same 8192 tokens bit for bit, and sampled tokens'
    y / dx / dgate equal the oracle run on those tokens alone."""
    from paper_2604_19241_b200 import moe as M
    from paper_2604_19241_b200.model import sample_routing
    H, F, E, k, T, W = 1024, 2048, 8, 2, 4096, 2
    sel, gw = sample_routing(E, k, T, W, 7)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(W * T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(W * T, H, device="cuda", generator=g) * 0.5).bfloat16()
    w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    ids = torch.from_numpy(sel.reshape(W * T, k).copy()).cuda()
    gws = torch.from_numpy(gw.reshape(W * T, k).copy()).cuda()
    one = M.EpMoE(H, F, E, k, W * T)
    y1 = one.forward(x, ids, gws, w_up, w_down)
    g1 = one.backward(dy, w_up, w_down)
    one.check()
    torch.cuda.synchronize()
    one.close()
    epr = E // W
    ranks = [M.EpMoE(H, F, E, k, T, rank=r, world=W, timeout_s=60.0) for r in range(W)]
    M.EpMoE.connect_local(ranks)
    for r in ranks:
        r.set_sm_budget(148 // W)
    streams = [torch.cuda.Stream() for _ in range(W)]
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
    assert torch.equal(torch.cat(ys), y1)
    for key in ("dx", "dgate", "dw_up", "dw_down"):
        assert torch.equal(torch.cat([gg[key] for gg in gs]), g1[key]), key
    toks = np.array([0, 5, T - 1, T, W * T - 1])
    ref = po.Oracle().moe_layer(1, E, k, H, F, sel.reshape(W * T, k)[toks].reshape(1, -1),
                                gw.reshape(W * T, k)[toks].reshape(1, -1), to_u16(x[toks]).reshape(1, -1, H),
                                to_u16(w_up), to_u16(w_down), to_u16(dy[toks]).reshape(1, -1, H), want_dw=False)
    assert_ulp(bf16_to_f32(to_u16(y1[toks])).reshape(-1), bf16_to_f32(ref["y"]).reshape(-1), "y", "act_longk")
    assert_ulp(bf16_to_f32(to_u16(g1["dx"][toks])).reshape(-1), bf16_to_f32(ref["dx"]).reshape(-1), "dx", "act_longk")
    assert_ulp(g1["dgate"][toks].cpu().numpy().reshape(-1), ref["dgate"].reshape(-1), "dgate", "dgate")
    for r in ranks:
        r.close()
