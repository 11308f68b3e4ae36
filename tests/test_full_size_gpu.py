"""Parity at BASELINE.json's full sizes (Mixtral-8x7B and Qwen3-30B-A3B layer shapes, 16K tokens,
EP=1), where the oracle cannot run the whole layer: size-independent checks.

* the device token map (permutation indices, per-expert counts, segment bases) is bit-exact with
  the C oracle's restatement of build_global_token_map on all 16K x k routing entries;
* the whole fwd+bwd step is bitwise deterministic (two runs, every output);
* y, dx and dgate are row-local: for a sample of tokens the oracle computes them from those
  tokens alone (with every expert's weights), within the tolerance of tests/test_moe_gpu.py;
* the weight gradients satisfy a linearity property: scaling dY by 2 (exact in bf16) scales
  dW_up / dW_down by exactly 2 (power-of-two scaling commutes with every rounding on the path).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pyoracle as po  # noqa: E402
from tests.test_moe_gpu import assert_close, bf16_to_f32, to_u16  # noqa: E402

SHAPES = {"mixtral": (4096, 14336, 8, 2, 16384), "qwen3": (2048, 768, 128, 8, 16384)}


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

    def step(dy_):
        y = layer.forward(x, ids, gws, w_up, w_down)
        gr = layer.backward(dy_, w_up, w_down)
        layer.check()
        torch.cuda.synchronize()
        return dict(y=y, **gr)

    a = step(dy)
    tr, le, off, rt, sb = layer.export_token_map()
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
        assert torch.equal(c[key].float(), a[key].float() * 2), f"{key}(2 dY) != 2 {key}(dY)"
    # row-local outputs of sampled tokens vs the oracle
    toks = np.array([0, 1, T // 3, T // 2, T - 2, T - 1])
    ref = po.Oracle().moe_layer(1, E, k, H, F, sel.reshape(T, k)[toks].reshape(1, -1),
                                gw.reshape(T, k)[toks].reshape(1, -1), to_u16(x[toks]).reshape(1, -1, H),
                                to_u16(w_up), to_u16(w_down), to_u16(dy[toks]).reshape(1, -1, H))
    assert_close(bf16_to_f32(to_u16(a["y"][toks])).reshape(-1), bf16_to_f32(ref["y"]).reshape(-1), "y")
    assert_close(bf16_to_f32(to_u16(a["dx"][toks])).reshape(-1), bf16_to_f32(ref["dx"]).reshape(-1), "dx")
    assert_close(a["dgate"][toks].cpu().numpy().reshape(-1), ref["dgate"].reshape(-1), "dgate")
    layer.close()
