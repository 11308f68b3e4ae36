"""GPU parity of the router kernels (csrc/kernels/router.cu) against the CPU
oracle (oracle/eplab_oracle.c orc_router_topk*): bit-exact ids, weights and logit gradients."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import pyoracle as po  # noqa: E402


def moe():
    from paper_2604_19241_b200 import moe as m
    return m


def logits_for(T, E, seed):
    rng = np.random.default_rng(seed)
    lg = (rng.standard_normal((T, E)) * 3).astype(np.float32)
    if T > 8:
        lg[3] = np.round(lg[3])      # ties
        lg[4] = 0.0                  # all equal
        lg[5, : min(E, 3)] = -np.inf  # masked experts
        lg[6] = -200.0 + lg[6]       # exp underflow of everything but the max
    return lg


@pytest.mark.parametrize("E,k", [(8, 2), (64, 8), (128, 8), (256, 8), (1000, 16), (1024, 32), (5, 5)])
@pytest.mark.parametrize("renorm", [True, False])
def test_router_fwd_bwd_bit_exact(E, k, renorm):
    m = moe()
    T = 1037
    lg = logits_for(T, E, E + k)
    ids, gw = m.router_topk(torch.from_numpy(lg).cuda(), k, renorm)
    rid, rgw = po.Oracle().router_topk(lg, k, renorm)
    assert (ids.cpu().numpy() == rid).all()
    assert (gw.cpu().numpy().view(np.uint32) == rgw.view(np.uint32)).all()
    dg = np.random.default_rng(3).standard_normal((T, k)).astype(np.float32)
    dl = m.router_topk_bwd(torch.from_numpy(lg).cuda(), ids, gw, torch.from_numpy(dg).cuda(), renorm)
    rdl = po.Oracle().router_topk_bwd(lg, rid, rgw, dg, renorm)
    assert (dl.cpu().numpy().view(np.uint32) == rdl.view(np.uint32)).all()


def test_router_empty_and_validation():
    m = moe()
    ids, gw = m.router_topk(torch.zeros(0, 8, device="cuda"), 2)
    assert ids.shape == (0, 2) and gw.shape == (0, 2)
    with pytest.raises(m.EplabError) as e:
        m.router_topk(torch.zeros(4, 8, device="cuda"), 9)
    assert e.value.code == 2
    with pytest.raises(m.EplabError):
        m.router_topk(torch.zeros(4, 2048, device="cuda"), 2)
    with pytest.raises(m.EplabError):
        m.router_topk(torch.zeros(4, 8, device="cuda", dtype=torch.bfloat16), 2)


def test_router_feeds_layer_and_autograd():
    """logits -> router -> EP-MoE layer -> loss; dlogits through both autograd functions equals
    router_topk_bwd(dgate of the layer)."""
    m = moe()
    T, H, F, E, k = 256, 256, 256, 8, 2
    g = torch.Generator(device="cuda").manual_seed(0)
    lg = torch.randn(T, E, device="cuda", generator=g).requires_grad_()
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    wu = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    wd = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    layer = m.EpMoE(H, F, E, k, T)
    ids, gw = m.RouterFunction.apply(lg, k, True)
    y = m.EpMoEFunction.apply(layer, x, ids, gw, wu, wd)
    dy = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    y.backward(dy)
    layer.check()
    # the same chain by hand
    layer2 = m.EpMoE(H, F, E, k, T)
    layer2.forward(x, ids.detach(), gw.detach(), wu, wd)
    gr = layer2.backward(dy, wu, wd)
    ref = m.router_topk_bwd(lg.detach(), ids, gw.detach(), gr["dgate"], True)
    assert torch.equal(lg.grad, ref)
    assert float(lg.grad.abs().sum()) > 0
    layer.close()
    layer2.close()
