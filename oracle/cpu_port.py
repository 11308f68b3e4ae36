"""CPU port of the MoE layer fwd+bwd for TIMING (bench.py's cpu_baseline and --impl reference arms).

TEST / BENCH INFRASTRUCTURE ONLY -- never imported by the product package. The reference computes
no layer numerics, so the CPU arm is a port of the layer contract that
oracle/eplab_oracle.c states: expert buffers in global (src, t, j) order, bf16
roundings of gu, h, o, dGU, HW, dX at the same points, the reference's k-ordered fold. The C oracle
is the CHECKER (sequential loops, the exact summation order the tests pin); this port runs the same
contraction with an optimised CPU BLAS (torch CPU fp32 matmul over MKL / oneDNN, every host thread),
so the baseline is a fair CPU implementation rather than a scalar triple loop. Its fp32 summation
order inside the GEMMs differs from the C oracle's (tests/test_oracle.py bounds the difference).
"""
import time

import numpy as np


def _bf(t):
    import torch
    return t.to(torch.bfloat16).to(torch.float32)


def moe_layer(sel, gw, x, w_up, w_down, dy, E, k, expand=True):
    """sel int [T*k], gw f32 [T*k]; x, dy float32 [T, H] (bf16 values); w_up [E, 2F, H], w_down [E, H, F]
    float32 (bf16 values). Returns (y, dx, dgate, dw_up, dw_down) as float32 (bf16 values except dgate)."""
    import torch
    T, H = x.shape
    F = w_down.shape[2]
    sel_t = torch.as_tensor(np.asarray(sel, np.int64))
    gw_t = torch.as_tensor(np.asarray(gw, np.float32))
    order = torch.argsort(sel_t, stable=True)  # expert buffers in (t, j) order per expert
    counts = torch.bincount(sel_t, minlength=E).tolist()
    y_rep = torch.empty(T * k, H)
    dx_rep = torch.empty(T * k, H)
    dgate = torch.empty(T * k)
    dw_up = torch.empty(E, 2 * F, H, dtype=torch.bfloat16)  # every expert's block is written below
    dw_down = torch.empty(E, H, F, dtype=torch.bfloat16)
    dwd_f = torch.empty(H, F)  # fp32 scratch of one expert's weight gradients
    dwu_f = torch.empty(2 * F, H)
    pos = 0
    for e in range(E):
        n = counts[e]
        if n == 0:
            dw_up[e].zero_()
            dw_down[e].zero_()
            continue
        idx = order[pos:pos + n]
        pos += n
        tok = idx // k
        xe, dye, we = x[tok], dy[tok], gw_t[idx]
        gu = _bf(xe @ w_up[e].t())                      # up GroupGEMM
        g, u = gu[:, :F], gu[:, F:]
        s = torch.sigmoid(g)
        h = _bf(g * s * u)                              # SwiGLU
        o = _bf(h @ w_down[e].t())                      # down GroupGEMM
        y_rep[idx] = o
        dyw = dye @ w_down[e]                           # down dgrad accumulator (before the gate weight)
        dgate[idx] = (dyw * h).sum(1)                   # gate gradient <dY, o> = <dY W_down, h>
        dh = we[:, None] * dyw
        dgu = torch.cat([_bf(dh * u * s * (1 + g * (1 - s))), _bf(dh * g * s)], 1)  # SwiGLU bwd
        hw = _bf(we[:, None] * h)
        dx_rep[idx] = _bf(dgu @ w_up[e])                # up dgrad
        torch.matmul(dye.t(), hw, out=dwd_f[:H, :F])   # down wgrad (fp32), one rounding to bf16
        dw_down[e].copy_(dwd_f[:H, :F])
        torch.matmul(dgu.t(), xe, out=dwu_f[:2 * F, :H])  # up wgrad
        dw_up[e].copy_(dwu_f[:2 * F, :H])
    # combine: the reference fold (k ascending, fp32 rounding of every product and sum), one RNE
    wk = gw_t.view(T, k)
    yr, dr = y_rep.view(T, k, H), dx_rep.view(T, k, H)
    y = wk[:, 0:1] * yr[:, 0]
    dx = dr[:, 0].clone()
    for j in range(1, k):
        y = y + wk[:, j:j + 1] * yr[:, j]
        dx = dx + dr[:, j]
    if not expand:  # the timed form: weight gradients stay bf16, as the GPU path writes them
        return _bf(y), _bf(dx), dgate, dw_up, dw_down
    return _bf(y), _bf(dx), dgate, dw_up.float(), dw_down.float()


def synthetic(H, F, E, k, T, seed=7):
    """Workload inputs of the bench (the reference's sample_routing; N(0,1) activations, N(0, 1/sqrt(K))
    weights, bf16-valued float32)."""
    import torch
    from oracle import pyoracle as po
    sel, gw = po.Oracle().sample_routing(E, k, T, 1, seed)
    g = torch.Generator().manual_seed(seed)
    x = _bf(torch.randn(T, H, generator=g))
    dy = _bf(torch.randn(T, H, generator=g) * 0.1)
    w_up = _bf(torch.randn(E, 2 * F, H, generator=g) * H ** -0.5)
    w_down = _bf(torch.randn(E, H, F, generator=g) * F ** -0.5)
    return sel[0], gw[0], x, dy, w_up, w_down


def time_step(H, F, E, k, n_tok, threads=None, seed=7):
    """Seconds of one fwd+bwd step of n_tok tokens (EP=1: every expert on this host)."""
    import torch
    if threads:
        torch.set_num_threads(threads)
    sel, gw, x, dy, w_up, w_down = synthetic(H, F, E, k, n_tok, seed)
    t0 = time.perf_counter()
    moe_layer(sel, gw, x, w_up, w_down, dy, E, k, expand=False)
    return time.perf_counter() - t0
