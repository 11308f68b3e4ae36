"""Unfused separate-kernel baseline of the EP-MoE layer (the paper's "Serial" = DeepEP + TE,
PAPER.md:588): permute -> NCCL all_to_all (EP > 1, counts exchanged first,
host-synchronising) -> per-expert cuBLAS bf16 GEMMs + separate SwiGLU -> NCCL all_to_all back ->
weighted scatter-add. Backward by torch autograd (same collectives reversed). Same routing,
weights and numerics class (bf16 in, fp32 accumulate) as the MegaKernels."""
import torch
import torch.distributed as dist
import torch.nn.functional as Fn


class _A2A(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, send, recv):
        ctx.send, ctx.recv = send, recv
        out = x.new_empty((sum(recv), x.shape[1]))
        dist.all_to_all_single(out, x.contiguous(), recv, send)
        return out

    @staticmethod
    def backward(ctx, g):
        out = g.new_empty((sum(ctx.send), g.shape[1]))
        dist.all_to_all_single(out, g.contiguous(), ctx.send, ctx.recv)
        return out, None, None


def layer(x, ids, gw, w_up, w_down, E, world, rank):
    """x [T,H]; ids/gw [T,k]; w_up [E_loc,2F,H]; w_down [E_loc,H,F] (this rank's experts)."""
    T, k = ids.shape
    epr = E // world
    F = w_down.shape[2]
    flat = ids.reshape(-1)
    order = torch.argsort(flat, stable=True)              # (dst rank, expert, t, j) order
    xs = x.index_select(0, order // k)
    counts = torch.bincount(flat, minlength=E)
    if world > 1:
        send = counts.view(world, epr).sum(1)
        all_counts = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(all_counts, counts)                # host sync below (splits)
        allc = torch.stack(all_counts)                     # [src][E]
        recv = allc[:, rank * epr:(rank + 1) * epr].sum(1)
        xr = _A2A.apply(xs, send.tolist(), recv.tolist())
        # received rows are grouped (src, local expert); regroup by local expert
        lc = allc[:, rank * epr:(rank + 1) * epr]          # [src][e_loc]
        e_of_row = torch.repeat_interleave(torch.arange(epr, device=x.device).repeat(world), lc.reshape(-1))
        perm = torch.argsort(e_of_row, stable=True)
        xe_all = xr.index_select(0, perm)
        per_e = lc.sum(0).tolist()
    else:
        xe_all = xs
        per_e = counts.tolist()
    outs = []
    s = 0
    for e in range(epr):
        n = per_e[e]
        xe = xe_all[s:s + n]
        gu = xe @ w_up[e].t()
        h = Fn.silu(gu[:, :F]) * gu[:, F:]
        outs.append(h @ w_down[e].t())
        s += n
    ye = torch.cat(outs)
    if world > 1:
        yr = torch.empty_like(ye).index_copy(0, perm, ye) if False else ye.new_zeros(ye.shape).index_add(0, perm, ye)
        ys = _A2A.apply(yr, recv.tolist(), send.tolist())
    else:
        ys = ye
    w = gw.reshape(-1).index_select(0, order).unsqueeze(1).to(ys.dtype)
    return torch.zeros_like(x).index_add(0, order // k, ys * w)
