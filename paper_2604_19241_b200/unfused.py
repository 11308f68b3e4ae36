"""The unfused EP-MoE baseline (SURVEY.md §8(d) "Unfused baseline"; a16): NCCL all-to-all ->
grouped GEMM (+SwiGLU) -> NCCL all-to-all back -> k-order reduce, forward and backward, as separate
kernels of libeplab_b200.so with the collectives issued through torch.distributed (NCCL) between
them. The split sizes need the all-gathered per-expert counts on the host (one synchronisation per
step), and no transfer overlaps a GEMM -- exactly what the MegaKernels remove.

Its GEMM tiles and reduce are the MegaKernels' own arithmetic, so a step here is BITWISE equal to the
fused step (the reference's fused_vs_sequential contract, precision.cpp:54-96); tests/
test_unfused_gpu.py checks that at EP=1 and EP=2.

  layers = [UnfusedEpMoE(H, F, E, k, T, rank=r, world=W) for r in local ranks]
  ys, grads = unfused_step(layers, comm, xs, ids, gws, dys, w_ups, w_downs)
comm: NcclComm() (one process per GPU, torch.distributed initialised) or LocalComm() (every rank in
this process: the exchanges become device copies -- the single-GPU test mode, and EP=1).
"""
import ctypes as C

import torch

from .moe import EpMoE, _check, _ptr, _stream, lib

_P = C.c_void_p
_I = C.c_int
_SIGS = {
    "eplab_unfused_plan_counts": [_P, _P, _P, _I, _P, _P],
    "eplab_unfused_plan_finish": [_P, _P, _P],
    "eplab_unfused_pack": [_P, _P, _P, _P, _P],
    "eplab_unfused_scatter": [_P, _P, _P, _I, _I, _P],
    "eplab_unfused_up": [_P, _P, _P],
    "eplab_unfused_down": [_P, _P, _P, _P],
    "eplab_unfused_combine": [_P, _P, _P, _I, _P],
    "eplab_unfused_dgate": [_P, _P, _P, _P],
    "eplab_unfused_bwd_down": [_P, _P, _P, _P, _P],
    "eplab_unfused_bwd_up": [_P, _P, _P, _P, _P],
}


def _lib():
    L = lib()
    if not getattr(L, "_eplab_unfused_sigs", False):
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _I
        L._eplab_unfused_sigs = True
    return L


class UnfusedEpMoE(EpMoE):
    """One rank of the unfused baseline (same context, buffers and receive layout as EpMoE)."""

    def plan_counts(self, topk_ids, gate_w, stream=None):
        n = topk_ids.shape[0]
        ids = self._need(topk_ids.contiguous(), "topk_ids", (n, self.k), torch.int32)
        gw = self._need(gate_w.contiguous(), "gate_w", (n, self.k), torch.float32)
        self._ids, self._gw = ids, gw
        row = torch.empty(self.E + 1, dtype=torch.int32, device=self.device)
        _check(_lib().eplab_unfused_plan_counts(self.h, _ptr(ids), _ptr(gw), n, _ptr(row), _stream(stream)))
        self.plan_epoch += 1
        return row

    def plan_finish(self, rows_all, stream=None):
        self._rows_all = rows_all.contiguous()
        _check(_lib().eplab_unfused_plan_finish(self.h, _ptr(self._rows_all), _stream(stream)))

    def splits(self, rows_host):
        """(send split per destination rank, receive split per source rank), rows_host [W][E+1]."""
        c = rows_host[:, :self.E].reshape(self.world, self.world, self.epr).sum(axis=2)  # [src][dst]
        return [int(v) for v in c[self.rank]], [int(v) for v in c[:, self.rank]]

    def pack(self, src, send, send_meta=None, stream=None):
        _check(_lib().eplab_unfused_pack(self.h, _ptr(src), _ptr(send), _ptr(send_meta), _stream(stream)))

    def scatter(self, recv, recv_meta, n_recv, phase, stream=None):
        _check(_lib().eplab_unfused_scatter(self.h, _ptr(recv), _ptr(recv_meta), n_recv, phase, _stream(stream)))

    def up(self, w_up, stream=None):
        _check(_lib().eplab_unfused_up(self.h, _ptr(w_up), _stream(stream)))

    def down(self, w_down, o_ret, stream=None):
        _check(_lib().eplab_unfused_down(self.h, _ptr(w_down), _ptr(o_ret), _stream(stream)))

    def combine(self, rows, out, phase, stream=None):
        _check(_lib().eplab_unfused_combine(self.h, _ptr(rows), _ptr(out), phase, _stream(stream)))

    def dgate(self, dgp_src, dgate, stream=None):
        _check(_lib().eplab_unfused_dgate(self.h, _ptr(dgp_src), _ptr(dgate), _stream(stream)))

    def bwd_down(self, w_down, dw_down, dgp_ret, stream=None):
        _check(_lib().eplab_unfused_bwd_down(self.h, _ptr(w_down), _ptr(dw_down), _ptr(dgp_ret), _stream(stream)))

    def bwd_up(self, w_up, dx_ret, dw_up, stream=None):
        _check(_lib().eplab_unfused_bwd_up(self.h, _ptr(w_up), _ptr(dx_ret), _ptr(dw_up), _stream(stream)))


class NcclComm:
    """One local rank per process; the collectives of torch.distributed (NCCL on GPUs).
    staged=True moves the buffers through host memory (gloo process groups, which have no CUDA
    all-to-all: the multi-process test of several ranks sharing one GPU, where NCCL refuses)."""

    def __init__(self, group=None, staged=False):
        import torch.distributed as dist
        self.dist, self.group, self.staged = dist, group, staged
        self.world = dist.get_world_size(group)

    def all_gather(self, rows):
        (row,) = rows
        if self.staged:
            parts = [torch.empty_like(row, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, row.cpu(), group=self.group)
            return [torch.stack(parts).to(row.device)]
        out = torch.empty(self.world, row.numel(), dtype=row.dtype, device=row.device)
        self.dist.all_gather_into_tensor(out, row, group=self.group)  # ncclAllGather
        return [out]

    def all_to_all(self, sends, send_splits, recv_splits, width, dtype):
        (send,), (ss,), (rs,) = sends, send_splits, recv_splits
        dev = send.device
        if self.staged:  # gloo all-to-all: host tensors of a 32-bit type (bf16 rows as int32 pairs)
            send = (send.view(torch.int32) if dtype == torch.bfloat16 else send).cpu()
            width = width // 2 if dtype == torch.bfloat16 else width
        out = torch.empty(sum(rs), width, dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(out, send, output_split_sizes=rs, input_split_sizes=ss,
                                    group=self.group)  # grouped ncclSend / ncclRecv
        if self.staged:
            out = out.to(dev)
            if dtype == torch.bfloat16:
                out = out.view(torch.bfloat16)
        return [out]


class LocalComm:
    """Every rank in this process (virtual ranks / EP=1): the same exchanges as device copies."""

    def all_gather(self, rows):
        out = torch.stack(rows)
        return [out for _ in rows]

    def all_to_all(self, sends, send_splits, recv_splits, width, dtype):
        W = len(sends)
        offs = [[sum(send_splits[s][:d]) for d in range(W)] for s in range(W)]
        outs = []
        for d in range(W):
            parts = [sends[s][offs[s][d]:offs[s][d] + send_splits[s][d]] for s in range(W)]
            outs.append(torch.cat(parts) if parts else torch.empty(0, width, dtype=dtype, device=sends[0].device))
        return outs


def unfused_step(layers, comm, xs, ids, gws, dys, w_ups, w_downs, stream=None):
    """One fwd+bwd step of every local rank in `layers` (lists indexed like `layers`). Returns
    (ys, grads) with grads[r] = dict(dx, dgate, dw_up, dw_down)."""
    n = len(layers)
    H = layers[0].H
    bf16 = torch.bfloat16
    rows = [L.plan_counts(ids[r], gws[r], stream) for r, L in enumerate(layers)]
    rows_all = comm.all_gather(rows)
    for r, L in enumerate(layers):
        L.plan_finish(rows_all[r], stream)
    host = rows_all[0].cpu().numpy()  # the split sizes: one host synchronisation per step
    sp = [L.splits(host) for L in layers]
    ss, rs = [s for s, _ in sp], [q for _, q in sp]
    n_send, n_recv = [sum(s) for s in ss], [sum(q) for q in rs]
    dev = xs[0].device
    # ---- forward: dispatch A2A, up GEMM + SwiGLU, down GEMM, return A2A, reduce
    send = [torch.empty(n_send[r], H, dtype=bf16, device=dev) for r in range(n)]
    meta = [torch.empty(n_send[r], 2, dtype=torch.int32, device=dev) for r in range(n)]
    for r, L in enumerate(layers):
        L.pack(xs[r], send[r], meta[r], stream)
    recv = comm.all_to_all(send, ss, rs, H, bf16)
    recv_meta = comm.all_to_all(meta, ss, rs, 2, torch.int32)
    o_ret = []
    for r, L in enumerate(layers):
        L.scatter(recv[r], recv_meta[r], n_recv[r], 0, stream)
        L.up(w_ups[r], stream)
        o_ret.append(torch.empty(n_recv[r], H, dtype=bf16, device=dev))
        L.down(w_downs[r], o_ret[r], stream)
    o_src = comm.all_to_all(o_ret, rs, ss, H, bf16)
    ys = []
    for r, L in enumerate(layers):
        ys.append(torch.empty(xs[r].shape[0], H, dtype=bf16, device=dev))
        L.combine(o_src[r], ys[r], 0, stream)
    # ---- backward: dY A2A, gate gradient, down dgrad + SwiGLU bwd + down wgrad, up dgrad + up
    # wgrad, return A2A, reduce
    for r, L in enumerate(layers):
        L.pack(dys[r], send[r], None, stream)
    recv = comm.all_to_all(send, ss, rs, H, bf16)
    ncb = layers[0].F // 256  # gate-gradient partials per row: one per down-dgrad column tile
    grads, dx_ret, dgp_ret = [], [], []
    for r, L in enumerate(layers):
        L.scatter(recv[r], None, n_recv[r], 1, stream)
        g = dict(dx=torch.empty_like(xs[r]), dgate=torch.empty(ids[r].shape, dtype=torch.float32, device=dev),
                 dw_up=torch.empty_like(w_ups[r]), dw_down=torch.empty_like(w_downs[r]))
        dgp_ret.append(torch.empty(n_recv[r], ncb, dtype=torch.float32, device=dev))
        L.bwd_down(w_downs[r], g["dw_down"], dgp_ret[r], stream)
        dx_ret.append(torch.empty(n_recv[r], H, dtype=bf16, device=dev))
        L.bwd_up(w_ups[r], dx_ret[r], g["dw_up"], stream)
        grads.append(g)
    dgp_src = comm.all_to_all(dgp_ret, rs, ss, ncb, torch.float32)
    dx_src = comm.all_to_all(dx_ret, rs, ss, H, bf16)
    for r, L in enumerate(layers):
        L.dgate(dgp_src[r], grads[r]["dgate"], stream)
        L.combine(dx_src[r], grads[r]["dx"], 1, stream)
    return ys, grads
