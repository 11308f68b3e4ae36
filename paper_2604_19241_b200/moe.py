"""Python mirror of the EP-MoE data path (drop-in for the reference's dispatch / group_gemm /
combine entry points), over the C-ABI of libeplab_b200.so.

PyTorch supplies device memory, streams and torch.distributed bootstrap only; every
computation runs in the library's sm_100a kernels. There is no CPU fallback: without the
library or a CUDA device every call raises.
"""
import ctypes as C
import weakref

import torch

from . import _lib

_P = C.c_void_p
_I = C.c_int


class InitArgs(C.Structure):
    _fields_ = [("rank", _I), ("world", _I), ("device", _I), ("max_tokens", _I), ("hidden", _I),
                ("ffn", _I), ("n_experts", _I), ("topk", _I), ("max_recv_rows", C.c_longlong),
                ("timeout_s", C.c_double)]


class TuneConfig(C.Structure):
    """Reference TuneConfig (types.hpp:45-53)."""
    _fields_ = [("n_disp", _I), ("n_relay", _I), ("n_comb", _I), ("n_red", _I), ("w", _I)]

    def __repr__(self):
        return f"TuneConfig({self.n_disp},{self.n_relay},{self.n_comb},{self.n_red},{self.w})"


class EplabError(RuntimeError):
    """Raised on a non-zero C-ABI return: .code is 1 (internal), 2 (validation, the reference's
    ValidationError) or 3 (deadlock / watchdog, the reference's DeadlockError)."""

    def __init__(self, code, msg):
        super().__init__(f"[eplab rc={code}] {msg}")
        self.code = code


_SIGS = {
    "eplab_init": [C.POINTER(InitArgs), C.POINTER(_P)],
    "eplab_destroy": [_P],
    "eplab_ipc_handle": [_P, _P],
    "eplab_connect_ipc": [_P, _P],
    "eplab_connect_local": [C.POINTER(_P), _I],
    "eplab_set_tune_config": [_P, C.POINTER(TuneConfig)],
    "eplab_get_tune_config": [_P, C.POINTER(TuneConfig)],
    "eplab_set_sm_budget": [_P, _I],
    "eplab_set_comm_options": [_P, _I, _I],
    "eplab_set_auto_tune": [_P, _I],
    "eplab_set_option": [_P, C.c_char_p, _I],
    "eplab_plan": [_P, _P, _P, _I, _P],
    "eplab_dispatch_group_gemm": [_P, _P, _P, _P],
    "eplab_group_gemm_combine": [_P, _P, _P, _P],
    "eplab_dispatch_group_gemm_bwd": [_P, _P, _P, _P, _P, _P],
    "eplab_group_gemm_combine_bwd": [_P, _P, _P, _P, _P],
    "eplab_moe_fwd": [_P, _P, _P, _I, _P, _P, _P, _P, _P],
    "eplab_moe_bwd": [_P, _P, _P, _P, _P, _P, _P, _P, _P],
    "eplab_moe_step_host": [_P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "eplab_moe_step_host_async": [_P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "eplab_host_join": [_P, _P],
    "eplab_bf16_accumulate": [_P, _P, C.c_size_t, _P],
    "eplab_check": [_P, _P],
    "eplab_export_token_map": [_P, _P, _P, _P, _P, _P],
    "eplab_export_schedule": [_P, _P, _P],
    "eplab_export_layout": [_P, _P, _P],
    "eplab_timeline_enable": [_P, _I],
    "eplab_timeline_export": [_P, C.c_char_p, C.POINTER(C.c_double)],
    "eplab_router_topk": [_P, _I, _I, _I, _I, _P, _P, _P],
    "eplab_stash_bytes": [_P, C.POINTER(C.c_size_t), _P],
    "eplab_stash_save": [_P, _P, C.c_size_t, _P, _P],
    "eplab_stash_restore": [_P, _P, _P, _P],
    "eplab_router_topk_bwd": [_P, _P, _P, _P, _I, _I, _I, _I, _P, _P],
}


def lib():
    L = _lib.lib()
    if not getattr(L, "_eplab_sigs", False):
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _I
        L.eplab_buffer.argtypes = [_P, C.c_char_p]
        L.eplab_buffer.restype = _P
        L.eplab_last_error.argtypes = [C.c_char_p, C.c_size_t]
        L.eplab_last_error.restype = C.c_size_t
        L._eplab_sigs = True
    return L


def _check(rc):
    if rc:
        buf = C.create_string_buffer(1024)
        lib().eplab_last_error(buf, 1024)
        raise EplabError(rc, buf.value.decode(errors="replace"))


def _ptr(t):
    return None if t is None else _P(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return _P(s.cuda_stream)


class StashInfo(C.Structure):
    """eplab_stash_info (include/eplab_b200.h)."""
    _fields_ = [("magic", C.c_uint32), ("epoch", C.c_uint32), ("n_tok", _I), ("rows", _I),
                ("topk_ids", _P), ("gate_w", _P), ("bytes", C.c_size_t)]


class Stash:
    """One iteration's state copied out of a context (EpMoE.stash / restore): the device buffer,
    the library's info record, and the routing tensors the plan points at (kept alive)."""

    def __init__(self, epoch, buf, info, ids, gw):
        self.epoch, self.buf, self.info, self.ids, self.gw = epoch, buf, info, ids, gw

    @property
    def nbytes(self):
        return self.info.bytes


_LIVE = weakref.WeakSet()  # open contexts (tests release them after a failure: live_contexts())


def live_contexts():
    """Contexts not yet closed (their device memory is the library's, not torch's allocator's)."""
    return [c for c in list(_LIVE) if c.h]


class EpMoE:
    """One rank of the expert-parallel MoE layer (experts sharded contiguously: rank = e // epr).

    Tensors: x, dy [n_tok, H] bf16; topk_ids [n_tok, k] int32; gate_w [n_tok, k] fp32;
    w_up [E_loc, 2F, H] bf16 (gate rows [0,F), up rows [F,2F)); w_down [E_loc, H, F] bf16.
    """

    def __init__(self, hidden, ffn, n_experts, topk, max_tokens, rank=0, world=1, device=None,
                 max_recv_rows=0, timeout_s=10.0):
        if not torch.cuda.is_available():
            raise RuntimeError("EpMoE needs a CUDA (sm_100a) device; there is no CPU path")
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        self.H, self.F, self.E, self.k, self.T_max = hidden, ffn, n_experts, topk, max_tokens
        self.rank, self.world, self.epr = rank, world, n_experts // world
        a = InitArgs(rank, world, dev.index, max_tokens, hidden, ffn, n_experts, topk, max_recv_rows,
                     timeout_s)
        h = _P()
        with torch.cuda.device(dev):
            _check(lib().eplab_init(C.byref(a), C.byref(h)))
        self.h = h
        _LIVE.add(self)
        self._ids = self._gw = None
        self.plan_epoch = 0  # id of the plan whose state the context holds (EpMoEFunction ties
        self._plans = 0      # its backward to it); ids are never reused
        self._pending = {}   # plan id -> weakref to the autograd node whose backward needs it
        self._stashes = {}   # plan id -> Stash (made when a later plan would overwrite it)

    def close(self):
        if self.h:
            lib().eplab_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ wiring
    @staticmethod
    def connect_local(ranks):
        arr = (_P * len(ranks))(*[r.h for r in ranks])
        _check(lib().eplab_connect_local(arr, len(ranks)))

    IPC_HANDLE_BYTES = 128  # EPLAB_IPC_HANDLE_BYTES: CUDA IPC handle + layout signature

    def ipc_handle(self):
        buf = (C.c_char * self.IPC_HANDLE_BYTES)()
        _check(lib().eplab_ipc_handle(self.h, buf))
        return bytes(buf)

    def connect_ipc(self, handles):
        blob = b"".join(handles)
        _check(lib().eplab_connect_ipc(self.h, C.c_char_p(blob)))

    def connect_distributed(self, group=None):
        """Bootstrap over torch.distributed (NCCL or gloo): all-gather the IPC handles."""
        import torch.distributed as dist
        hs = [None] * self.world
        dist.all_gather_object(hs, self.ipc_handle(), group=group)
        self.connect_ipc(hs)

    def set_tune_config(self, cfg):
        if isinstance(cfg, (tuple, list)):
            cfg = TuneConfig(*cfg)
        _check(lib().eplab_set_tune_config(self.h, C.byref(cfg)))

    def set_comm_options(self, spare_warps=3, bulk_mover=False):
        """spare_warps: bit 0 = comm pool, bit 1 = backward reduce pool (True = 3, False = 0)."""
        sw = 3 if spare_warps is True else (0 if spare_warps is False else int(spare_warps))
        _check(lib().eplab_set_comm_options(self.h, sw, int(bulk_mover)))

    def set_option(self, name, value):
        """Experiment knob (eplab_set_option): engine_pair, spare, comm_bulk, rgp, tngp, tngp_d,
        bwd_disp_scale, dbg (dbg != 0 skips work: wrong results, measurements only)."""
        _check(lib().eplab_set_option(self.h, name.encode(), int(value)))

    def set_auto_tune(self, on=True):
        """Per-plan launch parameters from the B200 model, cached per 4096-token bucket (default
        until set_tune_config)."""
        _check(lib().eplab_set_auto_tune(self.h, int(on)))

    def tune_config(self):
        c = TuneConfig()
        lib().eplab_get_tune_config(self.h, C.byref(c))
        return c

    def set_sm_budget(self, n_sm):
        _check(lib().eplab_set_sm_budget(self.h, n_sm))

    # ------------------------------------------------------------------ argument checks
    def _need(self, t, name, shape, dtype=torch.bfloat16):
        """Every tensor crossing the C-ABI: on this context's device, contiguous, exact dtype and
        shape (the kernels read raw pointers with this layout). Raises EplabError(2)."""
        if not isinstance(t, torch.Tensor):
            raise EplabError(2, f"{name}: expected a torch.Tensor, got {type(t).__name__}")
        if t.device != self.device:
            raise EplabError(2, f"{name}: on {t.device}, the context is on {self.device}")
        if t.dtype != dtype:
            raise EplabError(2, f"{name}: dtype {t.dtype}, expected {dtype}")
        if tuple(t.shape) != tuple(shape):
            raise EplabError(2, f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
        if not t.is_contiguous():
            raise EplabError(2, f"{name}: must be contiguous")
        return t

    def _need_planned(self):
        if self._ids is None:
            raise EplabError(2, "no plan: call plan() (or forward()) first")
        return self._ids.shape[0]

    def _need_weights(self, w_up=None, w_down=None):
        if w_up is not None:
            self._need(w_up, "w_up", (self.epr, 2 * self.F, self.H))
        if w_down is not None:
            self._need(w_down, "w_down", (self.epr, self.H, self.F))

    # ------------------------------------------------------------------ data path
    def plan(self, topk_ids, gate_w, stream=None):
        if topk_ids.dim() != 2 or topk_ids.shape[1] != self.k:
            raise EplabError(2, f"topk_ids: shape {tuple(topk_ids.shape)}, expected (n_tok, {self.k})")
        n = topk_ids.shape[0]
        ids = self._need(topk_ids.contiguous(), "topk_ids", (n, self.k), torch.int32)
        gw = self._need(gate_w.contiguous(), "gate_w", (n, self.k), torch.float32)
        self._evict(stream)
        self._ids, self._gw = ids, gw
        _check(lib().eplab_plan(self.h, _ptr(ids), _ptr(gw), n, _stream(stream)))
        self._plans += 1
        self.plan_epoch = self._plans

    # ------------------------------------------------------------------ several forwards in flight
    def stash(self, stream=None):
        """Copy the current iteration's state (plan tables, received rows and slot metadata, saved
        g/u and h) into a new device buffer sized to its receive rows (eplab_stash_save)."""
        self._need_planned()
        nb = C.c_size_t()
        _check(lib().eplab_stash_bytes(self.h, C.byref(nb), _stream(stream)))
        buf = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
        info = StashInfo()
        _check(lib().eplab_stash_save(self.h, _ptr(buf), nb.value, C.byref(info), _stream(stream)))
        if stream is not None:
            buf.record_stream(stream)
        return Stash(self.plan_epoch, buf, info, self._ids, self._gw)

    def restore(self, st, stream=None):
        """Make a stashed iteration the current one again: its backward may run next. The live
        iteration is stashed first if an autograd backward still needs it."""
        self._evict(stream)
        _check(lib().eplab_stash_restore(self.h, _ptr(st.buf), C.byref(st.info), _stream(stream)))
        self._ids, self._gw = st.ids, st.gw
        self.plan_epoch = st.epoch

    def _evict(self, stream):
        """Before the context's state is overwritten: stash it if a pending autograd backward
        (one whose graph is still alive) needs it; forget stashes whose graphs were freed."""
        for e in [e for e, r in self._pending.items() if r() is None]:
            self._pending.pop(e)
            self._stashes.pop(e, None)
        e = self.plan_epoch
        if e in self._pending and e not in self._stashes:
            self._stashes[e] = self.stash(stream)

    def dispatch_group_gemm(self, x, w_up, stream=None):
        n = self._need_planned()
        self._need(x, "x", (n, self.H))
        self._need_weights(w_up=w_up)
        _check(lib().eplab_dispatch_group_gemm(self.h, _ptr(x), _ptr(w_up), _stream(stream)))

    def group_gemm_combine(self, w_down, y=None, stream=None):
        n = self._need_planned()
        self._need_weights(w_down=w_down)
        if y is None:
            y = torch.empty(n, self.H, dtype=torch.bfloat16, device=self.device)
        self._need(y, "y", (n, self.H))
        _check(lib().eplab_group_gemm_combine(self.h, _ptr(w_down), _ptr(y), _stream(stream)))
        return y

    def forward(self, x, topk_ids, gate_w, w_up, w_down, stream=None):
        self.plan(topk_ids, gate_w, stream)
        self.dispatch_group_gemm(x, w_up, stream)
        return self.group_gemm_combine(w_down, stream=stream)

    def backward(self, dy, w_up, w_down, stream=None, out=None):
        n = self._need_planned()
        dev = self.device
        self._need(dy, "dy", (n, self.H))
        self._need_weights(w_up, w_down)
        if out is None:
            out = dict(dx=torch.empty(n, self.H, dtype=torch.bfloat16, device=dev),
                       dw_up=torch.empty_like(w_up), dw_down=torch.empty_like(w_down),
                       dgate=torch.empty(n, self.k, dtype=torch.float32, device=dev))
        self._need(out["dx"], "dx", (n, self.H))
        self._need(out["dgate"], "dgate", (n, self.k), torch.float32)
        self._need_weights(out["dw_up"], out["dw_down"])
        self._dispatch_bwd(dy, w_down, out, stream)
        self._combine_bwd(w_up, out, stream)
        return out

    def step_split(self, x, topk_ids, gate_w, dy, w_up, w_down, n_sub=2, stream=None):
        """Opt-in NON-BITWISE (NB) split-batch step: the
        tokens are cut into n_sub contiguous sub-batches, each runs plan + the four MegaKernels,
        and the weight gradients are summed in bf16 (eplab_bf16_accumulate). y, dx and dgate are
        bitwise identical to the full-batch step (row-local); dw_up / dw_down differ by the
        changed accumulation tree (the divergence precision.cpp:98-134 measures)."""
        n = x.shape[0]
        dev = self.device
        y = torch.empty(n, self.H, dtype=torch.bfloat16, device=dev)
        out = dict(dx=torch.empty(n, self.H, dtype=torch.bfloat16, device=dev),
                   dw_up=torch.empty_like(w_up), dw_down=torch.empty_like(w_down),
                   dgate=torch.empty(n, self.k, dtype=torch.float32, device=dev))
        part = dict(dw_up=torch.empty_like(w_up), dw_down=torch.empty_like(w_down))
        bounds = [n * i // n_sub for i in range(n_sub + 1)]
        for i in range(n_sub):
            lo, hi = bounds[i], bounds[i + 1]
            self.plan(topk_ids[lo:hi], gate_w[lo:hi], stream)
            self.dispatch_group_gemm(x[lo:hi], w_up, stream)
            self.group_gemm_combine(w_down, y[lo:hi], stream)
            o = dict(dx=out["dx"][lo:hi], dgate=out["dgate"][lo:hi],
                     dw_up=out["dw_up"] if i == 0 else part["dw_up"],
                     dw_down=out["dw_down"] if i == 0 else part["dw_down"])
            self._dispatch_bwd(dy[lo:hi], w_down, o, stream)
            self._combine_bwd(w_up, o, stream)
            if i:
                for key in ("dw_up", "dw_down"):
                    _check(lib().eplab_bf16_accumulate(_ptr(out[key]), _ptr(part[key]), out[key].numel(),
                                                       _stream(stream)))
        return y, out

    def _dispatch_bwd(self, dy, w_down, out, stream=None):
        _check(lib().eplab_dispatch_group_gemm_bwd(self.h, _ptr(dy), _ptr(w_down), _ptr(out["dw_down"]),
                                                   _ptr(out["dgate"]), _stream(stream)))

    def _combine_bwd(self, w_up, out, stream=None):
        _check(lib().eplab_group_gemm_combine_bwd(self.h, _ptr(w_up), _ptr(out["dx"]), _ptr(out["dw_up"]),
                                                  _stream(stream)))

    def step_host(self, ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dgate_h, dw_up, dw_down,
                  stream=None):
        """fwd+bwd through the C-ABI with HOST routing/activations (copies inside the call)."""
        _check(lib().eplab_moe_step_host(self.h, _ptr(ids_h), _ptr(gw_h), ids_h.shape[0], _ptr(x_h),
                                         _ptr(dy_h), _ptr(w_up), _ptr(w_down), _ptr(y_h), _ptr(dx_h),
                                         _ptr(dgate_h), _ptr(dw_up), _ptr(dw_down), _stream(stream)))

    def step_host_async(self, ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dgate_h, dw_up, dw_down,
                        stream=None):
        """The same step enqueued without a host sync; consecutive steps overlap their copies with
        each other's MegaKernels. Outputs are valid after host_join(stream) + stream sync."""
        _check(lib().eplab_moe_step_host_async(self.h, _ptr(ids_h), _ptr(gw_h), ids_h.shape[0], _ptr(x_h),
                                               _ptr(dy_h), _ptr(w_up), _ptr(w_down), _ptr(y_h), _ptr(dx_h),
                                               _ptr(dgate_h), _ptr(dw_up), _ptr(dw_down), _stream(stream)))

    def host_join(self, stream=None):
        _check(lib().eplab_host_join(self.h, _stream(stream)))

    def check(self, stream=None):
        _check(lib().eplab_check(self.h, _stream(stream)))

    # ------------------------------------------------------------------ exports
    def export_token_map(self):
        import numpy as np
        n = self._ids.shape[0] * self.k
        tr = np.zeros(n, np.int32)
        le = np.zeros(n, np.int32)
        off = np.zeros(n, np.int64)
        rt = np.zeros(self.world * self.epr, np.int64)
        sb = np.zeros(self.world * self.epr, np.int64)
        _check(lib().eplab_export_token_map(self.h, tr.ctypes.data, le.ctypes.data, off.ctypes.data,
                                            rt.ctypes.data, sb.ctypes.data))
        return tr, le, off, rt, sb

    def export_schedule(self):
        import numpy as np
        n = self._ids.shape[0] * self.k
        tok = np.zeros(n, np.int64)
        slot = np.zeros(n, np.int32)
        _check(lib().eplab_export_schedule(self.h, tok.ctypes.data, slot.ctypes.data))
        return tok, slot

    def export_layout(self):
        import numpy as np
        sb = np.zeros(self.epr, np.int32)
        rows = np.zeros(self.epr, np.int32)
        _check(lib().eplab_export_layout(self.h, sb.ctypes.data, rows.ctypes.data))
        return sb, rows

    def buffer(self, name, rows, cols):
        """bf16 view of an internal device buffer (tests / profiling)."""
        p = lib().eplab_buffer(self.h, name.encode())
        if not p:
            raise KeyError(name)
        return _DeviceView(p, rows, cols, self.device).tensor()

    def timeline_enable(self, cap=1 << 20):
        _check(lib().eplab_timeline_enable(self.h, cap))

    def timeline_export(self, path=""):
        f = C.c_double()
        _check(lib().eplab_timeline_export(self.h, path.encode(), C.byref(f)))
        return f.value


class _DeviceView:
    """Wraps a raw device pointer as a torch tensor via __cuda_array_interface__."""

    def __init__(self, ptr, rows, cols, device):
        self.__cuda_array_interface__ = {"shape": (rows, cols), "typestr": "<i2", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self.device = device

    def tensor(self):
        with torch.cuda.device(self.device):
            return torch.as_tensor(self, device=self.device).view(torch.bfloat16)


class EpMoEFunction(torch.autograd.Function):
    """Autograd wrapper: y = MoE(x; routing, gate weights, W_up, W_down). Gradients flow to x,
    gate_w (the router output), w_up and w_down; routing ids are integer inputs."""

    @staticmethod
    def forward(ctx, layer, x, topk_ids, gate_w, w_up, w_down):
        y = layer.forward(x.contiguous(), topk_ids, gate_w, w_up, w_down)
        ctx.layer = layer
        # The backward reads this plan's state (receive rows, g/u, h, slot metadata, plan tables)
        # from the context. Several forwards may be in flight (pipelined micro-batches, layers
        # sharing a context, activation recomputation): a later plan stashes this state first
        # (EpMoE._evict) and the backward restores it, in any order.
        ctx.plan_epoch = layer.plan_epoch
        layer._pending[layer.plan_epoch] = weakref.ref(ctx)
        ctx.save_for_backward(w_up, w_down)
        return y

    @staticmethod
    def backward(ctx, dy):
        w_up, w_down = ctx.saved_tensors
        L, e = ctx.layer, ctx.plan_epoch
        if L.plan_epoch != e:
            st = L._stashes.get(e)
            if st is None:
                raise EplabError(2, f"the state of plan {e} is gone (the context holds plan {L.plan_epoch} "
                                    f"and no stash of plan {e} exists: a second backward of a freed graph?)")
            L.restore(st)
        try:
            g = L.backward(dy.contiguous(), w_up, w_down)
        finally:
            L._pending.pop(e, None)
            L._stashes.pop(e, None)
        return None, g["dx"], None, g["dgate"], g["dw_up"], g["dw_down"]


def router_topk(logits, topk, renorm=True, stream=None):
    """Router step in front of plan: fp32 logits [T][E] -> (topk_ids [T][k]
    int32, gate_w [T][k] fp32) on device (eplab_router_topk; semantics in include/eplab_b200.h)."""
    _need_cuda(logits, torch.float32)
    T, E = logits.shape
    ids = torch.empty(T, topk, dtype=torch.int32, device=logits.device)
    gw = torch.empty(T, topk, dtype=torch.float32, device=logits.device)
    st = stream if stream is not None else torch.cuda.current_stream(logits.device)
    _check(lib().eplab_router_topk(logits.data_ptr(), T, E, topk, int(renorm), ids.data_ptr(), gw.data_ptr(),
                                   st.cuda_stream))
    return ids, gw


def router_topk_bwd(logits, topk_ids, gate_w, dgate, renorm=True, stream=None):
    """dgate [T][k] -> dlogits [T][E] (eplab_router_topk_bwd)."""
    _need_cuda(logits, torch.float32)
    T, E = logits.shape
    dl = torch.empty(T, E, dtype=torch.float32, device=logits.device)
    st = stream if stream is not None else torch.cuda.current_stream(logits.device)
    _check(lib().eplab_router_topk_bwd(logits.data_ptr(), topk_ids.data_ptr(), gate_w.data_ptr(),
                                       dgate.contiguous().data_ptr(), T, E, topk_ids.shape[1], int(renorm),
                                       dl.data_ptr(), st.cuda_stream))
    return dl


def _need_cuda(t, dtype):
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous() and t.dim() == 2):
        raise EplabError(2, f"expected a contiguous 2-D {dtype} CUDA tensor, got {t.dtype} on {t.device}")


class RouterFunction(torch.autograd.Function):
    """Autograd wrapper: (topk_ids, gate_w) = router(logits); gradients flow from gate_w (e.g.
    EpMoEFunction's dgate) back to the logits."""

    @staticmethod
    def forward(ctx, logits, topk, renorm=True):
        logits = logits.contiguous()
        ids, gw = router_topk(logits, topk, renorm)
        ctx.renorm = renorm
        ctx.save_for_backward(logits, ids, gw)
        ctx.mark_non_differentiable(ids)
        return ids, gw

    @staticmethod
    def backward(ctx, d_ids, d_gw):
        logits, ids, gw = ctx.saved_tensors
        if d_gw is None:
            return None, None, None
        return router_topk_bwd(logits, ids, gw, d_gw, ctx.renorm), None, None


class MoELayer(torch.nn.Module):
    """A trainable MoE FFN block on the MegaKernels: router (fp32 logits = x W_gate, softmax top-k on the
    device, RouterFunction) -> EpMoEFunction (dispatch + up GroupGEMM + SwiGLU, down GroupGEMM + combine,
    and their backward). Parameters: gate [H][E] fp32, this rank's experts w_up [E_loc][2F][H] and
    w_down [E_loc][H][F] bf16. x [n_tok][H] bf16 -> y [n_tok][H] bf16; gradients reach x (through both
    the experts and the router), the gate and the expert weights. Multi-rank: one module per rank,
    connected with `self.experts.connect_distributed()` before the first forward."""

    def __init__(self, hidden, ffn, n_experts, topk, max_tokens, rank=0, world=1, renorm=True, device=None,
                 seed=0):
        super().__init__()
        self.experts = EpMoE(hidden, ffn, n_experts, topk, max_tokens, rank=rank, world=world, device=device)
        dev = self.experts.device
        epr = n_experts // world
        # the router is replicated (the same gate on every rank); the experts are this rank's shard
        g = torch.Generator(device=dev).manual_seed(seed)
        self.gate = torch.nn.Parameter(torch.randn(hidden, n_experts, device=dev, generator=g) * hidden ** -0.5)
        g = torch.Generator(device=dev).manual_seed(seed + 1 + rank)
        self.w_up = torch.nn.Parameter(
            (torch.randn(epr, 2 * ffn, hidden, device=dev, generator=g) * hidden ** -0.5).bfloat16())
        self.w_down = torch.nn.Parameter(
            (torch.randn(epr, hidden, ffn, device=dev, generator=g) * ffn ** -0.5).bfloat16())
        self.topk, self.renorm = topk, renorm

    def forward(self, x):
        logits = x.float() @ self.gate
        ids, gw = RouterFunction.apply(logits, self.topk, self.renorm)
        return EpMoEFunction.apply(self.experts, x, ids, gw, self.w_up, self.w_down)
