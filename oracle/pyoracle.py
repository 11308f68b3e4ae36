"""ctypes bindings to the CPU ORACLE (liborc.so) and the reference build (_ref/libeplab_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libeplab_ref.so")


class Hw(C.Structure):
    _fields_ = [("n_sm", C.c_int), ("p_peak", C.c_double), ("bw_hbm", C.c_double),
                ("bw_nvl", C.c_double), ("w_sat", C.c_double), ("tau_sync", C.c_double),
                ("world_size", C.c_int)]


class Shape(C.Structure):
    _fields_ = [("h_dim", C.c_int), ("h_inter", C.c_int), ("n_exp", C.c_int), ("topk", C.c_int),
                ("n_tok", C.c_longlong), ("s_tok", C.c_longlong), ("b_m", C.c_int), ("b_n", C.c_int),
                ("mu_n", C.c_int), ("mu_w", C.c_int * 8), ("mu_v", C.c_double * 8)]


class Cfg(C.Structure):
    _fields_ = [("n_disp", C.c_int), ("n_relay", C.c_int), ("n_comb", C.c_int), ("n_red", C.c_int),
                ("w", C.c_int)]

    def tup(self):
        return (self.n_disp, self.n_relay, self.n_comb, self.n_red, self.w)


class Traffic(C.Structure):
    _fields_ = [("v_allgather", C.c_double), ("v_alltoall", C.c_double),
                ("v_megakernel_nvl", C.c_double), ("v_megakernel_hbm", C.c_double)]


class Breakdown(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_up", "t_down", "l_swiglu", "l_disp", "l_up", "l_comb",
                                          "l_down", "t_red", "l_s1", "l_s2", "l_total")] + \
               [("n_tiles_up", C.c_longlong), ("n_tiles_down", C.c_longlong)] + \
               [(n, C.c_double) for n in ("w_gap", "w_red", "w_rem")]


class LayerDims(C.Structure):
    _fields_ = [("world", C.c_int), ("n_exp", C.c_int), ("topk", C.c_int), ("H", C.c_int),
                ("F", C.c_int), ("n_tok", C.c_longlong)]


def make_hw(n_sm, p_peak, bw_hbm, bw_nvl, world, w_sat=1024.0, tau_sync=2e-6):
    return Hw(n_sm, p_peak, bw_hbm, bw_nvl, w_sat, tau_sync, world)


def make_shape(h_dim, h_inter, n_exp, topk, n_tok, s_tok=0, b_m=128, b_n=256,
               mu=((8, 0.7), (16, 0.65), (32, 0.6))):
    s = Shape()
    s.h_dim, s.h_inter, s.n_exp, s.topk, s.n_tok = h_dim, h_inter, n_exp, topk, n_tok
    s.s_tok = s_tok if s_tok else 2 * h_dim
    s.b_m, s.b_n = b_m, b_n
    s.mu_n = len(mu)
    for i, (w, v) in enumerate(mu):
        s.mu_w[i], s.mu_v[i] = w, v
    return s


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class _Lib:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing (build with `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.pre = prefix
        L = self.lib
        for name in ("round_to_bf16",):
            f = getattr(L, prefix + name)
            f.restype = C.c_float
            f.argtypes = [C.c_float]
        f = getattr(L, prefix + "fold")
        f.restype = C.c_float

    def fn(self, name):
        return getattr(self.lib, self.pre + name)

    # a2
    def sample_routing(self, n_exp, topk, n_tok, world, seed):
        sel = np.zeros(world * n_tok * topk, np.int32)
        gw = np.zeros(world * n_tok * topk, np.float32)
        rc = self.fn("sample_routing")(n_exp, topk, C.c_longlong(n_tok), world, C.c_uint64(seed),
                                       _p(sel), _p(gw))
        if rc:
            raise ValueError(f"sample_routing rc={rc}")
        return sel.reshape(world, n_tok * topk), gw.reshape(world, n_tok * topk)

    # a5
    def token_map(self, sel, n_exp, topk):
        sel = np.ascontiguousarray(sel, np.int32)
        world = sel.shape[0]
        n_tok = sel.shape[1] // topk
        n = world * n_tok * topk
        tr = np.zeros(n, np.int32)
        le = np.zeros(n, np.int32)
        off = np.zeros(n, np.int64)
        epr = n_exp // world if world else 0
        rt = np.zeros(world * max(epr, 1), np.int64)
        sb = np.zeros(world * max(epr, 1), np.int64)
        rc = self.fn("token_map")(_p(sel), world, n_exp, C.c_longlong(n_tok), topk, _p(tr), _p(le),
                                  _p(off), _p(rt), _p(sb))
        if rc:
            raise ValueError(f"token_map rc={rc}")
        shp = (world, n_tok * topk)
        return tr.reshape(shp), le.reshape(shp), off.reshape(shp), rt, sb

    def round_to_bf16(self, x):
        return self.fn("round_to_bf16")(x)

    def fold(self, w, v, bf16):
        w = np.ascontiguousarray(w, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        return self.fn("fold")(_p(w), _p(v), len(w), int(bf16))

    def predict_latency(self, shape, hw, cfg, traffic, redistributed=False):
        b = Breakdown()
        rc = self.fn("predict_latency")(C.byref(shape), C.byref(hw), C.byref(cfg), C.byref(traffic),
                                        int(redistributed), C.byref(b))
        if rc:
            raise ValueError(f"predict_latency rc={rc}")
        return b


class Oracle(_Lib):
    def __init__(self):
        super().__init__(ORC_PATH, "orc_")
        L = self.lib
        L.orc_effective_bandwidth.restype = C.c_double
        L.orc_effective_bandwidth.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        L.orc_swiglu.restype = C.c_double
        L.orc_tiles_up.restype = C.c_longlong
        L.orc_tiles_down.restype = C.c_longlong

    def send_schedule(self, tr, le, off, topk, world, epr, rank):
        n = tr.shape[1]
        out = (np.zeros(n, np.int64), np.zeros(n, np.int32), np.zeros(n, np.int32),
               np.zeros(n, np.int32), np.zeros(n, np.int64))
        self.lib.orc_send_schedule(_p(np.ascontiguousarray(tr[rank])), _p(np.ascontiguousarray(le[rank])),
                                   _p(np.ascontiguousarray(off[rank])), C.c_longlong(n // topk), topk,
                                   world, epr, *[_p(a) for a in out])
        return out

    def primary_flags(self, item_token, item_dst_rank, world):
        p = np.zeros(len(item_token), np.int8)
        self.lib.orc_primary_flags(_p(item_token), _p(item_dst_rank), C.c_longlong(len(item_token)),
                                   world, _p(p))
        return p

    def stirling2(self, n, k):
        hi, lo = C.c_uint64(), C.c_uint64()
        rc = self.lib.orc_stirling2(n, k, C.byref(hi), C.byref(lo))
        if rc:
            raise ValueError("stirling2")
        return (hi.value << 64) | lo.value

    def distinct_rank_distribution(self, world, topk):
        x = min(world, topk)
        hi = np.zeros(x, np.uint64)
        lo = np.zeros(x, np.uint64)
        pr = np.zeros(x, np.float64)
        ex, sv = C.c_double(), C.c_double()
        rc = self.lib.orc_distinct_rank_distribution(world, topk, _p(hi), _p(lo), _p(pr), C.byref(ex),
                                                     C.byref(sv))
        if rc:
            raise ValueError("distinct_rank_distribution")
        nums = [(int(h) << 64) | int(l) for h, l in zip(hi, lo)]
        return nums, pr, ex.value, sv.value

    def volume_expected(self, n_tok, topk, s_tok, world, remote_only=False):
        t = Traffic()
        rc = self.lib.orc_volume_expected(C.c_longlong(n_tok), topk, C.c_longlong(s_tok), world,
                                          int(remote_only), C.byref(t))
        if rc:
            raise ValueError("volume_expected")
        return t

    def volume_exact(self, sel, n_exp, topk, s_tok, remote_only=False):
        sel = np.ascontiguousarray(sel, np.int32)
        t = Traffic()
        world = sel.shape[0]
        rc = self.lib.orc_volume_exact(_p(sel), world, n_exp, C.c_longlong(sel.shape[1] // topk), topk,
                                       C.c_longlong(s_tok), int(remote_only), C.byref(t))
        if rc:
            raise ValueError("volume_exact")
        return t

    def space_sizes(self, n_sm):
        a, b, c = C.c_longlong(), C.c_longlong(), C.c_longlong()
        rc = self.lib.orc_space_sizes(n_sm, C.byref(a), C.byref(b), C.byref(c))
        if rc:
            raise ValueError("space")
        return a.value, b.value, c.value

    def search(self, shape, hw, traffic, redistributed=False):
        best, lmin, ev = Cfg(), C.c_double(), C.c_longlong()
        rc = self.lib.orc_search(C.byref(shape), C.byref(hw), C.byref(traffic), int(redistributed),
                                 C.byref(best), C.byref(lmin), C.byref(ev))
        if rc:
            raise ValueError("search")
        return best, lmin.value, ev.value

    def moe_layer(self, world, n_exp, topk, H, F, sel, gw, x, w_up, w_down, dy, threads=0,
                  want_grads=True, want_dw=True):
        """bf16 tensors as uint16 numpy arrays. Returns dict of outputs (want_dw=False skips the
        weight gradients: the row-local outputs of a token sample need only its rows)."""
        n_tok = sel.shape[1] // topk
        d = LayerDims(world, n_exp, topk, H, F, n_tok)
        y = np.zeros((world, n_tok, H), np.uint16)
        dx = np.zeros((world, n_tok, H), np.uint16) if want_grads else None
        dg = np.zeros((world, n_tok * topk), np.float32) if want_grads else None
        dwu = np.zeros((n_exp, 2 * F, H), np.uint16) if (want_grads and want_dw) else None
        dwd = np.zeros((n_exp, H, F), np.uint16) if (want_grads and want_dw) else None
        arrs = [np.ascontiguousarray(a) for a in (sel.astype(np.int32), gw.astype(np.float32), x, w_up,
                                                  w_down)]
        dyc = np.ascontiguousarray(dy) if (dy is not None and want_grads) else None
        nul = C.c_void_p(0)
        rc = self.lib.orc_moe_layer(C.byref(d), *[_p(a) for a in arrs],
                                    _p(dyc) if dyc is not None else nul, _p(y),
                                    _p(dx) if dx is not None else nul, _p(dg) if dg is not None else nul,
                                    _p(dwu) if dwu is not None else nul,
                                    _p(dwd) if dwd is not None else nul, threads)
        if rc:
            raise ValueError(f"moe_layer rc={rc}")
        return {"y": y, "dx": dx, "dgate": dg, "dw_up": dwu, "dw_down": dwd}

    def fill_normal_bf16(self, n, seed, scale=1.0):
        out = np.zeros(n, np.uint16)
        self.lib.orc_fill_normal_bf16(_p(out), C.c_longlong(n), C.c_uint64(seed), C.c_float(scale))
        return out

    # §8 f1 router (semantics defined in eplab_oracle.h)
    def router_topk(self, logits, topk, renorm=True):
        lg = np.ascontiguousarray(logits, np.float32)
        T, E = lg.shape
        ids = np.zeros((T, topk), np.int32)
        gw = np.zeros((T, topk), np.float32)
        rc = self.lib.orc_router_topk(_p(lg), C.c_longlong(T), E, topk, int(renorm), _p(ids), _p(gw))
        if rc:
            raise ValueError(f"router_topk rc={rc}")
        return ids, gw

    def router_topk_bwd(self, logits, ids, gw, dgate, renorm=True):
        lg = np.ascontiguousarray(logits, np.float32)
        T, E = lg.shape
        ids = np.ascontiguousarray(ids, np.int32)
        gw = np.ascontiguousarray(gw, np.float32)
        dg = np.ascontiguousarray(dgate, np.float32)
        out = np.zeros((T, E), np.float32)
        rc = self.lib.orc_router_topk_bwd(_p(lg), _p(ids), _p(gw), _p(dg), C.c_longlong(T), E, ids.shape[1],
                                          int(renorm), _p(out))
        if rc:
            raise ValueError(f"router_topk_bwd rc={rc}")
        return out


class Reference(_Lib):
    """The unmodified reference eplab (oracle/_ref)."""

    def __init__(self):
        super().__init__(REF_PATH, "ref_")

    def send_schedule(self, sel, n_exp, topk, rank):
        sel = np.ascontiguousarray(sel, np.int32)
        world = sel.shape[0]
        n = sel.shape[1]
        out = (np.zeros(n, np.int64), np.zeros(n, np.int32), np.zeros(n, np.int32),
               np.zeros(n, np.int32), np.zeros(n, np.int64))
        rc = self.lib.ref_send_schedule(_p(sel), world, n_exp, C.c_longlong(n // topk), topk, rank,
                                        *[_p(a) for a in out])
        if rc:
            raise ValueError(f"ref_send_schedule rc={rc}")
        return out

    def distinct_rank_distribution(self, world, topk):
        x = min(world, topk)
        lo = np.zeros(x, np.uint64)
        pr = np.zeros(x, np.float64)
        ex, sv = C.c_double(), C.c_double()
        rc = self.lib.ref_distinct_rank_distribution(world, topk, _p(lo), _p(pr), C.byref(ex), C.byref(sv))
        if rc:
            raise ValueError("ref distinct")
        return [int(v) for v in lo], pr, ex.value, sv.value

    def volume_expected(self, shape, hw, remote_only=False):
        t = Traffic()
        rc = self.lib.ref_volume_expected(C.byref(shape), C.byref(hw), int(remote_only), C.byref(t))
        if rc:
            raise ValueError("ref volume_expected")
        return t

    def volume_exact(self, sel, shape, hw, remote_only=False):
        sel = np.ascontiguousarray(sel, np.int32)
        t = Traffic()
        rc = self.lib.ref_volume_exact(_p(sel), C.byref(shape), C.byref(hw), sel.shape[0], int(remote_only),
                                       C.byref(t))
        if rc:
            raise ValueError("ref volume_exact")
        return t

    def search(self, shape, hw, traffic, workers=1):
        best, lmin, ev, wall = Cfg(), C.c_double(), C.c_longlong(), C.c_double()
        rc = self.lib.ref_search(C.byref(shape), C.byref(hw), C.byref(traffic), workers, C.byref(best),
                                 C.byref(lmin), C.byref(ev), C.byref(wall))
        if rc:
            raise ValueError(f"ref search rc={rc}")
        return best, lmin.value, ev.value, wall.value

    def space_sizes(self, n_sm):
        a, b, c = C.c_longlong(), C.c_longlong(), C.c_longlong()
        rc = self.lib.ref_space_sizes(n_sm, C.byref(a), C.byref(b), C.byref(c))
        if rc:
            raise ValueError("ref space")
        return a.value, b.value, c.value

    def build_task_list(self, sel, shape, cfg, rank):
        sel = np.ascontiguousarray(sel, np.int32)
        cs = np.zeros(2 * max(cfg.n_disp, 1), np.int64)
        rr = np.zeros(2 * max(cfg.n_relay, 1), np.int64)
        nc = C.c_longlong()
        rc = self.lib.ref_build_task_list(_p(sel), sel.shape[0], C.byref(shape), C.byref(cfg), rank, _p(cs),
                                          _p(rr), C.byref(nc))
        if rc:
            raise ValueError(f"ref build_task_list rc={rc}")
        return cs.reshape(-1, 2)[:cfg.n_disp], rr.reshape(-1, 2)[:cfg.n_relay], nc.value

    def time_addressing(self, n_exp, topk, n_tok, world, seed):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        rc = self.lib.ref_time_addressing(n_exp, topk, C.c_longlong(n_tok), world, C.c_uint64(seed),
                                          C.byref(a), C.byref(b), C.byref(c))
        if rc:
            raise ValueError("ref time")
        return a.value, b.value, c.value


def has_reference():
    return os.path.exists(REF_PATH)
