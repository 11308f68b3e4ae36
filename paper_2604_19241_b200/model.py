"""Performance model + tuner of the MegaKernels (reference perf_model.cpp /
tuner.cpp), exposed from the C++ host library through the C-ABI.

  predict_latency(...)  reference-compatible forward model (Alg. 2)
  search(...)           reference exhaustive tuner
  predict_layer(...)    B200 fwd+bwd model of this build's four MegaKernels
  choose_config(...)    launch parameters for a layer shape (search_layer)
"""
import ctypes as C

from . import _lib
from .moe import TuneConfig, _check


class Hw(C.Structure):
    _fields_ = [("n_sm", C.c_int), ("p_peak", C.c_double), ("bw_hbm", C.c_double), ("bw_nvl", C.c_double),
                ("w_sat", C.c_double), ("tau_sync", C.c_double), ("world_size", C.c_int)]


class Shape(C.Structure):
    _fields_ = [("h_dim", C.c_int), ("h_inter", C.c_int), ("n_exp", C.c_int), ("topk", C.c_int),
                ("n_tok", C.c_longlong), ("s_tok", C.c_longlong), ("b_m", C.c_int), ("b_n", C.c_int),
                ("mu_n", C.c_int), ("mu_w", C.c_int * 8), ("mu_v", C.c_double * 8)]


class Traffic(C.Structure):
    _fields_ = [("v_allgather", C.c_double), ("v_alltoall", C.c_double), ("v_megakernel_nvl", C.c_double),
                ("v_megakernel_hbm", C.c_double)]


class Breakdown(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_up", "t_down", "l_swiglu", "l_disp", "l_up", "l_comb", "l_down",
                                          "t_red", "l_s1", "l_s2", "l_total")] + \
               [("n_tiles_up", C.c_longlong), ("n_tiles_down", C.c_longlong)] + \
               [(n, C.c_double) for n in ("w_gap", "w_red", "w_rem")]


class Calib(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mu", "tile_overhead", "comm_bw_per_sm", "relay_bw_per_sm",
                                          "reduce_bw", "launch", "epi_bw_per_sm", "spare_sm_equiv",
                                          "hbm_overlap", "startup")]


class LayerPrediction(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("fwd_dispatch", "fwd_combine", "bwd_dispatch", "bwd_combine",
                                          "total", "t_gemm_bound", "t_nvl_bound")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


# B200 calibration of this build (DESIGN.md §Performance model; refit by tools/fit_model.py)
# fitted over 94 measured cases, EP=1 and EP=2/4/8 on virtual ranks (profiles/r02_perf_model_validation.md)
B200_CALIB = Calib(0.935, 0.2e-6, 28.94e9, 8.88e9, 6.5e12, 31.45e-6, 199.1e9, 29.04, 0.528, 2.0)


def hw(world, n_sm=148, p_peak=1408.1e12, bw_hbm=6468.9e9, bw_nvl=770e9, w_sat=1024.0, tau_sync=1e-6):
    return Hw(n_sm, p_peak, bw_hbm, bw_nvl, w_sat, tau_sync, world)


def shape(h_dim, h_inter, n_exp, topk, n_tok, s_tok=0, b_m=128, b_n=256,
          mu=((8, 0.7), (16, 0.65), (32, 0.6))):
    s = Shape()
    s.h_dim, s.h_inter, s.n_exp, s.topk, s.n_tok = h_dim, h_inter, n_exp, topk, n_tok
    s.s_tok, s.b_m, s.b_n = s_tok or 2 * h_dim, b_m, b_n
    s.mu_n = len(mu)
    for i, (w, v) in enumerate(mu):
        s.mu_w[i], s.mu_v[i] = w, v
    return s


def _L():
    L = _lib.lib()
    return L


def sample_routing(n_exp, topk, n_tok, world, seed):
    """The reference's synthetic routing (routing.cpp:32-73, sample_routing) from this library's
    host implementation: sel int32 / gw fp32, [world][n_tok * topk]."""
    import numpy as np
    sel = np.empty((world, n_tok * topk), dtype=np.int32)
    gw = np.empty((world, n_tok * topk), dtype=np.float32)
    L = _L()
    L.eplab_sample_routing.argtypes = [C.c_int, C.c_int, C.c_longlong, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p]
    L.eplab_sample_routing.restype = C.c_int
    _check(L.eplab_sample_routing(n_exp, topk, n_tok, world, seed, sel.ctypes.data, gw.ctypes.data))
    return sel, gw


def rank_token_map(sel_rank, counts_all, rank, world, n_exp, topk):
    """One rank's Alg. 1 token map from its own routing + the all-gathered per-expert counts of every
    rank (eplab_host_rank_token_map): (target_rank, local_expert, offset) per (t, j)."""
    import numpy as np
    sel = np.ascontiguousarray(sel_rank, np.int32).reshape(-1)
    cnt = np.ascontiguousarray(counts_all, np.int64).reshape(world, n_exp)
    n = sel.size
    tr, le, off = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int64)
    L = _L()
    L.eplab_host_rank_token_map.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_longlong,
                                            C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.eplab_host_rank_token_map.restype = C.c_int
    _check(L.eplab_host_rank_token_map(sel.ctypes.data, cnt.ctypes.data, rank, world, n_exp, n // topk, topk,
                                       tr.ctypes.data, le.ctypes.data, off.ctypes.data))
    return tr, le, off


def volume_expected(s, h, remote_only=False):
    t = Traffic()
    _check(_L().eplab_volume_expected(C.byref(s), C.byref(h), int(remote_only), C.byref(t)))
    return t


def predict_latency(s, h, cfg, traffic, redistributed=False):
    b = Breakdown()
    _check(_L().eplab_predict_latency(C.byref(s), C.byref(h), C.byref(cfg), C.byref(traffic),
                                      int(redistributed), C.byref(b)))
    return b


def search(s, h, traffic, n_workers=0, redistributed=False):
    best, lmin, ev = TuneConfig(), C.c_double(), C.c_longlong()
    _check(_L().eplab_search(C.byref(s), C.byref(h), C.byref(traffic), n_workers, int(redistributed),
                             C.byref(best), C.byref(lmin), C.byref(ev)))
    return best, lmin.value, ev.value


def predict_layer(s, h, cfg, calib=None):
    p = LayerPrediction()
    _check(_L().eplab_predict_layer(C.byref(s), C.byref(h), C.byref(cfg),
                                    C.byref(calib or B200_CALIB), C.byref(p)))
    return p


def search_layer(s, h, calib=None):
    best, lmin, ev = TuneConfig(), C.c_double(), C.c_longlong()
    _check(_L().eplab_search_layer(C.byref(s), C.byref(h), C.byref(calib or B200_CALIB), C.byref(best),
                                   C.byref(lmin), C.byref(ev)))
    return best, lmin.value, ev.value


def choose_config(H, F, E, k, tokens, world, n_sm=148, spare=True):
    """TuneConfig for one layer shape from the B200 model (n_red = all SMs; w = 8). spare=False:
    the GEMM CTAs' spare warps stay out of the comm pool (eplab_set_comm_options bit 0 clear)."""
    calib = B200_CALIB
    if not spare:
        calib = Calib(*[getattr(B200_CALIB, n) for n, _ in Calib._fields_])
        calib.spare_sm_equiv = 0.0
    best, _, _ = search_layer(shape(H, F, E, k, tokens), hw(world, n_sm=n_sm), calib)
    best.n_red = n_sm
    if not spare and best.n_disp == 0:
        best.n_disp = 1  # somebody must move the rows
    # No floor on n_disp (round 1 forced >= 16 comm CTAs): the model's GEMM start-up term (the first
    # wave's rows landing at the comm pool's rate) and the comm CTAs' SM time now order the choices
    # as measured -- in-process A/B, profiles/r02_ndisp_ab.txt: 0 comm CTAs is best or within noise
    # for Mixtral, Qwen3, DSv3 and the top-k sweep shapes.
    return best
