"""BW (bitwise, full batch) vs NB (split-batch) step on a BASELINE shape:
step time of both and the weight-gradient divergence in the reference's PrecisionReport terms
(precision.hpp: elements, non_bitwise, frac_non_bitwise, max_abs_diff, max_rel_diff)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from oracle import pyoracle as po
from paper_2604_19241_b200 import moe as M
from paper_2604_19241_b200.model import choose_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
H, F, E, k, T = bench.CONFIGS[args.config]
sel, gw = po.Oracle().sample_routing(E, k, T, 1, 7)
ids = torch.from_numpy(sel[0].reshape(T, k).copy()).cuda(); gws = torch.from_numpy(gw[0].reshape(T, k).copy()).cuda()
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(T, H, device="cuda", generator=g).bfloat16(); dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
L = M.EpMoE(H, F, E, k, T); L.set_tune_config(choose_config(H, F, E, k, T, 1))


def bw():
    y = L.forward(x, ids, gws, w_up, w_down)
    return y, L.backward(dy, w_up, w_down)


def nb():
    return L.step_split(x, ids, gws, dy, w_up, w_down, n_sub=2)


def timed(fn):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        r = fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / args.steps, r


t_bw, (y0, g0) = timed(bw)
t_nb, (y1, g1) = timed(nb)
L.check()
rep = {"config": args.config, "bw_ms": t_bw, "nb_ms": t_nb, "nb_speedup": t_bw / t_nb,
       "y_bitwise": bool(torch.equal(y0, y1)), "dx_bitwise": bool(torch.equal(g0["dx"], g1["dx"])),
       "dgate_bitwise": bool(torch.equal(g0["dgate"], g1["dgate"]))}
for key in ("dw_up", "dw_down"):
    a, b = g0[key].float(), g1[key].float()
    d = (a - b).abs()
    rel = d / a.abs().clamp_min(1e-30)
    rep[key] = {"elements": a.numel(), "non_bitwise": int((g0[key] != g1[key]).sum()),
                "frac_non_bitwise": float((g0[key] != g1[key]).float().mean()),
                "max_abs_diff": float(d.max()), "max_rel_diff": float(rel[a != 0].max())}
print(json.dumps(rep))
L.close()
