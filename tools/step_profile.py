"""One Mixtral-shape (or --config) step with the device timeline on: per-MegaKernel role
statistics and overlap fraction; optional --ncu mode runs 1 warm-up + 1 step only (for ncu)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from oracle import pyoracle as po
from paper_2604_19241_b200 import moe as M
from paper_2604_19241_b200.model import choose_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--out", default="gpurun_out")
ap.add_argument("--cfg", default="")
ap.add_argument("--sms", type=int, default=0, help="persistent-grid SM budget (0: all)")
ap.add_argument("--opt", action="append", default=[], help="eplab_set_option name=value")
args = ap.parse_args()
H, F, E, k, T = bench.CONFIGS[args.config]
sel, gw = po.Oracle().sample_routing(E, k, T, 1, 7)
ids = torch.from_numpy(sel[0].reshape(T, k).copy()).cuda(); gws = torch.from_numpy(gw[0].reshape(T, k).copy()).cuda()
g = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn(T, H, device="cuda", generator=g).bfloat16(); dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
L = M.EpMoE(H, F, E, k, T)
if args.sms:
    L.set_sm_budget(args.sms)
cfg = choose_config(H, F, E, k, T, 1, n_sm=args.sms or 148) if not args.cfg else M.TuneConfig(*[int(v) for v in args.cfg.split(",")])
L.set_tune_config(cfg)
for o in args.opt:
    L.set_option(o.split("=")[0], int(o.split("=")[1]))
y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(w_up),
           dw_down=torch.empty_like(w_down), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
def step():
    L.plan(ids, gws); L.dispatch_group_gemm(x, w_up); L.group_gemm_combine(w_down, y); L.backward(dy, w_up, w_down, out=out)
step(); L.check()
if args.ncu:
    step(); torch.cuda.synchronize(); sys.exit(0)
L.timeline_enable(1 << 20)
os.makedirs(args.out, exist_ok=True)
stats = {}
for name, fn in [("fwd_dispatch", lambda: (L.plan(ids, gws), L.dispatch_group_gemm(x, w_up))),
                 ("fwd_combine", lambda: L.group_gemm_combine(w_down, y)),
                 ("bwd_dispatch", lambda: L._dispatch_bwd(dy, w_down, out)),
                 ("bwd_combine", lambda: L._combine_bwd(w_up, out))]:
    torch.cuda.synchronize(); fn(); torch.cuda.synchronize()
    path = os.path.join(args.out, f"trace_{args.config}_{name}.json")
    ov = L.timeline_export(path)
    ev = json.load(open(path))["traceEvents"]
    t0 = min(e["ts"] for e in ev); t1 = max(e["ts"] + e["dur"] for e in ev)
    roles = {}
    for e in ev:
        r = roles.setdefault(e["name"], [0, 0.0, 1e30, 0.0])
        r[0] += 1; r[1] += e["dur"]; r[2] = min(r[2], e["ts"] - t0); r[3] = max(r[3], e["ts"] + e["dur"] - t0)
    comp_busy = roles.get("comp", [0, 0.0])[1]
    stats[name] = {"span_us": t1 - t0, "overlap_frac": ov,
                   "roles": {k2: {"n": v[0], "mean_us": v[1] / v[0], "first_start_us": v[2], "last_end_us": v[3]} for k2, v in roles.items()},
                   "comp_sm_util": comp_busy / ((t1 - t0) * 148)}
print(json.dumps(stats, indent=1))
json.dump(stats, open(os.path.join(args.out, f"timeline_{args.config}.json"), "w"), indent=1)
