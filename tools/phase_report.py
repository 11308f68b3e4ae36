"""Per-tile-type phases of the four MegaKernels from the device timeline (one EP=1 step): for each
GEMM tile type (up / down / down-dgrad / down-wgrad / up-dgrad / up-wgrad) the number of tiles,
first start, last end and mean duration, plus the comm / reduce role spans, in us from the
kernel's first record. Traces go to --out (default /tmp, they are large).
  python tools/phase_report.py --config qwen3 [--opt dbg=512 ...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_19241_b200 import moe as M  # noqa: E402
from paper_2604_19241_b200.model import choose_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3")
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--out", default="/tmp/phase_report")
ap.add_argument("--cfg", default="", help="n_disp,n_relay,n_comb,n_red,w instead of the model's choice")
ap.add_argument("--warm-first", action="store_true",
                help="one step with default options before --opt applies (dbg 512 then times the GEMM "
                     "roles on the real rows the skipped copies would have moved, not on zeros)")
args = ap.parse_args()
H, F, E, k, T = bench.CONFIGS[args.config]
inp = bench.make_inputs(args.config, 1, 0)
L = M.EpMoE(H, F, E, k, T)
cfg = M.TuneConfig(*[int(v) for v in args.cfg.split(",")]) if args.cfg else choose_config(H, F, E, k, T, 1)
L.set_tune_config(cfg)
y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(inp["w_up"]),
           dw_down=torch.empty_like(inp["w_down"]), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
steps = [("fwd_dispatch", lambda: (L.plan(inp["ids"], inp["gws"]), L.dispatch_group_gemm(inp["x"], inp["w_up"]))),
         ("fwd_combine", lambda: L.group_gemm_combine(inp["w_down"], y)),
         ("bwd_dispatch", lambda: L._dispatch_bwd(inp["dy"], inp["w_down"], out)),
         ("bwd_combine", lambda: L._combine_bwd(inp["w_up"], out))]
if args.warm_first:
    for _, fn in steps:
        fn()
    L.check()
for o in args.opt:
    n, v = o.split("=")
    L.set_option(n, int(v))
for _, fn in steps:
    fn()
L.check()
# tile counts per type (CTA-pair engine): 256-row pairs per expert x column blocks
cnt = np.bincount(inp["ids"].cpu().numpy().reshape(-1), minlength=E)
mpairs = int(sum((-(-int(c) // 128) + 1) // 2 for c in cnt))
n_pre = cfg.n_disp + cfg.n_relay
first = {"fwd_dispatch": ("up", mpairs * (F // 128)), "fwd_combine": ("down", mpairs * (H // 256)),
         "bwd_dispatch": ("down_dgrad", mpairs * (F // 256)), "bwd_combine": ("up_dgrad", mpairs * (H // 256))}
second = {"bwd_dispatch": "down_wgrad", "bwd_combine": "up_wgrad"}
L.timeline_enable(1 << 20)
os.makedirs(args.out, exist_ok=True)
rep = {"config": args.config, "opts": args.opt, "tune": [cfg.n_disp, cfg.n_relay, cfg.n_comb, cfg.n_red, cfg.w]}
for name, fn in steps:
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    path = os.path.join(args.out, f"phase_{args.config}_{name}.json")
    L.timeline_export(path)
    ev = json.load(open(path))["traceEvents"]
    t0 = min(e["ts"] for e in ev)
    t1 = max(e["ts"] + e["dur"] for e in ev)
    kinds = {}
    nm1, n1 = first[name]
    for e in ev:
        tid = e["args"]["task"]
        if e["name"] == "comp":
            if tid < 0:
                continue
            kind = nm1 if tid < n_pre + n1 else second.get(name, "post")
        else:
            kind = e["name"]
        s = kinds.setdefault(kind, [0, 0.0, 1e30, 0.0])
        s[0] += 1
        s[1] += e["dur"]
        s[2] = min(s[2], e["ts"] - t0)
        s[3] = max(s[3], e["ts"] + e["dur"] - t0)
    rep[name] = {"span_us": round(t1 - t0, 1),
                 **{kd: {"n": v[0], "mean_us": round(v[1] / v[0], 2), "first_us": round(v[2], 1),
                         "last_us": round(v[3], 1)} for kd, v in kinds.items()}}
L.check()
print(json.dumps(rep), flush=True)
