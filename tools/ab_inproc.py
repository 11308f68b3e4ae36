"""In-process A/B of launch options (eplab_set_option knobs, or tune configs): the variants
alternate step by step in one process, so power/thermal drift hits all of them alike.
  python tools/ab_inproc.py --config qwen3 --variants "EPLAB_SPARE=1;EPLAB_SPARE=0" --rounds 20
  a variant is ';'-separated; each is a ','-list of KNOB=VAL (eplab_set_option names or the old EPLAB_*
  spellings) or tune=n_disp:n_relay:n_comb:n_red:w
"""
import argparse, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from oracle import pyoracle as po
from paper_2604_19241_b200 import moe as M
from paper_2604_19241_b200.model import choose_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3")
ap.add_argument("--variants", required=True)
ap.add_argument("--rounds", type=int, default=20)
ap.add_argument("--shape", default="", help="H,F,E,k,T instead of a bench config")
ap.add_argument("--whole", action="store_true",
                help="events at step boundaries only (kernels back to back, e.g. for programmatic dependent launch)")
args = ap.parse_args()
H, F, E, k, T = [int(v) for v in args.shape.split(",")] if args.shape else bench.CONFIGS[args.config]
if args.shape:
    args.config = "shape_" + args.shape.replace(",", "_")
sel, gw = po.Oracle().sample_routing(E, k, T, 1, 7)
ids = torch.from_numpy(sel[0].reshape(T, k).copy()).cuda()
gws = torch.from_numpy(gw[0].reshape(T, k).copy()).cuda()
g = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
L = M.EpMoE(H, F, E, k, T)
base_cfg = choose_config(H, F, E, k, T, 1)
y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(w_up),
           dw_down=torch.empty_like(w_down), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
st = torch.cuda.current_stream()
variants = [v.strip() for v in args.variants.split(";")]


# knob names of eplab_set_option (the old EPLAB_* spellings are accepted) and their defaults
ALIASES = {"EPLAB_SPARE": "spare", "EPLAB_COMM": "comm_bulk", "EPLAB_DBG": "dbg", "EPLAB_RGP": "rgp",
           "EPLAB_TNGP": "tngp", "EPLAB_TNGP_D": "tngp_d", "EPLAB_BWD_DISP_SCALE": "bwd_disp_scale",
           "EPLAB_ENGINE": "engine_pair"}
DEFAULTS = {"spare": 3, "comm_bulk": 0, "dbg": 0, "rgp": 8, "tngp": 4, "tngp_d": 4, "bwd_disp_scale": 2,
            "engine_pair": 1}


def apply(v):
    cfg = base_cfg
    opts = dict(DEFAULTS)  # every variant starts from the defaults
    for kv in [p for p in v.split(",") if p]:
        key, val = kv.split("=")
        if key == "tune":
            cfg = M.TuneConfig(*[int(q) for q in val.split(":")])
        else:
            name = ALIASES.get(key, key)
            opts[name] = {"bulk": 1, "warp": 0, "single": 0, "pair": 1}.get(val, None) if not val.lstrip("-").isdigit() \
                else int(val)
    for name, val in opts.items():
        L.set_option(name, val)
    L.set_tune_config(cfg)


def step_timed():
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    if args.whole:
        ev[0].record(st)
        L.plan(ids, gws); L.dispatch_group_gemm(x, w_up); L.group_gemm_combine(w_down, y)
        L._dispatch_bwd(dy, w_down, out); L._combine_bwd(w_up, out)
        for e in ev[1:]:
            e.record(st)
        return ev
    ev[0].record(st)
    L.plan(ids, gws); L.dispatch_group_gemm(x, w_up); ev[1].record(st)
    L.group_gemm_combine(w_down, y); ev[2].record(st)
    L._dispatch_bwd(dy, w_down, out); ev[3].record(st)
    L._combine_bwd(w_up, out); ev[4].record(st)
    return ev


res = {v: [] for v in variants}
for v in variants:  # warm-up
    apply(v)
    for _ in range(3):
        step_timed()
torch.cuda.synchronize()
for r in range(args.rounds):
    for v in variants:
        apply(v)
        ev = step_timed()
        torch.cuda.synchronize()
        res[v].append([ev[j].elapsed_time(ev[j + 1]) for j in range(4)])
L.check()
for v in variants:
    per = list(zip(*res[v]))
    med = [statistics.median(p) for p in per]
    print(json.dumps({"config": args.config, "variant": v, "median_ms": round(sum(med), 4),
                      "kernels_ms": [round(m, 4) for m in med],
                      "min_step_ms": round(min(sum(s) for s in res[v]), 4)}), flush=True)
