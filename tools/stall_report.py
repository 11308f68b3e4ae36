"""Stall accounting of the GEMM roles per MegaKernel (device timeline on, one EP=1 step):
MMA issuer (per CTA pair): waiting for a tile (scheduler / scoreboard), for a free accumulator
(epilogue), for operand stages (TMA producer); epilogue warp 0 (per CTA): waiting for the
accumulator, the epilogue, the release after the hand-back -- each as % of the kernel's tile span.
  python tools/step_profile.py-like: python tools/stall_report.py --config qwen3 [--opt dbg=0 ...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_19241_b200 import moe as M  # noqa: E402
from paper_2604_19241_b200.model import choose_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3")
ap.add_argument("--opt", action="append", default=[], help="eplab_set_option name=value")
ap.add_argument("--out", default="gpurun_out")
ap.add_argument("--warm-first", action="store_true", help="one default step before --opt applies (real rows for dbg 512)")
ap.add_argument("--shape", default="", help="H,F,E,k,T instead of a bench config")
args = ap.parse_args()
H, F, E, k, T = [int(v) for v in args.shape.split(",")] if args.shape else bench.CONFIGS[args.config]
if args.shape:
    args.config = "shape_" + args.shape.replace(",", "_")
bench.CONFIGS[args.config] = (H, F, E, k, T)
inp = bench.make_inputs(args.config, 1, 0)
L = M.EpMoE(H, F, E, k, T)
L.set_tune_config(choose_config(H, F, E, k, T, 1))
y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(inp["w_up"]),
           dw_down=torch.empty_like(inp["w_down"]), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
steps = [("fwd_dispatch", lambda: (L.plan(inp["ids"], inp["gws"]), L.dispatch_group_gemm(inp["x"], inp["w_up"]))),
         ("fwd_combine", lambda: L.group_gemm_combine(inp["w_down"], y)),
         ("bwd_dispatch", lambda: L._dispatch_bwd(inp["dy"], inp["w_down"], out)),
         ("bwd_combine", lambda: L._combine_bwd(inp["w_up"], out))]
for _, fn in steps if args.warm_first else []:
    fn()
for o in args.opt:
    n, v = o.split("=")
    L.set_option(n, int(v))
for _, fn in steps:  # warm-up step
    fn()
L.check()
L.timeline_enable(1 << 20)
os.makedirs(args.out, exist_ok=True)
NAMES = {-9001: "mma_wait_tile", -9002: "mma_wait_acc", -9003: "mma_wait_ops",
         -9004: "epi_wait_acc", -9005: "epi_work", -9006: "epi_release",
         # dbg 1024: down-dgrad epilogue sections of warp 0, cycles (shares of their sum below)
         -9011: "sec_loads_issue", -9012: "sec_tmem_ld", -9013: "sec_compute", -9014: "sec_stage_acquire",
         -9015: "sec_stage_store",
         # dbg 2048: comm-round sections of each comm warp (lane 0), cycles
         -9021: "com_meta", -9022: "com_copy", -9023: "com_release",
         -9024: "com_loads", -9025: "com_stores",  # the copy section split: loads of a pass, its stores
         # MMA issuer per tile type: main-loop time and its operand waits (NT tiles / transposed tiles)
         -9031: "ty_loop_nt", -9032: "ty_loop_tn", -9033: "ty_ops_nt", -9034: "ty_ops_tn"}
rep = {"config": args.config, "opts": args.opt}
for name, fn in steps:
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    path = os.path.join(args.out, f"stall_{args.config}_{name}.json")
    L.timeline_export(path)
    ev = json.load(open(path))["traceEvents"]
    tiles = [e for e in ev if e["name"] == "comp" and e["args"]["task"] >= 0]
    if not tiles:
        continue
    t0 = min(e["ts"] for e in tiles)
    t1 = max(e["ts"] + e["dur"] for e in tiles)
    span = t1 - t0
    acc = {}
    for e in ev:
        tid = e["args"]["task"]
        if tid in NAMES:
            a = acc.setdefault(NAMES[tid], [0.0, 0])
            a[0] += e["dur"]
            a[1] += 1
    rep[name] = {"tile_span_us": round(span, 1), "tiles": len(tiles),
                 **{n: round(100.0 * s / c / span, 1) for n, (s, c) in acc.items() if n[:4] not in ("sec_", "com_", "ty_l", "ty_o")}}
    for ty in ("nt", "tn"):  # operand-wait share of each tile type's main loops
        lp, op = acc.get("ty_loop_" + ty, (0.0, 0))[0], acc.get("ty_ops_" + ty, (0.0, 0))[0]
        if lp > 0:
            rep[name]["ops_wait_in_loop_" + ty] = round(100.0 * op / lp, 1)
            rep[name]["loop_us_per_pair_" + ty] = round(lp / max(1, acc["ty_loop_" + ty][1]), 1)
    com = {n: (s, c) for n, (s, c) in acc.items() if n.startswith("com_")}
    if com:
        rep[name]["comm_round_cycles"] = {n: round(s * 1000.0 / c) for n, (s, c) in com.items()}
        rep[name]["comm_rounds"] = com["com_meta"][1]
    sec = {n: s for n, (s, c) in acc.items() if n.startswith("sec_")}
    if sec:
        rep[name]["epi_sections_pct"] = {n: round(100.0 * s / sum(sec.values()), 1) for n, s in sec.items()}
        rep[name]["epi_cycles_per_tile"] = round(sum(sec.values()) * 1000.0 / acc["sec_tmem_ld"][1])
L.check()
print(json.dumps(rep), flush=True)
