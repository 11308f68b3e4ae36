#!/usr/bin/env python
"""Benchmark of the EP-MoE layer fwd+bwd (Dispatch+GroupGEMM / GroupGEMM+Combine MegaKernels).

Workload (BASELINE.json configs[1]): Mixtral-8x7B-style layer, 8 experts top-2, hidden 4096,
ffn 14336, 16K tokens per GPU, experts sharded over the N GPUs (EP=N). One step = device token
map + forward (2 MegaKernels) + backward (2 MegaKernels) over one batch of synthetic tokens
(routing: the reference's sample_routing; random-init bf16 weights). Weak scaling: 16K tokens
per GPU. Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config mixtral|qwen3|dsv3|small]
  (N > 1: torchrun --nproc-per-node N bench.py --gpus N ...)
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (H, F, E, k, tokens per GPU)
    "mixtral": (4096, 14336, 8, 2, 16384),
    "qwen3": (2048, 768, 128, 8, 16384),
    "dsv3": (7168, 2048, 256, 8, 16384),
    "small": (1024, 2048, 8, 2, 4096),
}
CONFIG_DESC = {
    "mixtral": "Mixtral-8x7B-style layer: 8 experts top-2, hidden 4096, ffn 14336, 16K tokens/GPU",
    "qwen3": "Qwen3-30B-A3B-style layer: 128 experts top-8, hidden 2048, moe_ffn 768, 16K tokens/GPU",
    "dsv3": "DeepSeek-V3-style layer: 256 experts top-8, hidden 7168, moe_ffn 2048, 16K tokens/GPU",
    "small": "Small MoE layer: 8 experts top-2, hidden 1024, ffn 2048, 4096 tokens/GPU",
}
METRIC = "MoE layer fwd+bwd tokens/sec"
NVL_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons, timestamped; only samples inside [mark_start, mark_end]
    (the timed region) are summarised."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append((time.time(), parts))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = [r for t, r in self.rows if self.t0 is None or (self.t0 <= t <= (self.t1 or t) + 0.06)]
        if not rows:
            rows = [r for _, r in self.rows[-3:]]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda v: v.replace(".", "", 1).isdigit()
        sm = sorted(float(r[1]) for r in rows if num(r[1]))
        mx = max(float(r[2]) for r in rows if num(r[2]))
        pw = [float(r[3]) for r in rows if num(r[3])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(rows)}


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_bytes_per_step(cfg_name, world):
    """Algorithmic HBM bytes of one fwd+bwd step on one GPU (balanced routing): every tensor of
    the layer read or written once per use: the dispatch copies, both GEMMs' operands
    and outputs, the saved activations, replica slots, the reductions, the weight gradients."""
    H, F, E, k, T = CONFIGS[cfg_name]
    R = T * k                      # rows received per GPU (balanced)
    El = E // world
    row = 2 * H
    w_up, w_down = El * 2 * F * H * 2, El * H * F * 2
    fwd_d = T * row + R * row + R * row + w_up + R * 2 * F * 2 + R * F * 2
    fwd_c = R * F * 2 + w_down + R * row + T * k * row + T * row
    bwd_d = T * row + R * row + T * k * row + R * row + w_down + R * 2 * F * 2 + R * 2 * F * 2 + R * F * 2 \
        + R * row + R * F * 2 + w_down
    bwd_c = R * 4 * F + w_up + R * row + R * 4 * F + R * row + w_up + T * k * row + T * row
    return float(fwd_d + fwd_c + bwd_d + bwd_c)


def algorithmic(cfg_name, world):
    """fwd+bwd FLOPs per token (18 k H F) and NVLink bytes per token per GPU."""
    H, F, E, k, T = CONFIGS[cfg_name]
    flops_tok = 18.0 * k * H * F
    if world > 1:
        from math import comb
        epr = E // world
        e_drem = (world - 1) * (1.0 - comb(E - epr, k) / comb(E, k))
        nvl_tok = 2.0 * (e_drem + k * (world - 1) / world) * 2 * H
    else:
        nvl_tok = 0.0
    return flops_tok, nvl_tok


# ---------------------------------------------------------------------------- CPU baseline
def cpu_layer_sample(cfg_name, n_tok, threads, seed=7):
    """The CPU oracle (port of the reference algorithm + the layer contract) on n_tok tokens of the
    workload (EP=1, full expert weights). Returns seconds."""
    import numpy as np
    from oracle import pyoracle as po
    H, F, E, k, _ = CONFIGS[cfg_name]
    orc = po.Oracle()
    sel, gw = orc.sample_routing(E, k, n_tok, 1, seed)
    rng = np.random.default_rng(seed)
    x = rng.integers(0x3c00, 0x3f80, size=(1, n_tok, H), dtype=np.uint16)
    dy = rng.integers(0x3c00, 0x3f80, size=(1, n_tok, H), dtype=np.uint16)
    w_up = rng.integers(0x3800, 0x3c00, size=(E, 2 * F, H), dtype=np.uint16)
    w_down = rng.integers(0x3800, 0x3c00, size=(E, H, F), dtype=np.uint16)
    t0 = time.perf_counter()
    orc.moe_layer(1, E, k, H, F, sel, gw, x, w_up, w_down, dy, threads=threads)
    return time.perf_counter() - t0


def cpu_baseline(cfg_name, budget_s=12.0):
    """The CPU port timed on two bounded samples (n1 < n2 tokens). A layer fwd+bwd has a per-token
    cost and a per-step cost independent of the token count (writing every expert's weight
    gradient), so the two samples give t(n) = a + b*n; `value` is the workload's T tokens over
    a + b*T (both terms measured, the T-token step itself is not run)."""
    T = CONFIGS[cfg_name][4]
    threads = os.cpu_count() or 1
    n1 = 2
    t1 = cpu_layer_sample(cfg_name, n1, threads)
    n2 = n1 + 8  # a few s of per-token work on top of the per-step cost
    t2 = cpu_layer_sample(cfg_name, n2, threads)
    b = max((t2 - t1) / (n2 - n1), 1e-9)
    a = max(t1 - b * n1, 0.0)
    return {"value": T / (a + b * T), "unit": "tokens/s", "cores": threads, "kind": "port",
            "per_token_s": b, "per_step_s": a,
            "sample": f"{n1} and {n2} tokens of the {cfg_name} layer fwd+bwd (EP=1, all {CONFIGS[cfg_name][2]} "
                      f"experts) through the C oracle (oracle/eplab_oracle.c, OpenMP): {t1:.2f} s and {t2:.2f} s "
                      f"-> t(n) = {a:.2f} s + {b * 1e3:.1f} ms * n, value = {T} / t({T})"}


def run_unfused(args):
    """Unfused NCCL all_to_all + cuBLAS grouped-GEMM baseline (tools/unfused_baseline.py)."""
    import torch
    rank, world, local = dist_info()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_19241_b200.model import sample_routing
    from tools import unfused_baseline as ub
    H, F, E, k, T = CONFIGS[args.config]
    epr = E // world
    sel, gw = sample_routing(E, k, T, world, 7)
    ids = torch.from_numpy(sel[rank].reshape(T, k).copy()).cuda().long()
    gws = torch.from_numpy(gw[rank].reshape(T, k).copy()).cuda()
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16().requires_grad_()
    dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
    w_up = ((torch.randn(epr, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()).requires_grad_()
    w_down = ((torch.randn(epr, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()).requires_grad_()
    gw_t = gws.requires_grad_()

    def step():
        y = ub.layer(x, ids, gw_t, w_up, w_down, E, world, rank)
        y.backward(dy)

    for _ in range(args.warmup):
        step()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    s0.record()
    for _ in range(args.steps):
        step()
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    if rank == 0:
        v = T * world / (ms / 1e3)
        print(json.dumps({"impl": "unfused", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                          "config": {"workload": CONFIG_DESC[args.config], "ep": world,
                                     "baseline": "NCCL all_to_all + per-expert cuBLAS GEMMs + torch SwiGLU, autograd bwd"}}),
              flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return
    cb = cpu_baseline(args.config, budget_s=max(3.0, 30.0 / max(1, args.steps + args.warmup)))
    extra = {}
    try:
        from oracle import pyoracle as po
        if po.has_reference():
            H, F, E, k, T = CONFIGS[args.config]
            tr, tm, ts = po.Reference().time_addressing(E, k, T, max(1, args.gpus), 7)
            extra = {"reference_addressing_s": {"sample_routing": tr, "build_global_token_map": tm,
                                                "build_send_schedule": ts,
                                                "note": "oracle/_ref (unmodified reference eplab), single thread"}}
    except Exception as e:  # reference build absent: the port alone is the arm
        extra = {"reference_addressing_s": f"unavailable: {e}"}
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": CONFIGS[args.config][4] * args.gpus / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic", "config": {"workload": CONFIG_DESC[args.config], "ep": args.gpus},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    line.update(extra)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import numpy as np
    import torch
    rank, world, local = dist_info()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    # EPLAB_BENCH_SHARE_DEVICE=1: every rank on cuda:0 with 148/N SMs (exercises the multi-rank
    # path on a single GPU; bootstrap over gloo since NCCL refuses two ranks on one device)
    share = os.environ.get("EPLAB_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_19241_b200 import moe as M
    from paper_2604_19241_b200.model import choose_config, sample_routing

    H, F, E, k, T = CONFIGS[args.config]
    epr = E // world
    sel, gw = sample_routing(E, k, T, world, 7)  # the reference's generator (library host code)
    ids = torch.from_numpy(sel[rank].reshape(T, k).copy()).cuda()
    gws = torch.from_numpy(gw[rank].reshape(T, k).copy()).cuda()
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
    w_up = (torch.randn(epr, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w_down = (torch.randn(epr, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    layer = M.EpMoE(H, F, E, k, T, rank=rank, world=world)
    if world > 1:
        layer.connect_distributed()
    n_sm = 148 // world if share else 148
    if share:
        layer.set_sm_budget(n_sm)
    cfg = choose_config(H, F, E, k, T, world, n_sm=n_sm)
    if args.tune:
        cfg = M.TuneConfig(*[int(v) for v in args.tune.split(",")])
    layer.set_tune_config(cfg)
    y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(w_up),
               dw_down=torch.empty_like(w_down), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.cuda.synchronize()
            torch.distributed.barrier()

    def step():
        layer.plan(ids, gws)
        layer.dispatch_group_gemm(x, w_up)
        layer.group_gemm_combine(w_down, y)
        layer.backward(dy, w_up, w_down, out=out)

    for _ in range(args.warmup):
        step()
    layer.check()
    # ---- per-kernel device times (events on the launching stream), separate pass
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        e = ev[i]
        e[0].record(st)
        layer.plan(ids, gws)
        layer.dispatch_group_gemm(x, w_up)
        e[1].record(st)
        layer.group_gemm_combine(w_down, y)
        e[2].record(st)
        layer._dispatch_bwd(dy, w_down, out)
        e[3].record(st)
        layer._combine_bwd(w_up, out)
        e[4].record(st)
    torch.cuda.synchronize()
    names = ["fwd_dispatch_gemm(+plan)", "fwd_gemm_combine", "bwd_dispatch_gemm", "bwd_gemm_combine"]
    kms = {n: sum(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(args.steps)) / args.steps
           for j, n in enumerate(names)}
    # ---- timed region: K whole steps
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    s0.record(st)
    for _ in range(args.steps):
        step()
    s1.record(st)
    torch.cuda.synchronize()
    clocks.mark_end()
    barrier()
    ms = s0.elapsed_time(s1) / args.steps
    clk = clocks.stop()
    layer.check()
    # ---- the same K steps replayed from one captured CUDA graph (plan + 4 MegaKernels + memsets):
    # the device-side epoch makes replays valid; reported next to the eager launches
    ms_graph = None
    try:
        graph = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        gs.wait_stream(st)
        with torch.cuda.stream(gs):
            step()
            with torch.cuda.graph(graph, stream=gs):
                step()
        torch.cuda.synchronize()
        graph.replay()
        barrier()
        torch.cuda.synchronize()
        s0.record(st)
        for _ in range(args.steps):
            graph.replay()
        s1.record(st)
        torch.cuda.synchronize()
        barrier()
        layer.check()
        ms_graph = s0.elapsed_time(s1) / args.steps
        del graph
    except Exception as e:  # report, keep the eager number
        print(f"# cuda graph capture failed: {e}", file=sys.stderr)
    # ---- overlap % from the device timeline (one extra, untimed step)
    layer.timeline_enable(1 << 20)
    overlap = {}
    layer.plan(ids, gws)
    layer.dispatch_group_gemm(x, w_up)
    overlap["fwd_dispatch_gemm"] = layer.timeline_export("")
    layer.group_gemm_combine(w_down, y)
    layer.timeline_export("")
    layer._dispatch_bwd(dy, w_down, out)
    overlap["bwd_dispatch_gemm"] = layer.timeline_export("")
    layer._combine_bwd(w_up, out)
    layer.timeline_export("")
    layer.timeline_enable(0)
    # ---- e2e through the C-ABI with host buffers (pinned), copies inside the timed region
    ids_h = ids.cpu().pin_memory()
    gw_h = gws.cpu().pin_memory()
    x_h = x.cpu().pin_memory()
    dy_h = dy.cpu().pin_memory()
    y_h = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    dx_h = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    dg_h = torch.empty(T, k, dtype=torch.float32).pin_memory()
    layer.step_host(ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dg_h, out["dw_up"], out["dw_down"])
    barrier()
    torch.cuda.synchronize()
    s0.record(st)
    for _ in range(args.steps):
        layer.step_host(ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dg_h, out["dw_up"], out["dw_down"])
    s1.record(st)
    torch.cuda.synchronize()
    barrier()
    ms_e2e_blocking = s0.elapsed_time(s1) / args.steps
    # pipelined: the same K steps through eplab_moe_step_host_async (step i+1's uploads run under
    # step i's MegaKernels); the timed region still holds every step's H2D and D2H copies
    for _ in range(2):
        layer.step_host_async(ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dg_h, out["dw_up"], out["dw_down"])
    layer.host_join(st)
    barrier()
    torch.cuda.synchronize()
    s0.record(st)
    for _ in range(args.steps):
        layer.step_host_async(ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dg_h, out["dw_up"], out["dw_down"])
    layer.host_join(st)
    s1.record(st)
    torch.cuda.synchronize()
    barrier()
    layer.check()
    ms_e2e = s0.elapsed_time(s1) / args.steps
    # max over ranks
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, ms_e2e, ms_e2e_blocking, ms_graph or 0.0] + [kms[n] for n in names], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e, ms_e2e_blocking = t[0].item(), t[1].item(), t[2].item()
        ms_graph = t[3].item() or None
        kms = {n: t[4 + j].item() for j, n in enumerate(names)}
    if rank == 0:
        peak_burst, peak_sust, hbm, peak_src = load_peaks()
        flops_tok, nvl_tok = algorithmic(args.config, world)
        tokens = T * world
        value = tokens / (ms / 1e3)
        # dominant kernel: bwd GroupGEMM+Combine (up dgrad 4kHF + up wgrad 4kHF per token)
        dom = "bwd_gemm_combine"
        dom_flops = 8.0 * k * H * F * T  # per launch, this rank's share (balanced routing)
        ach = dom_flops / (kms[dom] / 1e3) / 1e12
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(f"{args.config}:{dom}")
        except Exception:
            pass
        t_gemm = flops_tok * T / (peak_sust * 1e12)
        t_nvl = nvl_tok * T / (NVL_GBS * 1e9)
        roof_ms = max(t_gemm, t_nvl) * 1e3
        t_hbm = hbm_bytes_per_step(args.config, world) / (hbm * 1e9)
        cpu = cpu_baseline(args.config) if (world == 1 and not args.no_cpu_baseline) else None  # N=1 only
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (routing: reference sample_routing seed 7; random-init bf16 weights)",
            "config": {"workload": CONFIG_DESC[args.config], "ep": world, "tokens_per_gpu": T,
                       "tune_config": [cfg.n_disp, cfg.n_relay, cfg.n_comb, cfg.n_red, cfg.w],
                       "l2": "inputs larger than L2 (weights %.1f GB/GPU, activations > 1 GB per step)"
                             % (3 * epr * H * F * 2 / 1e9)},
            "e2e": {"value": tokens / (ms_e2e / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(T * k * 8 + 2 * T * H * 2),
                    "d2h_bytes_per_step": int(2 * T * H * 2 + T * k * 4),
                    "mode": "K steps back to back through eplab_moe_step_host_async (pinned host "
                            "buffers; step i+1's uploads overlap step i's MegaKernels), joined on the stream",
                    "blocking_value": tokens / (ms_e2e_blocking / 1e3),
                    "blocking_mode": "eplab_moe_step_host, host-synchronised every step"},
            "gpu_launches": 9 * args.steps,
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak_sust, "unit": "TFLOP/s",
                         "frac": ach / peak_sust, "traffic": traffic, "kernel": dom,
                         "peak_source": f"{peak_src} bf16 sustained (kernel timed inside the step)",
                         "frac_of_burst": ach / peak_burst},
            "roofline_step": {"roofline_ms": roof_ms, "frac": roof_ms / ms, "t_gemm_ms": t_gemm * 1e3,
                              "t_nvlink_ms": t_nvl * 1e3, "t_hbm_ms": t_hbm * 1e3,
                              "hbm_bytes": hbm_bytes_per_step(args.config, world),
                              "note": "roofline_ms = max(18kHF*T / sustained bf16 peak, NVLink bytes / 770 GB/s) "
                                      "(the north-star definition); t_hbm_ms = algorithmic HBM bytes of the step / "
                                      "measured HBM bandwidth, a second bound that the tensor and HBM traffic share"},
            "kernel_ms": kms,
            "graph": {"ms_per_step": ms_graph, "value": tokens / (ms_graph / 1e3) if ms_graph else None,
                      "note": "the same step replayed from one CUDA graph (launch gaps removed); "
                              "value/ms_per_step above are eager launches"},
            "overlap": {"fraction": overlap,
                        "definition": "time with >=1 comm/relay task AND >=1 GEMM tile active / time with "
                                      ">=1 comm/relay task active (device %globaltimer task log)"},
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "unfused"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tune", default="", help="override n_disp,n_relay,n_comb,n_red,w")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.impl == "unfused":
        run_unfused(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
