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
    return float(sum(hbm_bytes_per_kernel(cfg_name, world).values()))


def hbm_bytes_per_kernel(cfg_name, world):
    """hbm_bytes_per_step split over the four MegaKernels (the roofline object compares the dominant
    kernel's ncu DRAM traffic with its share)."""
    H, F, E, k, T = CONFIGS[cfg_name]
    R = T * k                      # rows received per GPU (balanced)
    El = E // world
    row = 2 * H
    w_up, w_down = El * 2 * F * H * 2, El * H * F * 2
    fwd_d = T * row + R * row + R * row + w_up + R * 2 * F * 2 + R * F * 2
    fwd_c = R * F * 2 + w_down + R * row + T * k * row + T * row
    bwd_d = T * row + R * row + R * row + w_down + R * 2 * F * 2 + R * 2 * F * 2 + R * F * 2 \
        + R * row + R * F * 2 + w_down
    bwd_c = R * 4 * F + w_up + R * row + R * 4 * F + R * row + w_up + T * k * row + T * row
    return {"fwd_dispatch_gemm": float(fwd_d), "fwd_gemm_combine": float(fwd_c), "bwd_dispatch_gemm": float(bwd_d),
            "bwd_gemm_combine": float(bwd_c)}


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
# Tokens of one CPU-arm step: a bounded sample of the workload's per-GPU batch (every expert's
# weights and weight gradients are still computed), sized for a few seconds per step on the host.
CPU_SAMPLE = {"mixtral": 4096, "qwen3": 8192, "dsv3": 2048, "small": 4096}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_threads():
    import torch
    n = os.cpu_count() or 1
    torch.set_num_threads(n)
    return torch.get_num_threads()


def cpu_sample_steps(cfg_name, n_tok, steps):
    """Wall seconds of `steps` fwd+bwd steps of n_tok tokens through oracle/cpu_port.py (the layer
    contract on CPU BLAS, EP=1: every expert on this host), one synthetic input set."""
    from oracle import cpu_port
    H, F, E, k, _ = CONFIGS[cfg_name]
    sel, gw, x, dy, w_up, w_down = cpu_port.synthetic(H, F, E, k, n_tok)
    out = []
    for _ in range(steps):
        t0 = time.perf_counter()
        cpu_port.moe_layer(sel, gw, x, w_up, w_down, dy, E, k, expand=False)
        out.append(time.perf_counter() - t0)
    return out


def cpu_extrapolation(cfg_name, n_small, t_small, n_big, t_big):
    """t(n) = a + b n from two measured sample sizes -> the full per-GPU batch (reported next to the
    measured value, never as it)."""
    T = CONFIGS[cfg_name][4]
    b = max((t_big - t_small) / max(n_big - n_small, 1), 1e-12)
    a = max(t_small - b * n_small, 0.0)
    return {"tokens_per_s": T / (a + b * T), "per_step_s": a, "per_token_s": b,
            "note": f"t(n) = a + b*n fitted to the {n_small}- and {n_big}-token samples, evaluated at the "
                    f"workload's {T} tokens (not run: ~{a + b * T:.0f} s per step)"}


def cpu_baseline(cfg_name, steps=3):
    """The reported CPU baseline of the N=1 line: `steps` timed steps of the bounded sample (~10-30 s
    of host work), plus a small sample for the full-batch extrapolation."""
    threads = cpu_threads()
    n = CPU_SAMPLE[cfg_name]
    ts = cpu_sample_steps(cfg_name, n, steps + 1)[1:]  # first step: warm-up (page faults, BLAS init)
    t_med = sorted(ts)[len(ts) // 2]
    n_small = max(16, n // 8)
    t_small = sorted(cpu_sample_steps(cfg_name, n_small, 2))[0]
    return {"value": n / t_med, "unit": "tokens/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "ms_per_step": t_med * 1e3,
            "sample": f"{n} of the workload's {CONFIGS[cfg_name][4]} tokens per step, fwd+bwd of the whole layer "
                      f"(all {CONFIGS[cfg_name][2]} experts, EP=1) through oracle/cpu_port.py (the layer contract "
                      f"on torch CPU BLAS, {threads} threads); median of {steps} steps",
            "extrapolated_full_batch": cpu_extrapolation(cfg_name, n_small, t_small, n, t_med)}


def run_reference(args):
    """The reference arm: the reference computes no layer numerics, so its CPU path
    for the workload is the port (oracle/cpu_port.py), timed on this host's cores with every thread,
    K steps after W warm-ups, each step the bounded sample of CPU_SAMPLE tokens; plus the reference's
    own compiled addressing functions (oracle/_ref) on the workload's routing."""
    rank, world, _ = dist_info()
    if rank != 0:
        return
    threads = cpu_threads()
    n = CPU_SAMPLE[args.config]
    ts = cpu_sample_steps(args.config, n, args.warmup + args.steps)[args.warmup:]
    ms = sum(ts) / len(ts) * 1e3
    ms_med = sorted(ts)[len(ts) // 2] * 1e3
    v = n / (ms / 1e3)
    n_small = max(16, n // 8)
    t_small = sorted(cpu_sample_steps(args.config, n_small, 2))[0]
    extra = {}
    try:
        from oracle import pyoracle as po
        if po.has_reference():
            H, F, E, k, T = CONFIGS[args.config]
            tr, tm, tsch = po.Reference().time_addressing(E, k, T, max(1, args.gpus), 7)
            extra = {"reference_addressing_s": {"sample_routing": tr, "build_global_token_map": tm,
                                                "build_send_schedule": tsch,
                                                "note": "oracle/_ref (unmodified reference eplab), single thread"}}
    except Exception as e:  # reference build absent: the port alone is the arm
        extra = {"reference_addressing_s": f"unavailable: {e}"}
    cb = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
          "sample": f"{n} of the workload's {CONFIGS[args.config][4]} tokens per step, fwd+bwd of the whole layer "
                    f"(all {CONFIGS[args.config][2]} experts on this host) through oracle/cpu_port.py on torch CPU "
                    f"BLAS, {threads} threads",
          "extrapolated_full_batch": cpu_extrapolation(args.config, n_small, t_small, n, ms_med / 1e3)}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": ms_med,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": DATA, "config": bench_config(args.config, args.gpus), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    line.update(extra)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
DATA = "synthetic (routing: reference sample_routing seed 7; random-init bf16 weights)"


def bench_config(cfg_name, world):
    """The config dict of every arm (identical for ours, unfused and reference)."""
    H, F, E, k, T = CONFIGS[cfg_name]
    touched = hbm_bytes_per_step(cfg_name, world)
    return {"workload": CONFIG_DESC[cfg_name], "ep": world, "tokens_per_gpu": T,
            "l2": ("inputs larger than L2: %.1f GB of algorithmic HBM traffic per step (weights %.2f GB/GPU) vs "
                   "126 MB of L2" % (touched / 1e9, 3 * (E // world) * H * F * 2 / 1e9))}


def make_inputs(cfg_name, world, rank):
    import torch
    from paper_2604_19241_b200.model import sample_routing
    H, F, E, k, T = CONFIGS[cfg_name]
    epr = E // world
    sel, gw = sample_routing(E, k, T, world, 7)  # the reference's generator (library host code)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    return dict(ids=torch.from_numpy(sel[rank].reshape(T, k).copy()).cuda(),
                gws=torch.from_numpy(gw[rank].reshape(T, k).copy()).cuda(),
                x=torch.randn(T, H, device="cuda", generator=g, dtype=torch.bfloat16),
                dy=(torch.randn(T, H, device="cuda", generator=g, dtype=torch.bfloat16) * 0.1),
                w_up=torch.randn(epr, 2 * F, H, device="cuda", generator=g, dtype=torch.bfloat16) * H ** -0.5,
                w_down=torch.randn(epr, H, F, device="cuda", generator=g, dtype=torch.bfloat16) * F ** -0.5)


def nvlink_kib(index):
    """(tx, rx) KiB summed over this GPU's NVLinks from the driver's link data-payload counters
    (`nvidia-smi nvlink -gt d`), or None where the links report nothing (a single-GPU box)."""
    import re
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True,
                             text=True, timeout=30).stdout
    except Exception:
        return None
    tot = {"Tx": 0, "Rx": 0}
    seen = False
    for m in re.finditer(r"Data (Tx|Rx):\s*(\d+)", out):
        tot[m.group(1)] += int(m.group(2))
        seen = True
    return (tot["Tx"], tot["Rx"]) if seen else None


def timed_steps(step, K, st, barrier):
    """K steps bracketed by barrier + synchronize, one event per step boundary on the launching
    stream: (mean ms over the bracket, median ms of the per-step intervals)."""
    import torch
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    barrier()
    torch.cuda.synchronize()
    ev[0].record(st)
    for i in range(K):
        step()
        ev[i + 1].record(st)
    torch.cuda.synchronize()
    barrier()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
    return ev[0].elapsed_time(ev[K]) / K, sorted(per)[K // 2]


def roofline_terms(cfg_name, world, ms):
    """The north-star roofline of one step: max(GEMM FLOPs at peak, NVLink bytes at
    770 / 900 GB/s), plus the HBM term."""
    peak_burst, peak_sust, hbm, _ = load_peaks()
    H, F, E, k, T = CONFIGS[cfg_name]
    flops_tok, nvl_tok = algorithmic(cfg_name, world)
    t_gemm_s = flops_tok * T / (peak_sust * 1e12)
    t_gemm_b = flops_tok * T / (peak_burst * 1e12)
    t_nvl = {bw: nvl_tok * T / (bw * 1e9) for bw in (770.0, 900.0)}
    roof_s = max(t_gemm_s, t_nvl[770.0]) * 1e3
    roof_b = max(t_gemm_b, t_nvl[900.0]) * 1e3
    return {"roofline_ms": roof_s, "frac": roof_s / ms, "roofline_ms_burst": roof_b, "frac_of_burst": roof_b / ms,
            "t_gemm_ms": t_gemm_s * 1e3, "t_gemm_ms_burst": t_gemm_b * 1e3,
            "t_nvlink_ms": {"770GBps": t_nvl[770.0] * 1e3, "900GBps": t_nvl[900.0] * 1e3},
            "t_hbm_ms": hbm_bytes_per_step(cfg_name, world) / (hbm * 1e9) * 1e3,
            "hbm_bytes": hbm_bytes_per_step(cfg_name, world),
            "note": "roofline_ms = max(18kHF*T / sustained bf16 peak, NVLink bytes / 770 GB/s measured); "
                    "_burst: burst peak and 900 GB/s nominal NVLink; t_hbm_ms = algorithmic HBM bytes / measured "
                    "HBM bandwidth, a second bound the tensor and HBM traffic share"}


def measure_config(M, cfg_name, world, rank, n_sm, share, steps, warmup, barrier, per_kernel=True):
    """Build one layer shape, warm up, time `steps` whole steps. Returns (layer, tensors, dict)."""
    import torch
    from paper_2604_19241_b200.model import choose_config
    H, F, E, k, T = CONFIGS[cfg_name]
    inp = make_inputs(cfg_name, world, rank)
    layer = M.EpMoE(H, F, E, k, T, rank=rank, world=world)
    if world > 1:
        layer.connect_distributed()
    if share:
        layer.set_sm_budget(n_sm)
    cfg = choose_config(H, F, E, k, T, world, n_sm=n_sm)
    layer.set_tune_config(cfg)
    y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(inp["w_up"]),
               dw_down=torch.empty_like(inp["w_down"]), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
    st = torch.cuda.current_stream()

    def step():
        layer.plan(inp["ids"], inp["gws"])
        layer.dispatch_group_gemm(inp["x"], inp["w_up"])
        layer.group_gemm_combine(inp["w_down"], y)
        layer.backward(inp["dy"], inp["w_up"], inp["w_down"], out=out)

    for _ in range(warmup):
        step()
    layer.check()
    res = {"cfg": cfg}
    if per_kernel:  # per-kernel device times (events on the launching stream), separate pass
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        for i in range(steps):
            e = ev[i]
            e[0].record(st)
            layer.plan(inp["ids"], inp["gws"])
            layer.dispatch_group_gemm(inp["x"], inp["w_up"])
            e[1].record(st)
            layer.group_gemm_combine(inp["w_down"], y)
            e[2].record(st)
            layer._dispatch_bwd(inp["dy"], inp["w_down"], out)
            e[3].record(st)
            layer._combine_bwd(inp["w_up"], out)
            e[4].record(st)
        torch.cuda.synchronize()
        names = ["fwd_dispatch_gemm(+plan)", "fwd_gemm_combine", "bwd_dispatch_gemm", "bwd_gemm_combine"]
        res["kernel_ms"] = {n: sorted(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(steps))[steps // 2]
                            for j, n in enumerate(names)}
    res["step"], res["inp"], res["y"], res["out"], res["layer"] = step, inp, y, out, layer
    return res


def measure_unfused(cfg_name, world, rank, steps, warmup, barrier):
    """The unfused NCCL baseline (paper_2604_19241_b200/unfused.py) on the same workload: (mean ms,
    median ms), max over ranks by the caller."""
    import torch
    from paper_2604_19241_b200.unfused import LocalComm, NcclComm, UnfusedEpMoE, unfused_step
    H, F, E, k, T = CONFIGS[cfg_name]
    inp = make_inputs(cfg_name, world, rank)
    L = UnfusedEpMoE(H, F, E, k, T, rank=rank, world=world)
    comm = NcclComm() if world > 1 else LocalComm()

    def step():
        unfused_step([L], comm, [inp["x"]], [inp["ids"]], [inp["gws"]], [inp["dy"]], [inp["w_up"]], [inp["w_down"]])

    for _ in range(warmup):
        step()
    L.check()
    ms, med = timed_steps(step, steps, torch.cuda.current_stream(), barrier)
    L.check()
    L.close()
    return ms, med


def run_ours(args):
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

    H, F, E, k, T = CONFIGS[args.config]
    n_sm = 148 // world if share else 148
    st = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.cuda.synchronize()
            torch.distributed.barrier()

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return t.tolist()

    res = measure_config(M, args.config, world, rank, n_sm, share, args.steps, args.warmup, barrier)
    layer, step, inp, y, out, cfg = res["layer"], res["step"], res["inp"], res["y"], res["out"], res["cfg"]
    kms = res["kernel_ms"]
    # ---- timed region: K whole steps, clocks sampled during it
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)
    clocks.mark_start()
    nvl0 = nvlink_kib(local) if world > 1 else None
    ms, ms_med = timed_steps(step, args.steps, st, barrier)
    nvl1 = nvlink_kib(local) if world > 1 else None
    clocks.mark_end()
    # NVLink payload bytes this GPU sent / received per step during the timed steps (link counters; the
    # barriers around the region add a few KiB)
    nvl = [(nvl1[0] - nvl0[0]) * 1024.0 / args.steps, (nvl1[1] - nvl0[1]) * 1024.0 / args.steps] \
        if nvl0 and nvl1 else [-1.0, -1.0]
    clk = clocks.stop()
    layer.check()
    # ---- the same steps replayed from one captured CUDA graph (plan + 4 MegaKernels + memsets):
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
        ms_graph, _ = timed_steps(graph.replay, args.steps, st, barrier)
        layer.check()
        del graph
    except Exception as e:  # report, keep the eager number
        print(f"# cuda graph capture failed: {e}", file=sys.stderr)
    # ---- overlap % from the device timeline (one extra, untimed step)
    layer.timeline_enable(1 << 20)
    overlap = {}
    layer.plan(inp["ids"], inp["gws"])
    layer.dispatch_group_gemm(inp["x"], inp["w_up"])
    overlap["fwd_dispatch_gemm"] = layer.timeline_export("")
    layer.group_gemm_combine(inp["w_down"], y)
    layer.timeline_export("")
    layer._dispatch_bwd(inp["dy"], inp["w_down"], out)
    overlap["bwd_dispatch_gemm"] = layer.timeline_export("")
    layer._combine_bwd(inp["w_up"], out)
    layer.timeline_export("")
    layer.timeline_enable(0)
    # ---- e2e through the C-ABI with host buffers (pinned), copies inside the timed region
    ids_h, gw_h = inp["ids"].cpu().pin_memory(), inp["gws"].cpu().pin_memory()
    x_h, dy_h = inp["x"].cpu().pin_memory(), inp["dy"].cpu().pin_memory()
    y_h = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    dx_h = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
    dg_h = torch.empty(T, k, dtype=torch.float32).pin_memory()
    host_args = (ids_h, gw_h, x_h, dy_h, inp["w_up"], inp["w_down"], y_h, dx_h, dg_h, out["dw_up"], out["dw_down"])
    layer.step_host(*host_args)
    ms_e2e_blocking, _ = timed_steps(lambda: layer.step_host(*host_args), args.steps, st, barrier)
    # pipelined: the same K steps through eplab_moe_step_host_async (step i+1's uploads run under
    # step i's MegaKernels); the timed region still holds every step's H2D and D2H copies
    for _ in range(2):
        layer.step_host_async(*host_args)
    layer.host_join(st)
    barrier()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(st)
    for _ in range(args.steps):
        layer.step_host_async(*host_args)
    layer.host_join(st)
    s1.record(st)
    torch.cuda.synchronize()
    barrier()
    layer.check()
    ms_e2e = s0.elapsed_time(s1) / args.steps
    layer.close()
    del res, layer, step, inp, y, out
    torch.cuda.empty_cache()
    # ---- the unfused NCCL baseline on the same box and workload
    unf_ms = unf_med = None
    if not args.no_unfused:
        try:
            unf_ms, unf_med = measure_unfused(args.config, world, rank, args.steps, args.warmup, barrier)
        except Exception as e:
            print(f"# unfused baseline failed: {e}", file=sys.stderr)
        torch.cuda.empty_cache()
    # ---- the other BASELINE shapes at this N (N=1 line: the paper's published shapes driver-timed)
    per_config = {}
    if world == 1 and not args.no_per_config:
        for name in [c for c in ("qwen3", "dsv3") if c != args.config]:
            r2 = measure_config(M, name, world, rank, n_sm, share, args.steps, args.warmup, barrier)
            c_ms, c_med = timed_steps(r2["step"], args.steps, st, barrier)
            r2["layer"].check()
            rt = roofline_terms(name, world, c_ms)
            per_config[name] = {"workload": CONFIG_DESC[name], "ms_per_step": c_ms, "ms_per_step_median": c_med,
                                "value": CONFIGS[name][4] * world / (c_ms / 1e3), "unit": "tokens/s",
                                "frac_of_sustained": rt["frac"], "frac_of_burst": rt["frac_of_burst"],
                                "roofline_ms": rt["roofline_ms"], "roofline_ms_burst": rt["roofline_ms_burst"],
                                "t_hbm_ms": rt["t_hbm_ms"], "kernel_ms": r2["kernel_ms"],
                                "tune_config": [r2["cfg"].n_disp, r2["cfg"].n_relay, r2["cfg"].n_comb,
                                                r2["cfg"].n_red, r2["cfg"].w]}
            r2["layer"].close()
            del r2
            torch.cuda.empty_cache()
    # ---- max over ranks
    names = list(kms)
    v = max_over_ranks([ms, ms_med, ms_e2e, ms_e2e_blocking, ms_graph or 0.0, unf_ms or 0.0, unf_med or 0.0]
                       + [kms[n] for n in names] + nvl)
    nvl = v[7 + len(names):]
    ms, ms_med, ms_e2e, ms_e2e_blocking = v[0], v[1], v[2], v[3]
    ms_graph, unf_ms, unf_med = v[4] or None, v[5] or None, v[6] or None
    kms = {n: v[7 + j] for j, n in enumerate(names)}
    if rank == 0:
        peak_burst, peak_sust, hbm, peak_src = load_peaks()
        tokens = T * world
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
        cpu = cpu_baseline(args.config) if (world == 1 and not args.no_cpu_baseline) else None  # N=1 only
        line = {
            "metric": METRIC, "value": tokens / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": ms_med,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": DATA,
            "config": bench_config(args.config, world),
            "tune_config": [cfg.n_disp, cfg.n_relay, cfg.n_comb, cfg.n_red, cfg.w],
            "e2e": {"value": tokens / (ms_e2e / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(T * k * 8 + 2 * T * H * 2),
                    "d2h_bytes_per_step": int(2 * T * H * 2 + T * k * 4),
                    "mode": "K steps back to back through eplab_moe_step_host_async (pinned host "
                            "buffers; step i+1's uploads overlap step i's MegaKernels), joined on the stream",
                    "blocking_value": tokens / (ms_e2e_blocking / 1e3),
                    "blocking_mode": "eplab_moe_step_host, host-synchronised every step"},
            "gpu_launches": 7 * args.steps,  # per step: 3 planning kernels + the 4 MegaKernels
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak_sust, "unit": "TFLOP/s",
                         "frac": ach / peak_sust, "traffic": traffic, "kernel": dom,
                         "algorithmic_bytes": hbm_bytes_per_kernel(args.config, world)[dom],
                         "peak_source": f"{peak_src} bf16 sustained (kernel timed inside the step)",
                         "frac_of_burst": ach / peak_burst},
            "roofline_step": roofline_terms(args.config, world, ms),
            "kernel_ms": kms,
            "unfused": {"ms_per_step": unf_ms, "ms_per_step_median": unf_med,
                        "value": tokens / (unf_ms / 1e3) if unf_ms else None,
                        "speedup_of_fused": unf_ms / ms if unf_ms else None,
                        "baseline": "paper_2604_19241_b200/unfused.py: NCCL all_to_all (host-synchronised splits) -> "
                                    "the same tcgen05 GroupGEMM tiles without collectives -> NCCL all_to_all back -> "
                                    "k-order reduce kernel; bitwise equal to the fused step (tests/test_unfused_gpu.py)"},
            "per_config": per_config or None,
            "graph": {"ms_per_step": ms_graph, "value": tokens / (ms_graph / 1e3) if ms_graph else None,
                      "note": "the same step replayed from one CUDA graph (launch gaps removed); "
                              "value/ms_per_step above are eager launches"},
            "overlap": {"fraction": overlap,
                        "definition": "time with >=1 comm/relay task AND >=1 GEMM tile active / time with "
                                      ">=1 comm/relay task active (device %globaltimer task log)"},
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        if world > 1:
            nvl_alg = algorithmic(args.config, world)[1] * T  # per GPU per direction per step
            line["nvlink"] = (
                {"tx_bytes_per_step_max": nvl[0], "rx_bytes_per_step_max": nvl[1],
                 "tx_GBps_max": nvl[0] / (ms / 1e3) / 1e9, "rx_GBps_max": nvl[1] / (ms / 1e3) / 1e9,
                 "algorithmic_bytes_per_step": nvl_alg,
                 "frac_of_900GBps_over_step": max(nvl) / (ms / 1e3) / 900e9,
                 "source": "nvidia-smi nvlink -gt d (link data payload) before/after the timed steps, max over ranks; "
                           "GB/s averaged over the whole step (the comm roles run inside the MegaKernels)"}
                if min(nvl) >= 0 else {"unavailable": "the NVLink counters report no data on this box"})
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unfused", action="store_true", help="skip the unfused NCCL baseline leg")
    ap.add_argument("--no-per-config", action="store_true", help="N=1: skip the qwen3/dsv3 legs")
    ap.add_argument("--tune", default="", help="override n_disp,n_relay,n_comb,n_red,w")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
