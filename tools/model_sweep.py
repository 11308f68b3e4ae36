"""Measures per-MegaKernel times over the unified-primitive sweep (BASELINE.json configs[4]:
top-k 1->16, tokens 2K->64K; Qwen3-like dims H=2048, F=768, 128 experts) plus the three
BASELINE shapes, at EP=1 (and EP=2 on virtual ranks when --ep2), and writes JSON lines that
tools/fit_model.py turns into the calibration + predicted-vs-measured table."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2604_19241_b200 import moe as M  # noqa: E402


def measure(H, F, E, k, T, cfg, steps=3, spare=1):
    sel, gw = po.Oracle().sample_routing(E, k, T, 1, 7)
    ids = torch.from_numpy(sel[0].reshape(T, k).copy()).cuda()
    gws = torch.from_numpy(gw[0].reshape(T, k).copy()).cuda()
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
    w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
    L = M.EpMoE(H, F, E, k, T)
    L.set_tune_config(cfg)
    L.set_comm_options(spare_warps=3 if spare else 0)
    y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(w_up),
               dw_down=torch.empty_like(w_down), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
    st = torch.cuda.current_stream()
    for _ in range(2):
        L.plan(ids, gws)
        L.dispatch_group_gemm(x, w_up)
        L.group_gemm_combine(w_down, y)
        L.backward(dy, w_up, w_down, out=out)
    L.check()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        e = ev[i]
        e[0].record(st)
        L.plan(ids, gws)
        L.dispatch_group_gemm(x, w_up)
        e[1].record(st)
        L.group_gemm_combine(w_down, y)
        e[2].record(st)
        L._dispatch_bwd(dy, w_down, out)
        e[3].record(st)
        L._combine_bwd(w_up, out)
        e[4].record(st)
    torch.cuda.synchronize()
    ms = [sum(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(steps)) / steps for j in range(4)]
    L.check()
    L.close()
    del x, dy, w_up, w_down, out, y
    torch.cuda.empty_cache()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/model_sweep.jsonl")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    cases = []
    for k in (1, 2, 4, 8, 16):
        for T in (2048, 8192, 32768):
            cases.append(("sweep", 2048, 768, 128, k, T))
    cases += [("mixtral", 4096, 14336, 8, 2, 16384), ("qwen3", 2048, 768, 128, 8, 16384),
              ("dsv3", 7168, 2048, 256, 8, 16384), ("sweep64k", 2048, 768, 128, 8, 65536)]
    with open(args.out, "w") as f:
        for name, H, F, E, k, T in cases:
            for nd, spare in ((0, 1), (16, 1), (64, 1), (64, 0)):
                ms = measure(H, F, E, k, T, M.TuneConfig(nd, 0, 1, 148, 8), spare=spare)
                rec = dict(name=name, H=H, F=F, E=E, k=k, T=T, world=1, n_disp=nd, n_relay=0, spare=spare, ms=ms)
                f.write(json.dumps(rec) + "\n")
                f.flush()
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
