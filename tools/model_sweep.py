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


def measure_virtual(H, F, E, k, T, W, relay, steps=3):
    """W virtual ranks on this GPU (148 // W SMs each, peers in local HBM): per-MegaKernel times,
    max over ranks (the EP > 1 protocol with the NVLink hop replaced by local memory)."""
    sel, gw = po.Oracle().sample_routing(E, k, T, W, 7)
    epr = E // W
    g = torch.Generator(device="cuda").manual_seed(1)
    ranks = [M.EpMoE(H, F, E, k, T, rank=r, world=W, timeout_s=60.0) for r in range(W)]
    M.EpMoE.connect_local(ranks)
    n_sm = 148 // W
    nd = max(2, 16 // W)
    for rk in ranks:
        rk.set_sm_budget(n_sm)
        rk.set_tune_config(M.TuneConfig(nd, relay, 1, n_sm, 8))
    ins = []
    for r in range(W):
        ins.append(dict(ids=torch.from_numpy(sel[r].reshape(T, k).copy()).cuda(),
                        gw=torch.from_numpy(gw[r].reshape(T, k).copy()).cuda(),
                        x=torch.randn(T, H, device="cuda", generator=g).bfloat16(),
                        dy=(torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16(),
                        w_up=(torch.randn(epr, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16(),
                        w_down=(torch.randn(epr, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16(),
                        y=torch.empty(T, H, device="cuda", dtype=torch.bfloat16)))
        ins[r]["out"] = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"),
                             dw_up=torch.empty_like(ins[r]["w_up"]), dw_down=torch.empty_like(ins[r]["w_down"]),
                             dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
    streams = [torch.cuda.Stream() for _ in range(W)]

    def step(evs=None):
        for r in range(W):
            with torch.cuda.stream(streams[r]):
                if evs:
                    evs[r][0].record(streams[r])
                ranks[r].plan(ins[r]["ids"], ins[r]["gw"], streams[r])
        torch.cuda.synchronize()
        for ph, fn in enumerate([lambda L, a, s: L.dispatch_group_gemm(a["x"], a["w_up"], s),
                                 lambda L, a, s: L.group_gemm_combine(a["w_down"], a["y"], s),
                                 lambda L, a, s: L._dispatch_bwd(a["dy"], a["w_down"], a["out"], s),
                                 lambda L, a, s: L._combine_bwd(a["w_up"], a["out"], s)]):
            for r in range(W):
                with torch.cuda.stream(streams[r]):
                    if evs and ph == 0:
                        evs[r][1].record(streams[r])  # after the plan (synchronised between ranks)
                    fn(ranks[r], ins[r], streams[r])
                    if evs:
                        evs[r][ph + 2].record(streams[r])

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    per = []
    for _ in range(steps):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(W)]
        step(evs)
        torch.cuda.synchronize()
        per.append([max(evs[r][j + 1].elapsed_time(evs[r][j + 2]) for r in range(W)) for j in range(4)])
    for rk in ranks:
        rk.check()
        rk.close()
    torch.cuda.empty_cache()
    return [sum(p[j] for p in per) / steps for j in range(4)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/model_sweep.jsonl")
    ap.add_argument("--ep", action="store_true", help="also the virtual-rank EP=2/4/8 cases")
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
            for nd, spare in ((0, 1), (16, 1), (48, 1), (48, 0)):
                ms = measure(H, F, E, k, T, M.TuneConfig(nd, 0, 1, 148, 8), spare=spare)
                rec = dict(name=name, H=H, F=F, E=E, k=k, T=T, world=1, n_disp=nd, n_relay=0, spare=spare, ms=ms)
                f.write(json.dumps(rec) + "\n")
                f.flush()
                print(json.dumps(rec), flush=True)
        if args.ep:
            for name, H, F, E, k, T in (("vep_qwen3", 2048, 768, 128, 8, 8192), ("vep_k2", 2048, 768, 128, 2, 8192),
                                        ("vep_mixtral", 4096, 14336, 8, 2, 4096)):
                for W in (2, 4, 8):
                    for relay in (0, 1):
                        ms = measure_virtual(H, F, E, k, T, W, relay)
                        rec = dict(name=name, H=H, F=F, E=E, k=k, T=T, world=W, virtual=1, n_sm=148 // W,
                                   n_disp=max(2, 16 // W), n_relay=relay, spare=1, ms=ms)
                        f.write(json.dumps(rec) + "\n")
                        f.flush()
                        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
