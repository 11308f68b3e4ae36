"""EP=1/2/4/8 on ONE B200 with virtual ranks (one process, W contexts, 148/W SMs each, peer rows
through the same symmetric buffers the NVLink path uses): the EP>1 machinery -- count exchange,
remote rows, relay, replica pushes to the source, top-k barrier -- at fixed total work (16K
tokens split over the ranks). Same total FLOPs at every W: time(W)/time(1) is the overhead of
the EP>1 code paths on one device (NVLink itself is not exercised: peers are local memory).
  python tools/virtual_ep.py --config qwen3 [--relay 4]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2604_19241_b200 import moe as M
from paper_2604_19241_b200.model import sample_routing

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3")
ap.add_argument("--relay", type=int, default=0)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--trace", type=int, default=0, help="EP size whose rank-0 fwd dispatch is traced")
args = ap.parse_args()
H, F, E, k, T_all = bench.CONFIGS[args.config]
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randn(T_all, H, device="cuda", generator=g).bfloat16()
dy = (torch.randn(T_all, H, device="cuda", generator=g) * 0.5).bfloat16()
w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
for W in (1, 2, 4, 8):
    if E % W:
        continue
    T, epr = T_all // W, E // W
    sel, gw = sample_routing(E, k, T, W, 7)
    ids = torch.from_numpy(sel.reshape(W * T, k).copy()).cuda()
    gws = torch.from_numpy(gw.reshape(W * T, k).copy()).cuda()
    ranks = [M.EpMoE(H, F, E, k, T, rank=r, world=W, max_recv_rows=T * k * 3 // 2 if W > 1 else 0, timeout_s=60.0)
             for r in range(W)]
    if W > 1:
        M.EpMoE.connect_local(ranks)
    n_sm = 148 // W
    for r in ranks:
        if W > 1:
            r.set_sm_budget(n_sm)
        r.set_tune_config((max(2, 16 // W), args.relay if W > 1 else 0, 1, n_sm, 8))
    streams = [torch.cuda.Stream() for _ in range(W)]
    outs = [dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"),
                 dw_up=torch.empty(epr, 2 * F, H, dtype=torch.bfloat16, device="cuda"),
                 dw_down=torch.empty(epr, H, F, dtype=torch.bfloat16, device="cuda"),
                 dgate=torch.empty(T, k, dtype=torch.float32, device="cuda")) for _ in range(W)]
    ys = [torch.empty(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(W)]

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(W)]

    def step(rec=False):
        for ph in range(4):
            for r in range(W):
                if rec:
                    evs[r][ph].record(streams[r])
                sl = slice(r * T, (r + 1) * T)
                with torch.cuda.stream(streams[r]):
                    if ph == 0:
                        ranks[r].plan(ids[sl], gws[sl], streams[r])
                    elif ph == 1:
                        ranks[r].dispatch_group_gemm(x[sl], w_up[r * epr:(r + 1) * epr], streams[r])
                    elif ph == 2:
                        ranks[r].group_gemm_combine(w_down[r * epr:(r + 1) * epr], ys[r], stream=streams[r])
                    else:
                        ranks[r].backward(dy[sl], w_up[r * epr:(r + 1) * epr], w_down[r * epr:(r + 1) * epr],
                                          stream=streams[r], out=outs[r])
        if rec:
            for r in range(W):
                evs[r][4].record(streams[r])

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_stream(main)
    for _ in range(args.steps):
        step()
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    for r in range(W):
        ranks[r].check(streams[r])
    if args.trace == W:
        ranks[0].timeline_enable(1 << 20)
        for ph in range(2):
            for r in range(W):
                sl = slice(r * T, (r + 1) * T)
                with torch.cuda.stream(streams[r]):
                    if ph == 0:
                        ranks[r].plan(ids[sl], gws[sl], streams[r])
                    else:
                        ranks[r].dispatch_group_gemm(x[sl], w_up[r * epr:(r + 1) * epr], streams[r])
        torch.cuda.synchronize()
        os.makedirs("gpurun_out", exist_ok=True)
        ranks[0].timeline_export(f"gpurun_out/vep_trace_{args.config}_ep{W}_relay{args.relay}.json")
        ranks[0].timeline_enable(0)
    ms = e0.elapsed_time(e1) / args.steps
    step(rec=True)
    torch.cuda.synchronize()
    per_rank = [[round(evs[r][j].elapsed_time(evs[r][j + 1]), 3) for j in range(4)] for r in range(W)]
    print(json.dumps({"config": args.config, "ep": W, "relay": args.relay if W > 1 else 0, "tokens_total": T_all,
                      "sm_per_rank": n_sm, "ms_per_step": round(ms, 3), "tokens_per_s": round(T_all / ms * 1e3),
                      "rank_phase_ms(plan,fwd_dispatch+fwd_combine,bwd)": per_rank[:2] + per_rank[-1:]}),
          flush=True)
    for r in ranks:
        r.close()
    torch.cuda.empty_cache()
