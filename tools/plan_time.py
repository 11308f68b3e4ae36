import os, sys, json, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2604_19241_b200 import moe as M
from paper_2604_19241_b200.model import choose_config
c = sys.argv[1] if len(sys.argv) > 1 else "qwen3"
H, F, E, k, T = bench.CONFIGS[c]
inp = bench.make_inputs(c, 1, 0)
L = M.EpMoE(H, F, E, k, T); L.set_tune_config(choose_config(H, F, E, k, T, 1))
st = torch.cuda.current_stream()
y = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(inp["w_up"]), dw_down=torch.empty_like(inp["w_down"]), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
def step():
    L.plan(inp["ids"], inp["gws"]); L.dispatch_group_gemm(inp["x"], inp["w_up"]); L.group_gemm_combine(inp["w_down"], y); L.backward(inp["dy"], inp["w_up"], inp["w_down"], out=out)
for _ in range(3): step()
res = {}
for name in ("plan", "mk0"):
    ts = []
    for _ in range(10):
        e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e0.record(st); L.plan(inp["ids"], inp["gws"]); e1.record(st); L.dispatch_group_gemm(inp["x"], inp["w_up"]); e2.record(st)
        L.group_gemm_combine(inp["w_down"], y); L.backward(inp["dy"], inp["w_up"], inp["w_down"], out=out)
        torch.cuda.synchronize(); ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    res = {"plan_ms": sorted(t[0] for t in ts)[5], "mk0_ms": sorted(t[1] for t in ts)[5]}
print(os.environ.get("EPLAB_LIB", "cur"), c, json.dumps(res))
