"""Host<->device copy bandwidth alone, concurrent H2D+D2H, and a Mixtral step with / without
copies running underneath (pipelined e2e diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from oracle import pyoracle as po
from paper_2604_19241_b200 import moe as M
from paper_2604_19241_b200.model import choose_config

n = 134 * 1024 * 1024
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / reps * 1e3
print("H2D %.2f ms" % t(lambda: d1.copy_(h1, non_blocking=True)))
print("D2H %.2f ms" % t(lambda: h2.copy_(d2, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("H2D||D2H %.2f ms" % t(both))
H, F, E, k, T = bench.CONFIGS["mixtral"]
sel, gw = po.Oracle().sample_routing(E, k, T, 1, 7)
ids = torch.from_numpy(sel[0].reshape(T, k).copy()).cuda(); gws = torch.from_numpy(gw[0].reshape(T, k).copy()).cuda()
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(T, H, device="cuda", generator=g).bfloat16(); dy = (torch.randn(T, H, device="cuda", generator=g) * 0.1).bfloat16()
w_up = (torch.randn(E, 2 * F, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
w_down = (torch.randn(E, H, F, device="cuda", generator=g) * F ** -0.5).bfloat16()
L = M.EpMoE(H, F, E, k, T); L.set_tune_config(choose_config(H, F, E, k, T, 1))
out = dict(dx=torch.empty(T, H, dtype=torch.bfloat16, device="cuda"), dw_up=torch.empty_like(w_up),
           dw_down=torch.empty_like(w_down), dgate=torch.empty(T, k, dtype=torch.float32, device="cuda"))
def step():
    L.forward(x, ids, gws, w_up, w_down); L.backward(dy, w_up, w_down, out=out)
step()
print("step alone %.2f ms" % t(step))
def step_copies():
    both(); both(); step()
print("step + 2x(H2D||D2H) underneath %.2f ms" % t(step_copies))
ids_h = ids.cpu().pin_memory(); gw_h = gws.cpu().pin_memory(); x_h = x.cpu().pin_memory(); dy_h = dy.cpu().pin_memory()
y_h = torch.empty(T, H, dtype=torch.bfloat16).pin_memory(); dx_h = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
dg_h = torch.empty(T, k, dtype=torch.float32).pin_memory()
st = torch.cuda.current_stream()
def host_async():
    L.step_host_async(ids_h, gw_h, x_h, dy_h, w_up, w_down, y_h, dx_h, dg_h, out["dw_up"], out["dw_down"])
for reps in (1, 5, 10):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): host_async()
    enq = (time.perf_counter() - a) * 1e3
    L.host_join(st); torch.cuda.synchronize()
    print("async x%d: %.2f ms/step (host enqueue %.2f ms total)" % (reps, (time.perf_counter() - a) * 1e3 / reps, enq))
L.check(); L.close()
