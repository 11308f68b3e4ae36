"""Staged GPU debug of the EP-MoE path: plan -> fwd dispatch -> fwd combine -> bwd, checking the
device error word after each stage."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import pyoracle as po
from paper_2604_19241_b200 import moe as m
from tests.test_moe_gpu import Problem, from_u16, to_u16

E, k, H, F, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
prob = Problem(1, E, k, H, F, T)
orc = po.Oracle()
L = m.EpMoE(H, F, E, k, T, timeout_s=3.0)
ids = torch.from_numpy(prob.sel.reshape(T, k).copy()).cuda()
gw = torch.from_numpy(prob.gw.reshape(T, k).copy()).cuda()
x = from_u16(prob.x[0]); dy = from_u16(prob.dy[0])
wu = from_u16(prob.w_up); wd = from_u16(prob.w_down)
def stage(name, fn):
    try:
        r = fn(); L.check(); print("OK  ", name, flush=True); return r
    except Exception as e:
        print("FAIL", name, e, flush=True); return None
stage("plan", lambda: L.plan(ids, gw))
tr, le, off, rt, sb = L.export_token_map()
otr, ole, ooff, ort, osb = orc.token_map(prob.sel, E, k)
print("token map equal:", (tr == otr[0]).all(), (le == ole[0]).all(), (off == ooff[0]).all(), (rt == ort).all(), (sb == osb).all())
sba, rows = L.export_layout(); print("layout", sba[:8], rows[:8])
print("sb dev", sb[:8], "orc", osb[:8])
bad = np.nonzero(off != ooff[0])[0]
print("n bad offsets", len(bad), "first", bad[:10], "dev", off[bad[:10]], "orc", ooff[0][bad[:10]], "experts", prob.sel[0][bad[:10]])
stage("fwd dispatch", lambda: L.dispatch_group_gemm(x, wu))
y = stage("fwd combine", lambda: L.group_gemm_combine(wd))
g = stage("bwd", lambda: L.backward(dy, wu, wd))
if y is not None:
    ref = prob.oracle()
    yr = (ref["y"][0].astype(np.uint32) << 16).view(np.float32)
    yg = (to_u16(y).astype(np.uint32) << 16).view(np.float32)
    print("y max abs err", np.abs(yr - yg).max(), "ref max", np.abs(yr).max())
    if g is not None:
        for key in ("dx", "dw_up", "dw_down"):
            a = (to_u16(g[key]).astype(np.uint32) << 16).view(np.float32).ravel()
            b = (ref[key].astype(np.uint32) << 16).view(np.float32).ravel()
            print(key, "max abs err", np.abs(a - b).max(), "ref max", np.abs(b).max())
        a = g["dgate"].cpu().numpy().ravel(); b = ref["dgate"].ravel()
        print("dgate max abs err", np.abs(a - b).max(), "ref max", np.abs(b).max())
