"""Small EP-MoE steps for compute-sanitizer (tools/sanitize.sh): EP=1 fused, EP=2 virtual ranks
(relay off and on), the unfused baseline, and an aborted iteration (bad routing), each checked."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests.test_moe_gpu import Problem, gather, run_layer  # noqa: E402
from tests.test_unfused_gpu import run_unfused  # noqa: E402

prob = Problem(1, 8, 2, 256, 256, 200, seed=3)
a = gather(run_layer(prob)[0][0])
b = gather(run_unfused(prob, 1))
assert all((a[k] == b[k]).all() for k in a), "EP=1 fused != unfused"
prob2 = Problem(2, 16, 4, 256, 256, 96, seed=5)
r0 = gather(run_layer(prob2, cfg=(4, 0, 1, 74, 8))[0][0])
r1 = gather(run_layer(prob2, cfg=(2, 2, 1, 74, 8))[0][0])
assert all((r0[k] == r1[k]).all() for k in r0), "EP=2 relay on != off"
from paper_2604_19241_b200 import moe as M  # noqa: E402
L = M.EpMoE(256, 256, 8, 2, 64, timeout_s=60.0)
ids = torch.stack([torch.arange(64) % 8, (torch.arange(64) + 1) % 8], 1).int().cuda()
ids[3, 1] = 9  # out of range: the iteration must abort without touching memory
L.forward(torch.zeros(64, 256, dtype=torch.bfloat16, device="cuda"), ids, torch.full((64, 2), 0.5, device="cuda"),
          torch.zeros(8, 512, 256, dtype=torch.bfloat16, device="cuda"),
          torch.zeros(8, 256, 256, dtype=torch.bfloat16, device="cuda"))
try:
    L.check()
    raise SystemExit("expected error 2")
except M.EplabError as e:
    assert e.code == 2
L.close()
torch.cuda.synchronize()
print("sanitize cases ok", flush=True)
