"""Per-element error histograms of the GPU layer against the CPU oracle, in bf16 ulps of the oracle
value (the basis of the per-element tolerance in tests/test_parity_gpu.py).

  python tools/ulp_report.py [--shapes small,mid]      (needs a GPU)
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tests.test_moe_gpu import Problem, bf16_to_f32, gather, run_layer  # noqa: E402
from tests.parity import ulp_stats  # noqa: E402

SHAPES = {
    "e8k2": (1, 8, 2, 512, 512, 384),
    "e16k4": (1, 16, 4, 512, 512, 200),
    "e32k8": (1, 32, 8, 1024, 256, 256),
    "ep2": (2, 16, 4, 256, 512, 192),
}

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default=",".join(SHAPES))
args = ap.parse_args()
for name in args.shapes.split(","):
    W, E, k, H, F, T = SHAPES[name]
    prob = Problem(W, E, k, H, F, T, seed=5)
    outs, _, _ = run_layer(prob)
    got = gather(outs[0])
    ref = prob.oracle()
    rep = {"shape": name}
    for key in ("y", "dx", "dw_up", "dw_down"):
        rep[key] = ulp_stats(bf16_to_f32(got[key]).reshape(-1), bf16_to_f32(ref[key]).reshape(-1))
    rep["dgate"] = ulp_stats(got["dgate"].reshape(-1), ref["dgate"].reshape(-1), fp32=True)
    print(json.dumps(rep), flush=True)
