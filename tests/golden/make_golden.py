"""Regenerates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref), so the
oracle and the device token map can be checked where /root/reference is absent.
Run: python tests/golden/make_golden.py   (needs `make -C oracle` with the reference mounted)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

REF = po.Reference()


def vectors(n_exp, topk, n_tok, world, seed):
    sel, gw = REF.sample_routing(n_exp, topk, n_tok, world, seed)
    tr, le, off, rt, sb = REF.token_map(sel, n_exp, topk)
    out = dict(n_exp=n_exp, topk=topk, n_tok=n_tok, world=world, seed=seed, sel=sel, gw=gw,
               target_rank=tr, local_expert=le, offset=off, recv_totals=rt, seg_base=sb)
    for r in range(world):
        tok, slot, dr, de, do = REF.send_schedule(sel, n_exp, topk, r)
        out[f"sched{r}_token"] = tok
        out[f"sched{r}_slot"] = slot
    return out


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    # C0-like small config (8 experts top-2, simulated EP=2), the reference's recurring seed 7
    np.savez_compressed(os.path.join(here, "reference_vectors.npz"), **vectors(8, 2, 512, 2, 7))
    # Qwen3-like routing at EP=8 (128 experts top-8), seed 1
    np.savez_compressed(os.path.join(here, "reference_vectors_ep8.npz"), **vectors(128, 8, 256, 8, 1))
    print("wrote fixtures")
