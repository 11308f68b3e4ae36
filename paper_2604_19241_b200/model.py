"""Launch-parameter selection for the MegaKernels (the paper's performance model + tuner,
PAPER.md:309-399; reference perf_model.cpp / tuner.cpp)."""
from .moe import TuneConfig


def choose_config(H, F, E, k, tokens, world, n_sm=148):
    """TuneConfig for one layer shape. EP=1: AllToAll-style local permute (every replica written
    by the comm warps, relay off). EP>1: AllGather-style dedup with relay workers."""
    if world == 1:
        return TuneConfig(32, 0, 0, n_sm, 8)
    return TuneConfig(24, 8, 0, n_sm, 8)
