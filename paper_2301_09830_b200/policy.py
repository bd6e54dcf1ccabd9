"""Host-side switches of Optimus-CC (§8(a) row a10).  Pure Python; decides
WHICH traffic goes through the compressed path, never computes it.

- Epilogue-only compression (§CB.Epilogue; 684 "schedule.py
  was modified to apply compression on the epilogue part").  Reading C10: the
  backward send of micro-batch k from stage s to s-1 is compressed iff the
  receiver s-1 is in its 1F1B cool-down, i.e. k >= M - (P - s).
- Selective stage compression (§SC; 775 "75% stage
  compression").  Reading C11: the ceil(0.75 P) earliest stages.
- Fused embedding synchronisation group (§FE; 687-689 name
  detection of `word_embeddings`): the first- and last-stage ranks of every
  DP replica, 2D ranks in one group.
- Warm-up bypass ("30K of warm-up iterations").
- Rank-1 parameters (bias, LayerNorm) are never compressed (reading C16).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Policy:
    cb_rank: int = 16            # PAPER.md:773 ("16 for compressed backpropagation")
    dp_rank: int = 128           # PAPER.md:773 ("128 for data-parallel gradient compression")
    sc_fraction: float = 0.75
    warmup_iters: int = 30000
    epilogue_only: bool = True
    lep: bool = True             # lazy error propagation on (Non-LEP = PAPER.md:893 ablation)
    fe: bool = True              # fused embedding synchronisation

    def kernel_rank(self, r: int) -> int:
        """The rank the library runs for a requested rank r: the largest built
        instance (4, 8, 16, 32, 64) not above r.  The paper's DP rank 128
         is not built, so DP compression driven by this policy
        runs at 64 (a smaller rank: fewer factor bytes, larger residual, which
        error feedback carries to the next step)."""
        built = (4, 8, 16, 32, 64)
        if r < built[0]:
            raise ValueError(f"rank {r} below the smallest built rank 4")
        return max(b for b in built if b <= r)


def epilogue_compressed(k: int, num_microbatches: int, num_stages: int, stage: int) -> bool:
    """Is the backward send of micro-batch k from `stage` to `stage - 1` compressed?"""
    if not 1 <= stage < num_stages:
        raise ValueError("backward sends leave stages 1..P-1")
    if not 0 <= k < num_microbatches:
        raise ValueError("micro-batch index out of range")
    return k >= num_microbatches - (num_stages - stage)


def cb_compressed(policy: Policy, iteration: int, k: int, num_microbatches: int, num_stages: int,
                  stage: int) -> bool:
    if iteration < policy.warmup_iters:
        return False
    if not policy.epilogue_only:
        return True
    return epilogue_compressed(k, num_microbatches, num_stages, stage)


def sc_stages(num_stages: int, fraction: float = 0.75) -> frozenset:
    """Stages whose DP traffic is compressed: the ceil(f P) earliest ones."""
    if not 0.0 <= fraction <= 1.0:
        raise ValueError("fraction in [0, 1]")
    return frozenset(range(math.ceil(fraction * num_stages - 1e-12)))


def dp_compressed(policy: Policy, iteration: int, stage: int, num_stages: int, numel_dims: int) -> bool:
    if numel_dims < 2 or iteration < policy.warmup_iters:
        return False
    return stage in sc_stages(num_stages, policy.sc_fraction)


def is_embedding(param_name: str) -> bool:
    """the embedding is found by the name `word_embeddings`."""
    return "word_embeddings" in param_name


def rank_of(stage: int, dp: int, dp_size: int) -> int:
    """Box layout: stage-major ranks (ranks 0..D-1 = stage 0, ...)."""
    return stage * dp_size + dp


def dp_group(stage: int, dp_size: int) -> list:
    return [rank_of(stage, d, dp_size) for d in range(dp_size)]


def pp_group(dp: int, dp_size: int, num_stages: int) -> list:
    return [rank_of(s, dp, dp_size) for s in range(num_stages)]


def fe_group(dp_size: int, num_stages: int) -> list:
    """2D ranks holding a copy of the tied embedding (first + last stage)."""
    if num_stages == 1:
        return dp_group(0, dp_size)
    return dp_group(0, dp_size) + dp_group(num_stages - 1, dp_size)


def fe_scale(dp_size: int) -> float:
    """Reading C12: sum over the 2D ranks of G / D = mean(first) + mean(last)."""
    return 1.0 / dp_size
