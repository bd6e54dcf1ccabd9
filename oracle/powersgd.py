"""Plain, slow, obviously-correct CPU oracle for the Optimus-CC hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this module.
The product path (`paper_2301_09830_b200`) never imports it, and this module
never imports the product path: the two share no code.

Everything is NumPy float64 (the paper fixes no precision: PAPER.md:678
"native PyTorch 1.8 APIs" only).  Each function follows the paper's algorithm
step by step, in the paper's order; library primitives used as single steps
are `@` (matmul) and `numpy.linalg.norm`.

Citations are PAPER.md line numbers (sections are unnumbered in the LaTeX, so
they are named: §Background, §CB (compressed backpropagation), §FE (fused
embedding synchronisation), §SC (selective stage compression), §Impl, §Eval)
plus SPEC.md line numbers for operation contracts.  Readings of points the
paper leaves open are the C-numbered readings of SURVEY.md §8(c) and are
listed in DESIGN.md §3.

Sign convention (reading C19): the paper adds a compression error
eps to the sent value (Eq. star2); here the stored error is
e = A - M' = -eps, exactly as the north_star states ("set e_new = M+e-M'").

Parity status: every function below is pinned by `tests/test_oracle_pins.py`
(hand-worked examples, closed forms, invariants, brute-force SVD bounds,
library-routine special cases).  No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------
# Deterministic fallback vectors for degenerate columns (reading C3).
# SPEC.md:43 / 64-65: "rank-deficient column ... replaced by a deterministic
# pseudo-random unit vector re-orthogonalized against previous columns".
# The generator is counter based (splitmix64), so the CUDA side implements the
# same formula independently (no shared code, per the task's rule ③).
# --------------------------------------------------------------------------

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def splitmix64(x: int) -> int:
    """splitmix64 finaliser of (x + golden gamma), 64-bit wraparound.

    splitmix64(0) is the first output of the seed-0 SplitMix64 stream,
    0xE220A8397B1DCDAF (pinned in tests/golden/splitmix64.json).
    """
    z = (x + _GOLDEN) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def fallback_vector(seed: int, j: int, n: int) -> np.ndarray:
    """Column j's fallback vector, length n, entries in [-1, 1).

    f[i] = (splitmix64(seed ^ (j << 32) ^ i) >> 40) * 2**-23 - 1.
    The 24-bit value k*2**-23 - 1 is exactly representable in fp32, so an
    fp32 GPU and this fp64 oracle hold bit-identical fallback columns.
    """
    out = np.empty(n, dtype=np.float64)
    base = (seed ^ (j << 32)) & _MASK64
    for i in range(n):
        out[i] = (splitmix64(base ^ i) >> 40) * 2.0 ** -23 - 1.0
    return out


# --------------------------------------------------------------------------
# Orthonormalisation (a4).  PAPER.md:1006 (§Eval "the orthogonalization phase
# is the main bottleneck"), PAPER.md:269 (PowerSGD power iteration);
# SPEC.md:39-47 (orthogonalize contract: MGS with re-normalisation + fallback).
# Reading C3: two-pass modified Gram-Schmidt (MGS2) in fp64; a column whose
# norm after projection is below tau * (its own norm before projection), or
# whose own norm is 0, is replaced by its fallback vector.
# --------------------------------------------------------------------------

def mgs2(P: np.ndarray, tau: float = 1e-5, fb_seed: int = 0):
    """Return (P_hat, fallback_columns) with P_hat^T P_hat = I.

    For full-column-rank P, P_hat spans the same space and P = P_hat R with
    R upper triangular, diag(R) > 0 (so P_hat is unique: reading C4).
    """
    P = np.asarray(P, dtype=np.float64)
    n, r = P.shape
    if r > n:
        raise ValueError("orthogonalize requires rows >= cols (SPEC.md:40)")
    Ph = np.zeros((n, r), dtype=np.float64)
    fallbacks = []
    for j in range(r):
        v = P[:, j].copy()
        n0 = np.linalg.norm(v)
        for _ in range(2):                       # two MGS passes
            for i in range(j):
                v = v - (Ph[:, i] @ v) * Ph[:, i]
        if n0 == 0.0 or np.linalg.norm(v) < tau * n0:
            v = fallback_vector(fb_seed, j, n)
            fallbacks.append(j)
            for _ in range(2):                   # re-orthogonalise the fallback
                for i in range(j):
                    v = v - (Ph[:, i] @ v) * Ph[:, i]
        Ph[:, j] = v / np.linalg.norm(v)
    return Ph, fallbacks


# --------------------------------------------------------------------------
# Output rounding (reading C7): M' is delivered in M's dtype.  bf16 rounding
# is round-to-nearest-even straight from fp64 (8 significant bits).
# --------------------------------------------------------------------------

def round_to(x: np.ndarray, out_dtype: str) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if out_dtype == "f64":
        return x.copy()
    if out_dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    if out_dtype == "bf16":
        m, ex = np.frexp(x)                      # x = m * 2**ex, 0.5 <= |m| < 1
        return np.ldexp(np.rint(m * 256.0), ex - 8)   # rint = half-to-even
    raise ValueError(out_dtype)


# --------------------------------------------------------------------------
# One LEP / P2P compression step (a1, a2, a4, a5, a7, a8, a9).
# PAPER.md:269-270 (one power iteration, reuse of the factor)
# (lazy error propagation worked example), PAPER.md:436-441 (Eq. star2),
# SPEC.md:114-136 (lowrank_compress / lowrank_decompress / lazy_step).
# --------------------------------------------------------------------------

def compress_step(M, e_old, Q_prev, *, out_dtype: str = "f64", tau: float = 1e-5,
                  fb_seed: int = 0, no_ef: bool = False, orient_t: bool = False,
                  wire_bf16: bool = False):
    """One warm-started power-iteration step with error feedback.

    A      = M + e_old                 (a1; Non-LEP / NO_EF: e_old treated as 0)
    P      = A Q_prev                  (a2)
    P_hat  = orth(P)                   (a4)
    Q      = A^T P_hat                 (a5; also the next Q_prev, a9)
    M'     = round(P_hat Q^T)          (a7)
    e_new  = A - M'                    (a8)

    orient_t (reading C6, used for the 50257-row embedding): compress A^T
    instead of A; M' and e_new are returned in A's stored layout.
    wire_bf16 (reading C7, OCC_WIRE_BF16): the factors are computed as above
    and then rounded to bf16 (RNE) for the wire; M' and e_new are taken
    against the rounded factors, which are also the returned P_hat and Q.
    Returns a dict with P_hat, Q, recon (M'), err (e_new), fallbacks.
    """
    M = np.asarray(M, dtype=np.float64)
    A = M.copy() if (no_ef or e_old is None) else M + np.asarray(e_old, dtype=np.float64)
    X = A.T if orient_t else A
    Q_prev = np.asarray(Q_prev, dtype=np.float64)
    P = X @ Q_prev
    P_hat, fb = mgs2(P, tau, fb_seed)
    Q = X.T @ P_hat
    if wire_bf16:
        P_hat, Q = round_to(P_hat, "bf16"), round_to(Q, "bf16")
    R = round_to(P_hat @ Q.T, out_dtype)
    if orient_t:
        R = R.T
    return {"P_hat": P_hat, "Q": Q, "recon": R, "err": A - R, "fallbacks": fb, "P": P}


def decompress(P_hat, Q, *, out_dtype: str = "f64", orient_t: bool = False):
    """SPEC.md:123-131 lowrank_decompress: M' = round(P_hat Q^T)."""
    R = round_to(np.asarray(P_hat, np.float64) @ np.asarray(Q, np.float64).T, out_dtype)
    return R.T if orient_t else R


# --------------------------------------------------------------------------
# Data-parallel step (a1-a9 with a3/a6 as sums over ranks), simulated
# in-process over the ranks of the group.  PAPER.md:676-677 (PowerSGD adopted
# for DP gradient compression), PAPER.md:657 (error sent to the next
# iteration), SPEC.md:141-144 (ef_step).  Reading C1: allreduce(P) BEFORE the
# orthonormalisation, allreduce(Q) after Q_w = A_w^T P_hat.  Reading C2: local
# error convention by default (e_w = A_w - P_hat Q_w^T); ef_global gives
# e_w = A_w - M'.  Reading C15: both exchanges are sums; Q is scaled after.
# --------------------------------------------------------------------------

def dp_step(M_list, e_list, Q_prev, *, scale: float, out_dtype: str = "f64",
            tau: float = 1e-5, fb_seed: int = 0, ef_global: bool = False,
            no_ef: bool = False, orient_t: bool = False):
    R = len(M_list)
    A = []
    for w in range(R):
        Mw = np.asarray(M_list[w], dtype=np.float64)
        if no_ef or e_list is None or e_list[w] is None:
            A.append(Mw.copy())
        else:
            A.append(Mw + np.asarray(e_list[w], dtype=np.float64))
    X = [a.T if orient_t else a for a in A]
    Q_prev = np.asarray(Q_prev, dtype=np.float64)
    P = sum(X[w] @ Q_prev for w in range(R))           # a2 + a3 (allreduce-sum P)
    P_hat, fb = mgs2(P, tau, fb_seed)                   # a4
    Q_w = [X[w].T @ P_hat for w in range(R)]            # a5
    Q_sum = sum(Q_w)                                    # a6 (allreduce-sum Q)
    Q_s = scale * Q_sum                                 # reading C15
    Rm = round_to(P_hat @ Q_s.T, out_dtype)             # a7 (same on every rank)
    errs = []
    for w in range(R):
        if ef_global:
            ew = X[w] - Rm
        else:
            ew = X[w] - P_hat @ Q_w[w].T                # local convention (C2)
        errs.append(ew.T if orient_t else ew)
    recon = Rm.T if orient_t else Rm
    return {"P_hat": P_hat, "Q_w": Q_w, "Q": Q_s, "recon": recon, "err": errs,
            "fallbacks": fb, "P": P}


# --------------------------------------------------------------------------
# Fused embedding synchronisation (FE).  PAPER.md:598-618: the two
# allreduces (EMB-DP over D ranks, EMB-sync over 2 ranks) are fused into one
# allreduce over 2D ranks; the mathematics is unchanged.  Reading C12: the
# tied embedding's gradient is the SUM of its two uses ("aggregate gradients
# from multiple paths"), each use averaged over its D replicas.
# --------------------------------------------------------------------------

def embed_sync_sequential(G_first, G_last):
    """Baseline: mean over D replicas per stage, then the 2-rank sum."""
    D = len(G_first)
    g1 = sum(np.asarray(g, np.float64) for g in G_first) / D
    g2 = sum(np.asarray(g, np.float64) for g in G_last) / D
    return g1 + g2


def embed_sync_fused(G_all, D: int):
    """Fused: one sum over all 2D ranks of (1/D) * G."""
    return sum((1.0 / D) * np.asarray(g, np.float64) for g in G_all)
