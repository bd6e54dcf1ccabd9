"""Seeded synthetic inputs shaped like the paper's workloads.

Shared by tests/, bench.py and __graft_entry__.smoke(); holds NONE of the
method's arithmetic (no compression, orthonormalisation or reconstruction),
only the value distributions of DESIGN.md §4:

  D1  i.i.d. N(0, 1e-3^2)                       flat spectrum, worst case
  D2  gradient-like: rank-64 part with sigma_i ~ 1/i plus 10% i.i.d. noise
  D3  LEP stream: M_t = B + N_t, B fixed from D2, N_t fresh per micro-batch
  D4  exact low rank: integer factors in {-2..2} (exact in fp32 and bf16)
  D5  embedding gradient: row-sparse (Zipf(1.1) token ids) or dense D2

Shapes come from the paper's GPT configurations (Table 1:
hidden 1920 / 3072, micro-batch 8) with seq 1024 (BASELINE.json configs);
[seq, mb, h] is matricised as (seq*mb) x h (reading C6).

Seed convention: seed = 1000*config + 10*rank + step; Q0 uses a seed that is
identical on every rank (reading C5).
"""
from __future__ import annotations

import numpy as np


def _rng(seed):
    return np.random.default_rng(seed)


def d1_iid(n, m, seed, sigma=1e-3):
    return (sigma * _rng(seed).standard_normal((n, m))).astype(np.float32)


def _orthonormal_basis(rng, n, k):
    # Gaussian matrix made orthonormal with numpy's QR: a data-generation step
    # (it only shapes the synthetic spectrum), not part of the method.
    g = rng.standard_normal((n, k))
    q, _ = np.linalg.qr(g)
    return q


def d2_gradlike(n, m, seed, rank=64, noise=0.1, scale=1e-2):
    rng = _rng(seed)
    k = min(rank, n, m)
    U = _orthonormal_basis(rng, n, k)
    V = _orthonormal_basis(rng, m, k)
    sig = scale / np.arange(1, k + 1, dtype=np.float64)
    B = (U * sig) @ V.T
    N = rng.standard_normal((n, m))
    N *= noise * np.linalg.norm(B) / np.linalg.norm(N)
    return (B + N).astype(np.float32)


def d3_lep_stream(n, m, seed, steps, rank=64, noise=0.1):
    base = d2_gradlike(n, m, seed, rank=rank, noise=0.0).astype(np.float64)
    rng = _rng(seed + 7)
    nb = np.linalg.norm(base)
    out = []
    for _ in range(steps):
        N = rng.standard_normal((n, m))
        N *= noise * nb / np.linalg.norm(N)
        out.append((base + N).astype(np.float32))
    return out


def d4_exact_lowrank(n, m, k, seed):
    rng = _rng(seed)
    U = rng.integers(-2, 3, size=(n, k)).astype(np.float64)
    V = rng.integers(-2, 3, size=(m, k)).astype(np.float64)
    return (U @ V.T).astype(np.float32)


def d5_embedding_sparse(vocab, h, seed, tokens=8192, zipf_a=1.1, scale=1e-3):
    """Input-embedding gradient: rows of the tokens seen in the micro-batch."""
    rng = _rng(seed)
    ids = rng.zipf(zipf_a, size=tokens) - 1
    ids = ids[ids < vocab]
    G = np.zeros((vocab, h), dtype=np.float64)
    np.add.at(G, ids, scale * rng.standard_normal((ids.size, h)))
    return G.astype(np.float32)


def q0(m, r, seed):
    """Initial warm-start factor, N(0,1), same seed on every rank (reading C5)."""
    return _rng(seed).standard_normal((m, r)).astype(np.float32)


def e0(n, m, seed, like=None, rel=0.1):
    """Initial stored error: rel * std(like) * N(0,1) (zero if like is None)."""
    if like is None:
        return np.zeros((n, m), dtype=np.float32)
    s = float(np.std(like.astype(np.float64))) or 1.0
    return (rel * s * _rng(seed).standard_normal((n, m))).astype(np.float32)


def make(dist, n, m, seed, **kw):
    if dist == "D1":
        return d1_iid(n, m, seed, **kw)
    if dist == "D2":
        return d2_gradlike(n, m, seed, **kw)
    if dist == "D4":
        return d4_exact_lowrank(n, m, kw.get("k", 4), seed)
    raise ValueError(dist)
