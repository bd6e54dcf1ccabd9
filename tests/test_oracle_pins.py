"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: hand-worked
exact values (tests/golden, with citations), closed forms, invariants the
mathematics fixes, library routines (numpy QR / SVD, torch bf16 cast) on the
special cases that reduce to them, and brute force on tiny inputs.  The set is
chosen so that a dropped term, a wrong sign or index, or a transposed operand
anywhere in oracle/ fails at least one test (see the comment on each).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import powersgd as ops
from workloads import synth


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# --------------------------------------------------------------- splitmix64
def test_splitmix64_published_vectors(golden_dir):
    g = _load(golden_dir, "splitmix64.json")
    assert oracle.splitmix64(0) == int(g["seed0_first"], 16)
    gamma = 0x9E3779B97F4A7C15
    s = 1234567
    got = [oracle.splitmix64((s + k * gamma) % 2**64) for k in range(5)]
    assert got == g["seed1234567_first5"]


def test_fallback_vector_range_and_fp32_exact():
    f = oracle.fallback_vector(7, 3, 1000)
    assert f.min() >= -1.0 and f.max() < 1.0
    assert np.array_equal(f.astype(np.float32).astype(np.float64), f)
    # different column index -> different vector (j enters the counter)
    assert not np.array_equal(f, oracle.fallback_vector(7, 4, 1000))


# ------------------------------------------------------- P1: hand example
def test_p1_hand_example_two_lep_steps(golden_dir):
    """Catches: dropped error add (step 2), transposed A (A is non-symmetric
    in step 2), sign of e, wrong warm-start factor."""
    g = _load(golden_dir, "p1_hand_example.json")
    M = np.array(g["M"], float)
    Q0 = np.array(g["Q0"], float)
    s1 = oracle.compress_step(M, None, Q0)
    h = g["step1"]
    np.testing.assert_allclose(s1["P_hat"], np.array(h["P_hat_num"]) / math.sqrt(h["P_hat_den_sqrt"]), atol=1e-15)
    np.testing.assert_allclose(s1["Q"], np.array(h["Q_num"]) / math.sqrt(h["Q_den_sqrt"]), atol=1e-15)
    np.testing.assert_allclose(s1["recon"], np.array(h["recon_num"]) / h["recon_den"], atol=1e-15)
    np.testing.assert_allclose(s1["err"], np.array(h["err_num"]) / h["err_den"], atol=1e-15)
    s2 = oracle.compress_step(M, s1["err"], s1["Q"])
    h = g["step2"]
    np.testing.assert_allclose(s2["P_hat"], np.array(h["P_hat_num"]) / math.sqrt(h["P_hat_den_sqrt"]), atol=1e-15)
    np.testing.assert_allclose(s2["Q"], np.array(h["Q_num"]) / math.sqrt(h["Q_den_sqrt"]), atol=1e-14)
    np.testing.assert_allclose(s2["recon"], np.array(h["recon_num"]) / h["recon_den"], atol=1e-14)
    A2 = np.array(h["A_num"]) / h["A_den"]
    np.testing.assert_allclose(s2["err"], A2 - np.array(h["recon_num"]) / h["recon_den"], atol=1e-14)
    # P9 on the hand example: M'_1 + M'_2 = 2M - e_2
    np.testing.assert_allclose(s1["recon"] + s2["recon"], 2 * M - s2["err"], atol=1e-14)


# ------------------------------------------------------- P2: orthonormalise
def test_p2_spec_examples():
    ph, fb = oracle.mgs2(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(ph, [[0.6], [0.8]], atol=1e-15)
    assert fb == []
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((16, 4)))
    q = q * np.sign(np.diag(np.linalg.qr(q)[1]))  # any orthonormal Q
    ph, _ = oracle.mgs2(q)
    s = np.sign(np.sum(ph * q, axis=0))
    np.testing.assert_allclose(ph, q * s, atol=1e-12)  # SPEC.md:45 idempotence


@pytest.mark.parametrize("n,r,seed", [(16, 4, 0), (200, 16, 1), (512, 64, 2)])
def test_p2_matches_numpy_qr_sign_fixed(n, r, seed):
    """Full-rank P: P_hat equals Householder QR's Q with diag(R) > 0 (a
    library routine).  Catches: one MGS pass only, wrong projection index."""
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((n, r)) @ np.diag(np.logspace(0, 2, r))
    ph, fb = oracle.mgs2(P)
    q, R = np.linalg.qr(P)
    q = q * np.sign(np.diag(R))
    assert fb == []
    np.testing.assert_allclose(ph, q, atol=1e-12)
    assert np.linalg.norm(ph.T @ ph - np.eye(r)) < 1e-13
    Rm = ph.T @ P
    assert np.allclose(np.tril(Rm, -1), 0, atol=1e-12) and np.all(np.diag(Rm) > 0)


def test_p2_degenerate_columns_take_fallback():
    n = 32
    rng = np.random.default_rng(3)
    a = rng.standard_normal(n)
    P = np.stack([a, 2 * a, np.zeros(n), rng.standard_normal(n)], axis=1)
    ph, fb = oracle.mgs2(P, fb_seed=11)
    assert fb == [1, 2]
    assert np.linalg.norm(ph.T @ ph - np.eye(4)) < 1e-13
    # column 1 is the fallback vector orthogonalised against column 0
    f = oracle.fallback_vector(11, 1, n)
    p0 = a / np.linalg.norm(a)
    v = f - (p0 @ f) * p0
    np.testing.assert_allclose(ph[:, 1], v / np.linalg.norm(v), atol=1e-13)


# ---------------------------------------------- P4 / P5: identities
@pytest.mark.parametrize("dist", ["D1", "D2"])
def test_p4_p5_ef_and_projection_identities(dist):
    n, m, r = 96, 160, 8
    M = synth.make(dist, n, m, 5).astype(np.float64)
    e = synth.e0(n, m, 6, like=M)
    Q0 = synth.q0(m, r, 7)
    s = oracle.compress_step(M, e, Q0)
    A = M + e
    # P4: EF identity M' + e_new = M + e_old      (catches a dropped term)
    np.testing.assert_allclose(s["recon"] + s["err"], A, atol=1e-15 * np.abs(A).max() * 10)
    # P5: P_hat^T e_new = 0; |A|^2 = |M'|^2 + |e|^2; |Q|_F = |M'|_F
    nA = np.linalg.norm(A)
    assert np.linalg.norm(s["P_hat"].T @ s["err"]) < 1e-13 * nA
    assert abs(nA**2 - np.linalg.norm(s["recon"])**2 - np.linalg.norm(s["err"])**2) < 1e-13 * nA**2
    assert abs(np.linalg.norm(s["Q"]) - np.linalg.norm(s["recon"])) < 1e-13 * nA
    # P = A Q0 exactly as defined (catches a transposed operand)
    np.testing.assert_allclose(s["P"], A @ Q0.astype(np.float64), rtol=1e-13, atol=1e-18)


# ---------------------------------------------- P6: SVD bounds
def test_p6_eckart_young_and_warm_start_convergence():
    rng = np.random.default_rng(8)
    A = rng.standard_normal((64, 64))
    r = 8
    sv = np.linalg.svd(A, compute_uv=False)
    opt = math.sqrt(np.sum(sv[r:] ** 2))
    Q = rng.standard_normal((64, r))
    errs = []
    for _ in range(10):
        s = oracle.compress_step(A, None, Q, no_ef=True)
        Q = s["Q"]
        errs.append(np.linalg.norm(s["err"]))
        assert errs[-1] >= opt * (1 - 1e-12)              # Eckart-Young
    assert all(b <= a * (1 + 1e-12) for a, b in zip(errs, errs[1:]))  # monotone
    assert errs[-1] <= 2 * opt


# ---------------------------------------------- P7 / P8: special cases
@pytest.mark.parametrize("k,r", [(1, 1), (3, 4), (4, 4), (2, 8)])
def test_p7_exact_low_rank_recovered(k, r):
    M = synth.d4_exact_lowrank(40, 56, k, seed=9).astype(np.float64)
    s = oracle.compress_step(M, None, synth.q0(56, r, 10))
    assert np.linalg.norm(s["err"]) <= 1e-12 * np.linalg.norm(M)
    assert len(s["fallbacks"]) == r - k


def test_p8_zero_input():
    s = oracle.compress_step(np.zeros((20, 30)), np.zeros((20, 30)), synth.q0(30, 4, 1))
    assert np.all(s["recon"] == 0) and np.all(s["err"] == 0)
    assert s["fallbacks"] == [0, 1, 2, 3]
    assert np.linalg.norm(s["P_hat"].T @ s["P_hat"] - np.eye(4)) < 1e-13


def test_p8_full_rank_is_lossless_and_zero_error_equals_no_ef():
    rng = np.random.default_rng(12)
    M = rng.standard_normal((6, 9))
    s = oracle.compress_step(M, None, rng.standard_normal((9, 6)))     # r = n <= m
    assert np.abs(s["err"]).max() < 1e-12
    Q0 = rng.standard_normal((9, 3))
    a = oracle.compress_step(M, np.zeros_like(M), Q0)
    b = oracle.compress_step(M, None, Q0, no_ef=True)
    np.testing.assert_array_equal(a["recon"], b["recon"])


def test_p8_scaling_invariance():
    rng = np.random.default_rng(13)
    M = rng.standard_normal((30, 20))
    Q0 = rng.standard_normal((20, 5))
    a = oracle.compress_step(M, None, Q0)
    b = oracle.compress_step(4.0 * M, None, Q0)
    np.testing.assert_allclose(b["P_hat"], a["P_hat"], atol=1e-13)
    np.testing.assert_allclose(b["Q"], 4.0 * a["Q"], atol=1e-12)


# ---------------------------------------------- P9: telescoping (LEP)
def test_p9_telescoping_over_micro_batches():
    n, m, r, T = 64, 48, 4, 12
    Ms = synth.d3_lep_stream(n, m, 21, T)
    e = synth.e0(n, m, 22, like=Ms[0]).astype(np.float64)
    e_init = e.copy()
    Q = synth.q0(m, r, 23)
    tot = np.zeros((n, m))
    for Mt in Ms:
        s = oracle.compress_step(Mt, e, Q)
        e, Q = s["err"], s["Q"]
        tot += s["recon"]
    expect = sum(x.astype(np.float64) for x in Ms) + e_init - e
    assert np.linalg.norm(tot - expect) <= 1e-12 * np.linalg.norm(expect)


# ---------------------------------------------- orientation (reading C6)
def test_orient_t_is_compression_of_the_transpose():
    rng = np.random.default_rng(14)
    M = rng.standard_normal((40, 12))
    e = rng.standard_normal((40, 12))
    Q0 = rng.standard_normal((40, 3))    # Q lives on the 40-row side
    a = oracle.compress_step(M, e, Q0, orient_t=True)
    b = oracle.compress_step(M.T, e.T, Q0)
    np.testing.assert_allclose(a["recon"], b["recon"].T, atol=1e-13)
    np.testing.assert_allclose(a["err"], b["err"].T, atol=1e-13)
    assert a["P_hat"].shape == (12, 3)


# ---------------------------------------------- P10: data parallel
def test_p10_dp_hand_example(golden_dir):
    g = _load(golden_dir, "p10_dp_hand_example.json")
    Ms = [np.array(x, float) for x in g["M"]]
    Q0 = np.array(g["Q0"], float)
    sc = g["scale_num"] / g["scale_den"]
    loc = oracle.dp_step(Ms, None, Q0, scale=sc)
    glo = oracle.dp_step(Ms, None, Q0, scale=sc, ef_global=True)
    np.testing.assert_allclose(loc["P_hat"], np.array(g["P_hat_num"]) / math.sqrt(2), atol=1e-15)
    np.testing.assert_allclose(loc["Q"], np.array(g["Q_num"]) / math.sqrt(2), atol=1e-15)
    np.testing.assert_allclose(loc["recon"], np.array(g["recon_num"]) / g["recon_den"], atol=1e-15)
    for w in range(2):
        np.testing.assert_allclose(loc["err"][w], np.array(g["err_local_num"][w]) / 2, atol=1e-15)
        np.testing.assert_allclose(glo["err"][w], np.array(g["err_global_num"][w]) / 2, atol=1e-15)
    np.testing.assert_allclose(sum(loc["err"]), np.array(g["err_sum"], float), atol=1e-15)
    np.testing.assert_allclose(sum(glo["err"]), np.array(g["err_sum"], float), atol=1e-15)


def test_p10_dp_invariants():
    rng = np.random.default_rng(15)
    n, m, r, D = 30, 44, 5, 4
    Ms = [rng.standard_normal((n, m)) for _ in range(D)]
    es = [0.1 * rng.standard_normal((n, m)) for _ in range(D)]
    Q0 = rng.standard_normal((m, r))
    d = oracle.dp_step(Ms, es, Q0, scale=1.0 / D)
    As = [Ms[w] + es[w] for w in range(D)]
    Ph = d["P_hat"]
    # M' = scale * P_hat P_hat^T sum_w A_w     (catches a wrong scale / order)
    np.testing.assert_allclose(d["recon"], (1.0 / D) * Ph @ Ph.T @ sum(As), atol=1e-12)
    # sum of local errors == sum of global errors when R*scale == 1
    g = oracle.dp_step(Ms, es, Q0, scale=1.0 / D, ef_global=True)
    np.testing.assert_allclose(sum(d["err"]), sum(g["err"]), atol=1e-12)
    # D = 1 reduces to the P2P step
    one = oracle.dp_step(Ms[:1], es[:1], Q0, scale=1.0)
    p2p = oracle.compress_step(Ms[0], es[0], Q0)
    np.testing.assert_allclose(one["recon"], p2p["recon"], atol=1e-13)
    np.testing.assert_allclose(one["err"][0], p2p["err"], atol=1e-13)


# ---------------------------------------------- P11: FE + cost model
def test_p11_fused_embedding_equals_sequential():
    rng = np.random.default_rng(16)
    D = 4
    first = [rng.standard_normal((50, 8)) for _ in range(D)]
    last = [rng.standard_normal((50, 8)) for _ in range(D)]
    a = oracle.embed_sync_sequential(first, last)
    b = oracle.embed_sync_fused(first + last, D)
    assert np.abs(a - b).max() <= 1e-12
    same = [np.ones((3, 3))] * (2 * D)
    assert np.array_equal(oracle.embed_sync_sequential(same[:D], same[D:]),
                          oracle.embed_sync_fused(same, D))


def test_p11_cost_model_closed_forms(golden_dir):
    g = _load(golden_dir, "paper_costmodel.json")
    V = Fraction(1)
    for D in range(1, 9):
        assert oracle.c_emb(V, D) == V * Fraction(3 * D - 2, D)
        assert oracle.c_emb_fused(V, D) == V * Fraction(2 * D - 1, D)
        assert oracle.c_emb_fused(V, D) <= oracle.c_emb(V, D)
    benefit = oracle.c_emb(V, 4) / oracle.c_emb_fused(V, 4) - 1
    assert benefit == Fraction(*g["fe_benefit_D4_exact"])
    assert round(float(benefit) * 100, 1) == g["fe_benefit_D4_percent_printed"]
    lim = oracle.c_emb(V, 10**6) / oracle.c_emb_fused(V, 10**6)
    assert abs(float(lim) - 1.5) < 1e-5
    ex = g["allreduce_example"]
    t = oracle.allreduce_cost(ex["V_bytes"], ex["R"]) / ex["bw_Bps"]
    assert abs(float(t) - ex["seconds"]) < 1e-15
    assert oracle.allreduce_cost(5, 1) == 0


def test_p12_compression_ratio(golden_dir):
    g = _load(golden_dir, "paper_costmodel.json")
    for n, m, r, want in g["compression_ratio_examples"]:
        assert oracle.compression_ratio(n, m, r) == want


# ---------------------------------------------- bf16 rounding (reading C7)
def test_round_bf16_matches_torch_and_ties_to_even():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(17).standard_normal(10000).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(oracle.round_to(x.astype(np.float64), "bf16"), want)
    ties = np.array([1 + 2.0**-8, 1 + 3 * 2.0**-8, -(1 + 2.0**-8)])
    np.testing.assert_array_equal(oracle.round_to(ties, "bf16"), [1.0, 1 + 2.0**-6, -1.0])


def test_wire_bf16_rounds_factors_to_bf16():
    """Reading C7 (OCC_WIRE_BF16): the returned factors are bf16 values (the low
    16 bits of their fp32 encoding are zero), each within half a bf16 ulp of
    the fp64 factor (RNE), and the EF identity M' + e_new = A still holds."""
    M = synth.d2_gradlike(64, 48, 1)
    e = synth.e0(64, 48, 2, like=M)
    Q0 = synth.q0(48, 4, 3)
    a = oracle.compress_step(M, e, Q0)
    b = oracle.compress_step(M, e, Q0, wire_bf16=True)
    for key in ("P_hat", "Q"):
        f32 = b[key].astype(np.float32)
        assert np.array_equal(f32.astype(np.float64), b[key])
        assert np.all((f32.view(np.uint32) & 0xFFFF) == 0)
        ulp = np.ldexp(1.0, np.frexp(np.abs(a[key]))[1] - 8)   # bf16 spacing at |x|
        assert np.all(np.abs(b[key] - a[key]) <= 0.5 * ulp + 1e-300)
    A = M.astype(np.float64) + e
    assert np.allclose(b["recon"] + b["err"], A, rtol=0, atol=1e-12)


# ---------------------------------------------- round-2 pins ("What's weak" 1)
def test_fallback_vector_formula_against_published_splitmix64(golden_dir):
    """f[i] = (splitmix64(seed ^ (j << 32) ^ i) >> 40) 2^-23 - 1 (reading C3).
    The counter is chosen so that it equals a published SplitMix64 state
    (s + k*gamma): then f[i] follows from the published output alone.  Catches
    a wrong shift of j, a wrong >> (e.g. 41), a wrong scale or offset."""
    g = _load(golden_dir, "splitmix64.json")
    gamma, s = 0x9E3779B97F4A7C15, 1234567
    for k, pub in enumerate(g["seed1234567_first5"]):
        j, i = k + 1, 5 + 3 * k
        x = (s + k * gamma) % 2**64                  # the published stream's k-th counter
        seed = x ^ (j << 32) ^ i                     # so that seed ^ (j<<32) ^ i == x
        f = oracle.fallback_vector(seed, j, i + 1)
        assert f[i] == (pub >> 40) * 2.0**-23 - 1.0
    # seed 0, j 0, i 0: splitmix64(0) = 0xE220A8397B1DCDAF -> 0xE220A8 / 2^23 - 1, exact
    f0 = oracle.fallback_vector(0, 0, 1)[0]
    assert f0 == Fraction(0xE220A8 - 2**23, 2**23)


def test_decompress_hand_values_and_orientation():
    """SPEC.md:123-131 lowrank_decompress: M' = round(P_hat Q^T).  Hand values
    (an outer product), the transpose under orient_t, bf16 RNE on a tie."""
    P = np.array([[1.0], [2.0]])
    Q = np.array([[3.0], [5.0], [7.0]])
    want = np.array([[3.0, 5, 7], [6, 10, 14]])
    np.testing.assert_array_equal(oracle.decompress(P, Q), want)
    np.testing.assert_array_equal(oracle.decompress(P, Q, orient_t=True), want.T)
    # rank 2: the sum of two outer products (a dropped column fails)
    P2 = np.array([[1.0, 0.0], [0.0, 1.0]])
    Q2 = np.array([[1.0, 2.0], [3.0, 4.0]])
    np.testing.assert_array_equal(oracle.decompress(P2, Q2), [[1.0, 3.0], [2.0, 4.0]])
    # bf16: 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> even (1.0); 1 + 3*2^-8 -> 1 + 2^-6
    tie = oracle.decompress(np.array([[1.0]]), np.array([[1.0 + 2.0**-8], [1.0 + 3 * 2.0**-8]]), out_dtype="bf16")
    np.testing.assert_array_equal(tie, [[1.0, 1.0 + 2.0**-6]])


def test_decompress_reproduces_the_compressors_recon(golden_dir):
    """decompress(P_hat, Q) is the M' that compress_step's e_new was taken
    against, on the P1 hand example (exact values) and with orient_t."""
    g = _load(golden_dir, "p1_hand_example.json")
    M = np.array(g["M"], float)
    s1 = oracle.compress_step(M, None, np.array(g["Q0"], float))
    d = oracle.decompress(s1["P_hat"], s1["Q"])
    np.testing.assert_allclose(d, np.array(g["step1"]["recon_num"]) / g["step1"]["recon_den"], atol=1e-15)
    np.testing.assert_array_equal(d, s1["recon"])
    rng = np.random.default_rng(31)
    A = rng.standard_normal((12, 7))
    s = oracle.compress_step(A, None, rng.standard_normal((12, 3)), orient_t=True)
    np.testing.assert_array_equal(oracle.decompress(s["P_hat"], s["Q"], orient_t=True), s["recon"])
    for dt in ("f32", "bf16"):
        s = oracle.compress_step(A, None, rng.standard_normal((7, 3)), out_dtype=dt)
        np.testing.assert_array_equal(oracle.decompress(s["P_hat"], s["Q"], out_dtype=dt), s["recon"])


def test_dp_orient_t_hand_example(golden_dir):
    """dp_step(orient_t=True) on a hand-worked D = 2 example with a
    non-symmetric A_1 (a dropped transpose fails every value)."""
    g = _load(golden_dir, "p10t_dp_orient_t_hand_example.json")
    As = [np.array(x, float) for x in g["A"]]
    Q0 = np.array(g["Q0"], float)
    sc = g["scale_num"] / g["scale_den"]
    loc = oracle.dp_step(As, None, Q0, scale=sc, orient_t=True)
    glo = oracle.dp_step(As, None, Q0, scale=sc, orient_t=True, ef_global=True)
    np.testing.assert_allclose(loc["P_hat"], np.array(g["P_hat_num"]) / math.sqrt(g["P_hat_den_sqrt"]), atol=1e-15)
    np.testing.assert_allclose(loc["Q"], np.array(g["Q_num"]) / math.sqrt(g["Q_den_sqrt"]), atol=1e-15)
    np.testing.assert_allclose(loc["recon"], np.array(g["recon_num"]) / g["recon_den"], atol=1e-15)
    for w in range(2):
        np.testing.assert_allclose(loc["err"][w], np.array(g["err_local_num"][w]) / g["err_local_den"], atol=1e-15)
        np.testing.assert_allclose(glo["err"][w], np.array(g["err_global_num"][w]) / g["err_global_den"], atol=1e-15)
    want_sum = np.array(g["err_sum_num"]) / g["err_sum_den"]
    np.testing.assert_allclose(sum(loc["err"]), want_sum, atol=1e-15)
    np.testing.assert_allclose(sum(glo["err"]), want_sum, atol=1e-15)


def test_dp_orient_t_equals_dp_step_on_transposes():
    """orient_t is the DP step on A_w^T, returned in A's layout (reading C6)."""
    rng = np.random.default_rng(32)
    n, m, r, D = 40, 18, 4, 3
    Ms = [rng.standard_normal((n, m)) for _ in range(D)]
    Es = [0.1 * rng.standard_normal((n, m)) for _ in range(D)]
    Q0 = rng.standard_normal((n, r))
    for eg in (False, True):
        a = oracle.dp_step(Ms, Es, Q0, scale=1.0 / D, orient_t=True, ef_global=eg)
        b = oracle.dp_step([x.T for x in Ms], [x.T for x in Es], Q0, scale=1.0 / D, ef_global=eg)
        np.testing.assert_allclose(a["recon"], b["recon"].T, atol=1e-13)
        for w in range(D):
            np.testing.assert_allclose(a["err"][w], b["err"][w].T, atol=1e-13)
        np.testing.assert_allclose(a["Q"], b["Q"], atol=1e-13)
        assert a["P_hat"].shape == (m, r)


def test_embed_sync_hand_values():
    """Reading C12: sum over the 2D ranks of G/D = mean(first) + mean(last).
    Ones on 2D = 8 ranks with D = 4 give 2 (a 1/(2D) scale would give 1); a
    D = 2 example with distinct values: mean(1,3) + mean(5,7) = 2 + 6 = 8."""
    D = 4
    ones = [np.ones((2, 3))] * (2 * D)
    np.testing.assert_array_equal(oracle.embed_sync_fused(ones, D), 2 * np.ones((2, 3)))
    np.testing.assert_array_equal(oracle.embed_sync_sequential(ones[:D], ones[D:]), 2 * np.ones((2, 3)))
    vals = [np.full((1, 2), v) for v in (1.0, 3.0, 5.0, 7.0)]
    np.testing.assert_array_equal(oracle.embed_sync_fused(vals, 2), np.full((1, 2), 8.0))
    np.testing.assert_array_equal(oracle.embed_sync_sequential(vals[:2], vals[2:]), np.full((1, 2), 8.0))
