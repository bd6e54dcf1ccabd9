"""GPU parity (-m gpu): the CUDA path through the C-ABI vs the fp64 oracle on
the same seeded inputs.

Tolerances (north_star): relative Frobenius error of M' and e_new (against
||A||_F) <= 1e-4 for fp32, <= 1e-2 for bf16 inputs/outputs; factor
orthonormality ||P_hat^T P_hat - I||_F <= 1e-5.  P_hat and Q are also compared
column by column where the factor is unique (no fallback fired, kappa(P) small;
reading C4).
"""
import numpy as np
import pytest

import oracle
from workloads import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2301_09830_b200 import build as occ_build  # noqa: E402
from paper_2301_09830_b200 import occ  # noqa: E402

TOL32, TOLBF, TOLORTH = 1e-4, 1e-2, 1e-5


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    occ_build.build()
    occ.lib()


def to_dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(dtype)


def run_gpu(M, e, Q0, r, *, bf16=False, flags=0, recon=True):
    n, m = M.shape
    Md = to_dev(M, torch.bfloat16 if bf16 else torch.float32)
    Ed = to_dev(e) if e is not None else None
    Qd = to_dev(Q0)
    Pd = torch.empty(n, r, device="cuda")
    Rd = torch.empty_like(Md) if recon else None
    ws = occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, flags=flags)
    torch.cuda.synchronize()
    st = occ.occ_read_stats(ws)
    M_used = Md.double().cpu().numpy()   # bf16-rounded input as the GPU saw it
    return {"P_hat": Pd.double().cpu().numpy(), "Q": Qd.double().cpu().numpy(),
            "recon": Rd.double().cpu().numpy() if recon else None,
            "err": Ed.double().cpu().numpy() if Ed is not None else None, "stats": st, "M_used": M_used}


def rel(a, b, ref):
    return np.linalg.norm(a - b) / max(np.linalg.norm(ref), 1e-300)


def elem(a, b, ref):
    """max |a - b| over max |ref|: the element-wise bound next to the Frobenius
    one (one bad element or tile edge cannot hide in a 1e-4 Frobenius norm)."""
    return np.abs(a - b).max() / max(np.abs(ref).max(), 1e-300)


def check_step(g, o, A, *, tol, check_factors=True, etol=None):
    """Frobenius bound `tol` (north_star) and an element-wise bound relative to
    max |A| on M' and e_new: fp32 1e-5 (tol / 10); bf16 1e-2, since an fp32-
    vs-fp64 difference may flip one bf16 rounding of the largest element, one
    ulp = up to 2^-7 of it; orthonormality; factors column-wise."""
    if etol is None:
        etol = tol / 10 if tol <= TOL32 else tol
    r = g["P_hat"].shape[1]
    orth = np.linalg.norm(g["P_hat"].T @ g["P_hat"] - np.eye(r))
    assert orth <= TOLORTH, orth
    if g["recon"] is not None:
        assert rel(g["recon"], o["recon"], A) <= tol
        assert elem(g["recon"], o["recon"], A) <= etol
    if g["err"] is not None:
        assert rel(g["err"], o["err"], A) <= tol
        assert elem(g["err"], o["err"], A) <= etol
    if check_factors and not o["fallbacks"]:
        assert rel(g["P_hat"], o["P_hat"], o["P_hat"]) <= 100 * tol
        assert rel(g["Q"], o["Q"], o["Q"]) <= tol * 10


SHAPES = [
    (128, 256, 4, "D1"),      # C1 (BASELINE configs[0])
    (128, 256, 4, "D2"),
    (200, 136, 8, "D2"),      # ragged tails in every tiling
    (1000, 392, 16, "D2"),
    (1024, 3072, 16, "D2"),   # north-star target T
    (777, 1208, 32, "D2"),
    (640, 1024, 64, "D2"),
]


@pytest.mark.parametrize("n,m,r,dist", SHAPES)
def test_compress_matches_oracle_fp32(n, m, r, dist):
    M = synth.make(dist, n, m, 1000 + n + r)
    e = synth.e0(n, m, 1001 + n, like=M)
    Q0 = synth.q0(m, r, 7)
    g = run_gpu(M, e, Q0, r)
    o = oracle.compress_step(M, e, Q0)
    A = M.astype(np.float64) + e
    check_step(g, o, A, tol=TOL32)
    assert g["stats"]["fallback_columns"] == len(o["fallbacks"])


@pytest.mark.parametrize("n,m,r", [(256, 512, 16), (1024, 3072, 16), (1000, 392, 8)])
def test_compress_bf16(n, m, r):
    M = synth.d2_gradlike(n, m, 31)
    e = synth.e0(n, m, 32, like=M)
    Q0 = synth.q0(m, r, 33)
    g = run_gpu(M, e, Q0, r, bf16=True)
    o = oracle.compress_step(g["M_used"], e, Q0, out_dtype="bf16")
    A = g["M_used"] + e
    check_step(g, o, A, tol=TOLBF, check_factors=False)
    # EF identity on the GPU: M'_bf16 + e_new == A up to fp32 rounding (reading C7)
    assert rel(g["recon"] + g["err"], A, A) <= 1e-6


def test_no_ef_and_null_err():
    n, m, r = 256, 512, 8
    M = synth.d2_gradlike(n, m, 41)
    Q0 = synth.q0(m, r, 42)
    g = run_gpu(M, None, Q0, r, flags=occ.OCC_NO_EF)
    o = oracle.compress_step(M, None, Q0, no_ef=True)
    check_step(g, o, M.astype(np.float64), tol=TOL32)


def test_paths_deterministic_and_consistent(monkeypatch):
    n, m, r = 1000, 1208, 16
    M = synth.d2_gradlike(n, m, 51)
    e = synth.e0(n, m, 52, like=M)
    Q0 = synth.q0(m, r, 53)
    a = run_gpu(M, e, Q0, r)                                   # default: TMEM-resident fused kernel
    c = run_gpu(M, e, Q0, r)
    assert a["stats"]["path"] == 3
    for k in ("P_hat", "Q", "recon", "err"):
        assert np.array_equal(a[k], c[k]), k                   # bitwise deterministic
    monkeypatch.setenv("OCC_PATH", "v1")
    b1 = run_gpu(M, e, Q0, r)                                  # v1 persistent kernel
    b2 = run_gpu(M, e, Q0, r, flags=occ.OCC_FORCE_MULTI)        # v1, one launch per phase
    assert b1["stats"]["path"] == 1 and b2["stats"]["path"] == 2
    for k in ("P_hat", "Q", "recon", "err"):
        assert np.array_equal(b1[k], b2[k]), k
    A = M.astype(np.float64) + e
    assert rel(a["recon"], b1["recon"], A) <= 1e-5
    assert rel(a["err"], b1["err"], A) <= 1e-5


@pytest.mark.parametrize("debug,fused", [(0, 1), (4, 0)])
def test_v2_control_flows(monkeypatch, debug, fused):
    """The fused kernel's phase-3 decision (reading C20), both branches against
    the oracle: the fused Q = (A^T P) Li^T (0), and the general path taken
    before phase 5 when the amp gate rejects it (4: amp gate -1)."""
    n, m, r = 1000, 1208, 16
    M = synth.d2_gradlike(n, m, 61)
    e = synth.e0(n, m, 62, like=M)
    Q0 = synth.q0(m, r, 63)
    monkeypatch.setenv("OCC_V2_DEBUG", str(debug))
    g = run_gpu(M, e, Q0, r)
    assert g["stats"]["path"] == 3
    assert g["stats"]["q_fused"] == fused
    assert 0 < g["stats"]["q_amp"] < 32
    o = oracle.compress_step(M, e, Q0)
    check_step(g, o, M.astype(np.float64) + e, tol=TOL32)


def test_amp_gate_rejects_collinear_factor():
    """Nearly collinear Q_prev columns make P nearly collinear: the fused
    Q = (A^T P) Li^T would amplify rounding by amp >> 32, so the kernel must
    recompute Q = A^T P_hat (q_fused = 0) and still match the oracle."""
    n, m, r = 1000, 1208, 16
    M = synth.d2_gradlike(n, m, 71)
    e = synth.e0(n, m, 72, like=M)
    base = synth.q0(m, 1, 73)
    Q0 = (base + 1e-3 * synth.q0(m, r, 74)).astype(np.float32)
    g = run_gpu(M, e, Q0, r)
    assert g["stats"]["q_fused"] == 0 and g["stats"]["q_amp"] > 32
    o = oracle.compress_step(M, e, Q0)
    # P is ill conditioned by construction (kappa ~ 1e3-1e4): rounding of the
    # fp32 factors is amplified by kappa, so the element-wise bound is the
    # Frobenius one (1e-4 of max |A|) here
    check_step(g, o, M.astype(np.float64) + e, tol=TOL32, check_factors=False, etol=TOL32)


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("multi", [False, True])
def test_orient_t_matches_oracle(bf16, multi):
    """OCC_ORIENT_T (reading C6): the step on A^T in A's stored layout; P is
    m x r (orthonormal, column side), Q is n x r (row side, warm start)."""
    n, m, r = 1000, 264, 16
    M = synth.d2_gradlike(n, m, 81)
    e = synth.e0(n, m, 82, like=M)
    Q0 = synth.q0(n, r, 83)
    flags = occ.OCC_ORIENT_T | (occ.OCC_FORCE_MULTI if multi else 0)
    Md = to_dev(M, torch.bfloat16 if bf16 else torch.float32)
    Ed, Qd = to_dev(e), to_dev(Q0)
    Pd = torch.empty(m, r, device="cuda")
    Rd = torch.empty_like(Md)
    ws = occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, flags=flags)
    torch.cuda.synchronize()
    assert occ.occ_read_stats(ws)["path"] == (2 if multi else 1)
    M_used = Md.double().cpu().numpy()
    o = oracle.compress_step(M_used, e, Q0, orient_t=True, out_dtype="bf16" if bf16 else "f64")
    g = {"P_hat": Pd.double().cpu().numpy(), "Q": Qd.double().cpu().numpy(), "recon": Rd.double().cpu().numpy(),
         "err": Ed.double().cpu().numpy()}
    check_step(g, o, M_used + e, tol=TOLBF if bf16 else TOL32)
    out = torch.empty_like(Md)
    occ.occ_decompress(Qd, Pd, out)   # M' = Q P^T in A's layout; bit-identical to the sender's (C8)
    torch.cuda.synchronize()
    assert torch.equal(out, Rd)


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("n,m,r,flags,path", [
    (1000, 1208, 16, 0, 3),                      # fused kernel
    (1000, 1208, 16, "FORCE_MULTI", 2),          # per-phase, multi-CTA Gram
    (8192, 3072, 32, 0, 1),                      # per-phase: the fused kernel's tile plan does not fit
    (640, 1024, 64, 0, 1),                       # r = 64 (v1 on both sides)
])
def test_decompress_bit_identical_to_sender_reconstruction(bf16, n, m, r, flags, path):
    """Reading C8: occ_decompress(P_hat, Q) on the receiver reproduces, bit for
    bit, the M' the sender's e_new was taken against, whichever path compressed."""
    M = synth.d2_gradlike(n, m, 91)
    e = synth.e0(n, m, 92, like=M)
    Q0 = synth.q0(m, r, 93)
    g = run_gpu(M, e, Q0, r, bf16=bf16, flags=getattr(occ, "OCC_" + flags) if flags else 0)
    assert g["stats"]["path"] == path
    Pd, Qd = to_dev(g["P_hat"]), to_dev(g["Q"])
    out = torch.empty(n, m, device="cuda", dtype=torch.bfloat16 if bf16 else torch.float32)
    occ.occ_decompress(Pd, Qd, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.double().cpu().numpy(), g["recon"])
    # and e_new was taken against that M' (fp32 rounding of A - M')
    A32 = (g["M_used"].astype(np.float32) + e.astype(np.float32)).astype(np.float64)
    assert np.abs(g["err"] + g["recon"] - A32).max() <= 1e-6 * np.abs(A32).max()


# BASELINE.json configs at full size, in the launch configuration bench.py times
# (the fused kernel for r <= 32, the per-phase path for r = 64), elementwise
# against the oracle (reading C6 matricisation; D2 gradient-like inputs).
FULL = [
    (4096, 1920, 16, 3),    # configs[1]: GPT-2.5B inter-stage, mb 4 (the bench line); fused kernel
    (8192, 3072, 32, 1),    # configs[2] shape: GPT-8.3B inter-stage, mb 8; v1 fused kernel (the v2 tile plan does not fit)
    (3072, 12288, 64, 1),   # configs[3] MLP weight gradient, r = 64: per-phase kernels
]


@pytest.mark.slow
@pytest.mark.parametrize("n,m,r,path", FULL)
def test_full_size_configs_match_oracle(n, m, r, path):
    M = synth.d2_gradlike(n, m, 1000 + n)
    e = synth.e0(n, m, 1001 + n, like=M)
    Q0 = synth.q0(m, r, 1002)
    g = run_gpu(M, e, Q0, r)
    assert g["stats"]["path"] == path
    o = oracle.compress_step(M, e, Q0)
    check_step(g, o, M.astype(np.float64) + e, tol=TOL32, check_factors=False)


@pytest.mark.parametrize("v1", [False, True])
def test_check_finite_reports_nonfinite_input(monkeypatch, v1):
    """OCC_CHECK_FINITE: a NaN in M (or err) sets the device status word that
    occ_check_status reports (and clears); clean input and calls without the
    flag report nothing."""
    if v1:
        monkeypatch.setenv("OCC_PATH", "v1")
    n, m, r = 300, 264, 8
    M = synth.d2_gradlike(n, m, 95)
    e = synth.e0(n, m, 96, like=M)
    Q0 = synth.q0(m, r, 97)
    occ.occ_check_status()                                    # clear anything pending
    run_gpu(M, e, Q0, r, flags=occ.OCC_CHECK_FINITE)
    occ.occ_check_status()                                    # clean: no error
    Mn = M.copy()
    Mn[17, 23] = np.nan
    run_gpu(Mn, e, Q0, r)                                     # no flag: nothing recorded
    occ.occ_check_status()
    g = run_gpu(Mn, e, Q0, r, flags=occ.OCC_CHECK_FINITE)
    assert g["stats"]["path"] == (1 if v1 else 3)
    with pytest.raises(occ.OccError) as exc:
        occ.occ_check_status()
    assert exc.value.name == "OCC_ERR_NONFINITE"
    occ.occ_check_status()                                    # cleared by the report


@pytest.mark.parametrize("mode", ["v2", "v1", "orient_t"])
def test_wire_bf16(monkeypatch, mode):
    """OCC_WIRE_BF16 (reading C7): P_hat and Q are bf16 values, the reconstruction
    and e_new use them (vs the oracle with wire_bf16), and the receiver's
    decompression of the bf16 factors is bit-identical to the sender's M' (C8)."""
    n, m, r = 1000, 1208, 16
    if mode == "v1":
        monkeypatch.setenv("OCC_PATH", "v1")
    ot = mode == "orient_t"
    M = synth.d2_gradlike(n, m, 101)
    e = synth.e0(n, m, 102, like=M)
    Q0 = synth.q0(n if ot else m, r, 103)
    flags = occ.OCC_WIRE_BF16 | (occ.OCC_ORIENT_T if ot else 0)
    Md, Ed, Qd = to_dev(M), to_dev(e), to_dev(Q0)
    Pd = torch.empty(m if ot else n, r, device="cuda")
    Rd = torch.empty_like(Md)
    ws = occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, flags=flags)
    torch.cuda.synchronize()
    assert occ.occ_read_stats(ws)["path"] == {"v2": 3, "v1": 1, "orient_t": 1}[mode]
    for t in (Pd, Qd):
        assert torch.equal(t, t.to(torch.bfloat16).float())
    o = oracle.compress_step(M, e, Q0, wire_bf16=True, orient_t=ot)
    A = M.astype(np.float64) + e
    g = {"P_hat": Pd.double().cpu().numpy(), "Q": Qd.double().cpu().numpy(), "recon": Rd.double().cpu().numpy(),
         "err": Ed.double().cpu().numpy()}
    # fp32-vs-fp64 factor differences can flip a bf16 rounding in a few
    # elements (one bf16 ulp, 2^-8 relative): 1e-3 bounds that with margin.
    assert rel(g["recon"], o["recon"], A) <= 1e-3
    assert rel(g["err"], o["err"], A) <= 1e-3
    assert rel(g["P_hat"], o["P_hat"], o["P_hat"]) <= TOLBF
    assert rel(g["Q"], o["Q"], o["Q"]) <= TOLBF
    assert np.linalg.norm(g["P_hat"].T @ g["P_hat"] - np.eye(r)) <= 1e-2   # orthonormal up to bf16 rounding
    assert np.array_equal(g["recon"] + g["err"], A.astype(np.float32).astype(np.float64)) or \
        np.abs(g["recon"] + g["err"] - A).max() <= 1e-5 * np.abs(A).max()
    out = torch.empty_like(Md)
    if ot:
        occ.occ_decompress(Qd, Pd, out)
    else:
        occ.occ_decompress(Pd, Qd, out)
    torch.cuda.synchronize()
    assert torch.equal(out, Rd)


def test_zero_input_all_fallbacks():
    n, m, r = 300, 264, 8
    M = np.zeros((n, m), np.float32)
    g = run_gpu(M, np.zeros((n, m), np.float32), synth.q0(m, r, 3), r)
    assert np.all(g["recon"] == 0) and np.all(g["err"] == 0)
    assert g["stats"]["fallback_columns"] == r
    o = oracle.compress_step(M, None, synth.q0(m, r, 3))
    assert np.linalg.norm(g["P_hat"].T @ g["P_hat"] - np.eye(r)) <= TOLORTH
    # same fallback vectors, same order -> same P_hat (counter-based generator on both sides)
    np.testing.assert_allclose(g["P_hat"], o["P_hat"], atol=1e-6)


@pytest.mark.parametrize("k,r", [(2, 8), (5, 16), (16, 16)])
def test_exact_low_rank_recovered(k, r):
    n, m = 512, 640
    M = synth.d4_exact_lowrank(n, m, k, seed=61)
    g = run_gpu(M, None, synth.q0(m, r, 62), r, flags=occ.OCC_NO_EF)
    assert np.linalg.norm(g["recon"] - M) <= 1e-5 * np.linalg.norm(M)
    assert g["stats"]["fallback_columns"] == r - k
    assert np.linalg.norm(g["P_hat"].T @ g["P_hat"] - np.eye(r)) <= TOLORTH


def test_forced_second_pass():
    n, m, r = 1024, 1024, 16
    M = synth.d2_gradlike(n, m, 71)
    Q0 = synth.q0(m, r, 72)
    g = run_gpu(M, None, Q0, r, flags=occ.OCC_NO_EF | occ.OCC_FORCE_TWO_PASS)
    assert g["stats"]["second_pass"] == 1
    o = oracle.compress_step(M, None, Q0, no_ef=True)
    check_step(g, o, M.astype(np.float64), tol=TOL32)


def test_lep_stream_free_running_16_steps():
    n, m, r, T = 512, 768, 16, 16
    Ms = synth.d3_lep_stream(n, m, 81, T)
    Q0 = synth.q0(m, r, 82)
    Md = torch.empty(n, m, device="cuda")
    Ed = torch.zeros(n, m, device="cuda")
    Qd = to_dev(Q0)
    Pd = torch.empty(n, r, device="cuda")
    Rd = torch.empty(n, m, device="cuda")
    ws = occ.alloc_workspace(n, m, r)
    e_o = np.zeros((n, m))
    Q_o = Q0.astype(np.float64)
    tot_g = np.zeros((n, m))
    for t, Mt in enumerate(Ms):
        Md.copy_(to_dev(Mt))
        occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, ws=ws)
        A = Mt.astype(np.float64) + e_o
        o = oracle.compress_step(Mt, e_o, Q_o)
        e_o, Q_o = o["err"], o["Q"]
        rg = Rd.double().cpu().numpy()
        tot_g += rg
        assert rel(rg, o["recon"], A) <= TOL32, t
    # telescoping on the GPU's own numbers: sum M'_t = sum M_t + e_0 - e_T (P9)
    expect = sum(x.astype(np.float64) for x in Ms) - Ed.double().cpu().numpy()
    assert rel(tot_g, expect, expect) <= 1e-5


def test_per_phase_warm_start_high_kappa():
    """The per-phase path (r = 64) warm started over a D3 stream: the unnormalised
    warm start drives kappa_est(P) past 1e4, where the per-phase path keeps a
    single CholQR pass (reading C3: fp64 Gram, kappa^2 u_64 << the
    fp32 rounding); every step against the oracle, orthonormality included."""
    n, m, r, T = 2048, 1536, 64, 4
    Ms = synth.d3_lep_stream(n, m, 83, T)
    Q0 = synth.q0(m, r, 84)
    Md = torch.empty(n, m, device="cuda")
    Ed = torch.zeros(n, m, device="cuda")
    Qd = to_dev(Q0)
    Pd = torch.empty(n, r, device="cuda")
    Rd = torch.empty(n, m, device="cuda")
    ws = occ.alloc_workspace(n, m, r)
    e_o = np.zeros((n, m))
    Q_o = Q0.astype(np.float64)
    kappas = []
    for t, Mt in enumerate(Ms):
        Md.copy_(to_dev(Mt))
        occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, ws=ws)
        torch.cuda.synchronize()
        st = occ.occ_read_stats(ws)
        kappas.append(st["kappa_est"])
        assert st["path"] != 3 and st["second_pass"] == (1 if st["kappa_est"] > 1e6 else 0), st
        A = Mt.astype(np.float64) + e_o
        o = oracle.compress_step(Mt, e_o, Q_o)
        g = {"P_hat": Pd.double().cpu().numpy(), "Q": Qd.double().cpu().numpy(),
             "recon": Rd.double().cpu().numpy(), "err": Ed.double().cpu().numpy()}
        # kappa(P) ~ 1e4: the fp32 rounding of P and Q is amplified as in the
        # ill-conditioned case above, so the element-wise bound is 1e-4 there
        # too (measured 1.75e-5 at step 1 WITH and without the CholQR2 pass:
        # profiles/round2_kappa_ab.jsonl); Frobenius and orthonormality as usual
        check_step(g, o, A, tol=TOL32, check_factors=False, etol=1e-4)
        e_o, Q_o = o["err"], o["Q"]
    assert max(kappas) > 1e4, kappas


def test_decompress_matches_oracle():
    n, m, r = 700, 1032, 16
    rng = np.random.default_rng(91)
    P = rng.standard_normal((n, r)).astype(np.float32)
    Q = rng.standard_normal((m, r)).astype(np.float32)
    for dt, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-2)):
        out = torch.empty(n, m, device="cuda", dtype=dt)
        occ.occ_decompress(to_dev(P), to_dev(Q), out)
        torch.cuda.synchronize()
        o = oracle.decompress(P, Q, out_dtype="f32" if dt == torch.float32 else "bf16")
        assert rel(out.double().cpu().numpy(), o, o) <= tol


def test_dp_single_rank_matches_oracle():
    # occ_allreduce_factors with no communicator = a DP group of one rank
    n, m, r = 512, 1024, 16
    M = synth.d2_gradlike(n, m, 101)
    e = synth.e0(n, m, 102, like=M)
    Q0 = synth.q0(m, r, 103)
    Gd, Ed, Qd = to_dev(M), to_dev(e), to_dev(Q0)
    Pd = torch.empty(n, r, device="cuda")
    occ.occ_allreduce_factors([Gd], [Ed], [Qd], [Pd], r, 1.0)
    torch.cuda.synchronize()
    o = oracle.dp_step([M], [e], Q0, scale=1.0)
    A = M.astype(np.float64) + e
    assert rel(Gd.double().cpu().numpy(), o["recon"], A) <= TOL32
    assert rel(Ed.double().cpu().numpy(), o["err"][0], A) <= TOL32
    assert rel(Qd.double().cpu().numpy(), o["Q"], o["Q"]) <= 1e-3


def test_init_q_is_standard_normal_and_seeded():
    Q = torch.empty(4096, 16, device="cuda")
    occ.occ_init_q(Q, 1234)
    Q2 = torch.empty_like(Q)
    occ.occ_init_q(Q2, 1234)
    torch.cuda.synchronize()
    assert torch.equal(Q, Q2)
    x = Q.double().cpu().numpy()
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1) < 0.02


@pytest.mark.parametrize("n,m,r,flags,path", [
    (1000, 1208, 16, 0, 3),                   # fused kernel
    (1000, 1208, 16, "FORCE_MULTI", 2),       # per-phase + decompress-with-EF kernel
    (640, 1024, 64, 0, 1),                    # r = 64 per-phase
    (1000, 264, 16, "ORIENT_T", 1),           # OCC_ORIENT_T
])
def test_inplace_compress_equals_out_of_place(n, m, r, flags, path):
    """recon may be M itself (check_step allows it): the in-place call must give
    the same M' and e_new, bit for bit, as the out-of-place one (ADVICE r1:
    the reconstruct kernel loads A = M + e before it stores M')."""
    fl = getattr(occ, "OCC_" + flags) if flags else 0
    ot = flags == "ORIENT_T"
    M = synth.d2_gradlike(n, m, 111)
    e = synth.e0(n, m, 112, like=M)
    Q0 = synth.q0(n if ot else m, r, 113)
    outs = []
    for inplace in (False, True):
        Md, Ed, Qd = to_dev(M), to_dev(e), to_dev(Q0)
        Pd = torch.empty(m if ot else n, r, device="cuda")
        Rd = Md if inplace else torch.empty_like(Md)
        ws = occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, flags=fl)
        torch.cuda.synchronize()
        assert occ.occ_read_stats(ws)["path"] == path
        outs.append((Rd.clone(), Ed.clone(), Qd.clone(), Pd.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    o = oracle.compress_step(M, e, Q0, orient_t=ot)
    A = M.astype(np.float64) + e
    assert rel(outs[1][0].double().cpu().numpy(), o["recon"], A) <= TOL32
    assert rel(outs[1][1].double().cpu().numpy(), o["err"], A) <= TOL32


def test_single_rank_nccl_allreduce_factors():
    """occ_allreduce_factors on a real 1-rank NCCL communicator: both
    ncclAllReduce calls (P, then Q: reading C1) run; the result matches the
    oracle's dp_step and, bit for bit, the no-communicator call."""
    n, m, r = 512, 1024, 16
    M = synth.d2_gradlike(n, m, 121)
    e = synth.e0(n, m, 122, like=M)
    Q0 = synth.q0(m, r, 123)
    comm = occ.Comm.single()
    try:
        res = []
        for cm in (comm, None):
            Gd, Ed, Qd = to_dev(M), to_dev(e), to_dev(Q0)
            Pd = torch.empty(n, r, device="cuda")
            occ.occ_allreduce_factors([Gd], [Ed], [Qd], [Pd], r, 1.0, comm=cm)
            occ.occ_check_status(comm=cm)
            res.append((Gd, Ed, Qd, Pd))
        for a, b in zip(*res):
            assert torch.equal(a, b)
        o = oracle.dp_step([M], [e], Q0, scale=1.0)
        A = M.astype(np.float64) + e
        G = res[0][0].double().cpu().numpy()
        assert rel(G, o["recon"], A) <= TOL32 and elem(G, o["recon"], A) <= TOL32 / 10
        assert rel(res[0][1].double().cpu().numpy(), o["err"][0], A) <= TOL32
    finally:
        comm.destroy()


@pytest.mark.parametrize("r,flags", [(64, 0), (32, "EF_GLOBAL"), (64, "ORIENT_T")])
def test_dplink_single_rank_matches_oracle(r, flags):
    """occ_allreduce_factors_link on a 1-rank group: the in-kernel exchange runs
    (push into the own mailbox, flag, sum, acknowledge; 5 calls so both slots
    are reused), the result matches the oracle's dp_step and, bit for bit, the
    NCCL call on the same communicator."""
    fl = {0: 0, "EF_GLOBAL": occ.OCC_EF_GLOBAL, "ORIENT_T": occ.OCC_ORIENT_T}[flags]
    shapes = [(640, 1024), (512, 776)]
    Ms = [synth.d2_gradlike(n, m, 141 + j) for j, (n, m) in enumerate(shapes)]
    es = [synth.e0(n, m, 151 + j, like=Ms[j]) for j, (n, m) in enumerate(shapes)]
    ot = fl & occ.OCC_ORIENT_T
    Q0s = [synth.q0(n if ot else m, r, 161 + j) for j, (n, m) in enumerate(shapes)]
    comm = occ.Comm.single()
    link = occ.DpLink.open(comm, max(sum(max(n, m) for n, m in shapes) * r, 1))
    try:
        res = {}
        for mode in ("link", "nccl"):
            G = [to_dev(x) for x in Ms]
            E = [to_dev(x) for x in es]
            Q = [to_dev(x) for x in Q0s]
            P = [torch.empty(m if ot else n, r, device="cuda") for n, m in shapes]
            for it in range(5):
                if it:   # fresh gradients each call, warm start and error carried
                    for j in range(len(shapes)):
                        G[j].copy_(to_dev(Ms[j]))
                if mode == "link":
                    occ.occ_allreduce_factors_link(G, E, Q, P, r, 1.0, link, flags=fl)
                else:
                    occ.occ_allreduce_factors(G, E, Q, P, r, 1.0, flags=fl, comm=comm)
                occ.occ_check_status(comm=comm)
                if it == 0:
                    res[mode + "0"] = [x.clone() for x in G] + [x.clone() for x in E]
            res[mode] = G + E + Q + P
        for a, b in zip(res["link"], res["nccl"]):
            assert torch.equal(a, b)
        for j in range(len(shapes)):   # each matrix of the bucket: a 1-rank dp_step
            o = oracle.dp_step([Ms[j]], [es[j]], Q0s[j], scale=1.0, ef_global=bool(fl & occ.OCC_EF_GLOBAL),
                               orient_t=bool(ot))
            A = Ms[j].astype(np.float64) + es[j]
            Gj = res["link0"][j].double().cpu().numpy()
            Ej = res["link0"][len(shapes) + j].double().cpu().numpy()
            assert rel(Gj, o["recon"], A) <= TOL32 and elem(Gj, o["recon"], A) <= TOL32 / 10
            assert rel(Ej, o["err"][0], A) <= TOL32
    finally:
        link.close()
        comm.destroy()


@pytest.mark.parametrize("wire", [False, True])
def test_single_rank_nccl_sendrecv_self(wire):
    """occ_sendrecv_factors on a 1-rank communicator, the stage its own peer:
    the NCCL send and recv of (P_hat, Q) run in one group; the received
    factors equal the sent ones and the decompressed M' equals the sender's
    own M' bit for bit (reading C8) and the oracle (C7 with OCC_WIRE_BF16)."""
    n, m, r = 1024, 3072, 16
    M = synth.d2_gradlike(n, m, 131)
    e = synth.e0(n, m, 132, like=M)
    Q0 = synth.q0(m, r, 133)
    flags = occ.OCC_WIRE_BF16 if wire else 0
    comm = occ.Comm.single()
    try:
        Md, Ed, Qd = to_dev(M), to_dev(e), to_dev(Q0)
        Pd = torch.empty(n, r, device="cuda")
        out = torch.empty(n, m, device="cuda")
        Pr, Qr = torch.empty(n, r, device="cuda"), torch.empty(m, r, device="cuda")
        occ.occ_sendrecv_factors(Md, Ed, Qd, Pd, r, 0, out, Pr, Qr, 0, comm, flags=flags)
        occ.occ_check_status(comm=comm)
        assert torch.equal(Pr, Pd) and torch.equal(Qr, Qd)
        own = torch.empty_like(out)
        occ.occ_decompress(Pd, Qd, own)
        torch.cuda.synchronize()
        assert torch.equal(out, own)
        o = oracle.compress_step(M, e, Q0, wire_bf16=wire)
        A = M.astype(np.float64) + e
        tol = 1e-3 if wire else TOL32
        assert rel(out.double().cpu().numpy(), o["recon"], A) <= tol
        # the sender's e_new + the receiver's M' = A (the EF identity across the link)
        assert rel(out.double().cpu().numpy() + Ed.double().cpu().numpy(), A, A) <= 1e-6
    finally:
        comm.destroy()


def test_single_rank_embed_sync_dense():
    """occ_embed_sync r = 0 on a 1-rank communicator: one PreMulSum allreduce,
    G <- scale * G (reading C12 with D = 1/scale); called twice with two
    scales so the cached PreMulSum op is re-created."""
    comm = occ.Comm.single()
    try:
        G0 = synth.d2_gradlike(256, 512, 141)
        for sc in (0.5, 0.25):
            G = to_dev(G0)
            occ.occ_embed_sync(G, None, None, None, 0, sc, comm)
            occ.occ_check_status(comm=comm)
            assert torch.equal(G, to_dev(G0) * sc)
    finally:
        comm.destroy()


def test_single_rank_exchange_only():
    """occ_sendrecv_factors with M = NULL and out = NULL: the library's factor
    exchange alone (what bench.py times as factor comm), here to self on a
    1-rank communicator; the received factors equal the sent ones bit for bit."""
    n, m, r = 1024, 3072, 16
    comm = occ.Comm.single()
    try:
        P = to_dev(synth.q0(n, r, 151))
        Q = to_dev(synth.q0(m, r, 152))
        Pr, Qr = torch.empty_like(P), torch.empty_like(Q)
        occ.occ_sendrecv_factors(None, None, Q, P, r, 0, None, Pr, Qr, 0, comm)
        occ.occ_check_status(comm=comm)
        assert torch.equal(Pr, P) and torch.equal(Qr, Q)
    finally:
        comm.destroy()


@pytest.mark.parametrize("n,m,r,flags", [
    (1024, 3072, 16, 0),              # fused kernel: its producer warp pushes during phase 5
    (1024, 3072, 16, "WIRE_BF16"),    # bf16-exact factors through the link
    (640, 1024, 64, 0),               # per-phase path: the push kernel
    (1000, 264, 16, "ORIENT_T"),      # P m x r, Q n x r; out = Q P^T
])
def test_link_self_ring_matches_oracle(n, m, r, flags):
    """occ_sendrecv_factors_link on a ring of one (the stage is its own
    neighbour): the factors travel through the NVLink mailbox protocol (flag,
    two slots, ack) with no NCCL call; over 5 steps (the slots are reused after
    their acks) the received factors equal the sent ones bit for bit, the
    decompressed M' equals the sender's own M' bit for bit (reading C8), and
    each step matches the oracle's LEP stream."""
    fl = getattr(occ, "OCC_" + flags) if flags else 0
    ot = flags == "ORIENT_T"
    comm = occ.Comm.single()
    link = occ.Link.open(comm, 0, 0, max(n, m), max(n, m), r)
    try:
        Ms = synth.d3_lep_stream(n, m, 161, 5)
        e_o = synth.e0(n, m, 162, like=Ms[0]).astype(np.float64)
        Q_o = synth.q0(n if ot else m, r, 163).astype(np.float64)
        Ed, Qd = to_dev(e_o), to_dev(Q_o)
        Pd = torch.empty(m if ot else n, r, device="cuda")
        Pr, Qr = torch.empty_like(Pd), torch.empty_like(Qd)
        out = torch.empty(n, m, device="cuda")
        ws = occ.alloc_workspace(n, m, r)
        for t, Mt in enumerate(Ms):
            Md = to_dev(Mt)
            occ.occ_sendrecv_factors_link(Md, Ed, Qd, Pd, r, out, Pr, Qr, link, flags=fl, ws=ws)
            occ.occ_check_status(comm=comm)
            assert torch.equal(Pr, Pd) and torch.equal(Qr, Qd), t
            own = torch.empty_like(out)
            if ot:
                occ.occ_decompress(Qd, Pd, own)
            else:
                occ.occ_decompress(Pd, Qd, own)
            torch.cuda.synchronize()
            assert torch.equal(out, own), t
            o = oracle.compress_step(Mt, e_o, Q_o, orient_t=ot, wire_bf16=flags == "WIRE_BF16")
            A = Mt.astype(np.float64) + e_o
            tol = 1e-3 if flags == "WIRE_BF16" else TOL32
            assert rel(out.double().cpu().numpy(), o["recon"], A) <= tol, t
            e_o, Q_o = o["err"], o["Q"]
        # exchange only: push P, Q as they are; receive without decompressing
        P2, Q2 = torch.randn_like(Pd), torch.randn_like(Qd)
        occ.occ_sendrecv_factors_link(None, None, Q2, P2, r, None, Pr, Qr, link)
        occ.occ_check_status(comm=comm)
        assert torch.equal(Pr, P2) and torch.equal(Qr, Q2)
    finally:
        link.close()
        comm.destroy()


@pytest.mark.parametrize("flags", ["", "EF_GLOBAL"])
@pytest.mark.parametrize("r", [16, 64])
def test_dp_orient_t_single_rank_matches_oracle(flags, r):
    """occ_allreduce_factors with OCC_ORIENT_T on a 1-rank communicator (the
    embedding's G^T form, reading C6): the tensor-core DP reconstruction with the
    row-side factors (scale V_sum for M', V_w for the local error) against the
    oracle's dp_step(orient_t=True); the row-side warm start goes to Q."""
    n, m = 1536, 512
    fl = occ.OCC_ORIENT_T | (occ.OCC_EF_GLOBAL if flags else 0)
    M = synth.d2_gradlike(n, m, 171)
    e = synth.e0(n, m, 172, like=M)
    Q0 = synth.q0(n, r, 173)
    comm = occ.Comm.single()
    try:
        Gd, Ed, Qd = to_dev(M), to_dev(e), to_dev(Q0)
        Pd = torch.empty(m, r, device="cuda")
        occ.occ_allreduce_factors([Gd], [Ed], [Qd], [Pd], r, 1.0, flags=fl, comm=comm)
        occ.occ_check_status(comm=comm)
        o = oracle.dp_step([M], [e], Q0, scale=1.0, orient_t=True, ef_global=bool(flags))
        A = M.astype(np.float64) + e
        G = Gd.double().cpu().numpy()
        assert rel(G, o["recon"], A) <= TOL32 and elem(G, o["recon"], A) <= TOL32 / 10
        assert rel(Ed.double().cpu().numpy(), o["err"][0], A) <= TOL32
        assert rel(Qd.double().cpu().numpy(), o["Q"], o["Q"]) <= 1e-3
    finally:
        comm.destroy()


def test_dp_mixed_shape_bucket_matches_oracle():
    """A DP bucket of matrices with different shapes (each matrix's
    sweep-1 partials need s1_i n_i rows, which can exceed those of the largest
    shape): the advisor's (3581, 304) + (4861, 184) at r = 64, and the C4
    shapes' aspect, each against the oracle's dp_step (1-rank group)."""
    r = 64
    shapes = [(3576, 304), (4856, 184), (512, 2048)]   # rows x cols (cols % 8 == 0)
    Ms = [synth.d2_gradlike(a, b, 181 + i) for i, (a, b) in enumerate(shapes)]
    Es = [synth.e0(a, b, 191 + i, like=Ms[i]) for i, (a, b) in enumerate(shapes)]
    Q0s = [synth.q0(b, r, 201 + i) for i, (_, b) in enumerate(shapes)]
    Gd = [to_dev(x) for x in Ms]
    Ed = [to_dev(x) for x in Es]
    Qd = [to_dev(x) for x in Q0s]
    Pd = [torch.empty(a, r, device="cuda") for a, _ in shapes]
    occ.occ_allreduce_factors(Gd, Ed, Qd, Pd, r, 1.0)
    torch.cuda.synchronize()
    for i in range(len(shapes)):
        o = oracle.dp_step([Ms[i]], [Es[i]], Q0s[i], scale=1.0)
        A = Ms[i].astype(np.float64) + Es[i]
        G = Gd[i].double().cpu().numpy()
        assert rel(G, o["recon"], A) <= TOL32 and elem(G, o["recon"], A) <= TOL32 / 10, i
        assert rel(Ed[i].double().cpu().numpy(), o["err"][0], A) <= TOL32, i


@pytest.mark.parametrize("n,m,r", [(1024, 3072, 16), (1000, 776, 64)])
def test_graph_replay_matches_eager(n, m, r):
    """bench.py times N = 1 steps as CUDA-graph replays of the same API calls:
    a replayed step (fused kernel, r16; per-phase tcgen05 path, r64) is bit-identical
    to the eagerly issued one, and both match the oracle."""
    M = synth.d2_gradlike(n, m, 171)
    e = synth.e0(n, m, 172, like=M)
    Q0 = synth.q0(m, r, 173)
    Md = to_dev(M)
    ws = occ.alloc_workspace(n, m, r)
    outs = {}
    for mode in ("eager", "graph"):
        Ed, Qd = to_dev(e), to_dev(Q0)
        Pd = torch.empty(n, r, device="cuda")
        Rd = torch.empty_like(Md)
        if mode == "eager":
            occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, ws=ws)
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, ws=ws)
            Ed.copy_(to_dev(e))
            Qd.copy_(to_dev(Q0))
            g.replay()
        torch.cuda.synchronize()
        outs[mode] = (Rd, Ed, Qd, Pd)
    for a, b in zip(outs["eager"], outs["graph"]):
        assert torch.equal(a, b)
    o = oracle.compress_step(M, e, Q0)
    A = M.astype(np.float64) + e
    assert rel(outs["graph"][0].double().cpu().numpy(), o["recon"], A) <= TOL32
