"""Per-CTA phase trace of the fused v2 kernel: work vs barrier wait, median / max over CTAs."""
import os, sys, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OCC_LIB"] = "trace"   # the instrumented library (build.py --trace)
from paper_2301_09830_b200 import build as _b
_b.build(trace=True)
import numpy as np, torch
from paper_2301_09830_b200 import occ
from workloads import synth

S = 24   # stamps per CTA (kTrStamps)
SEG = [("phase1", 0, 1), ("B1 wait", 1, 2), ("ph2 w0: Pband + Q~part", 2, 3), ("ph2 w15: Pband + gram", 2, 14),
       ("B2 (w0 arrive -> release)", 3, 4), ("grpA G reduce", 4, 6), ("w15 LDL (after G)", 6, 8), ("Q~ reduce (after G)", 6, 7),
       ("Li ready (after G)", 6, 5), ("w15 inverse", 8, 15), ("apply Li (or general path)", 5, 12),
       ("tables", 12, 13), ("B3 wait", 9, 10), ("phase5", 10, 11), ("p5: Q prefetch", 10, 16), ("p5: 1st tmem ld", 16, 17),
       ("p5: 1st MMAs", 17, 18), ("p5: 1st stores", 18, 19), ("p5: rest of 1st cg", 19, 20), ("p5: other cg", 20, 11)]


def run(n, m, r, reps=8):
    M = torch.from_numpy(synth.d2_gradlike(n, m, 5)).cuda()
    E = torch.from_numpy(synth.e0(n, m, 6, like=synth.d2_gradlike(64, 64, 1))).cuda()
    Q = torch.from_numpy(synth.q0(m, r, 7)).cuda()
    P = torch.empty(n, r, device="cuda")
    R = torch.empty_like(M)
    ws = occ.alloc_workspace(n, m, r)
    pair = bool(os.environ.get("PAIR"))   # warm-code experiment: a call on other data right before the traced one
    if pair:
        M2 = torch.from_numpy(synth.d2_gradlike(n, m, 15)).cuda()
        E2 = torch.from_numpy(synth.e0(n, m, 16, like=synth.d2_gradlike(64, 64, 1))).cuda()
        Q2, P2, R2 = Q.clone(), P.clone(), torch.empty_like(M)
    flush = torch.ones(64 * 1024 * 1024, device="cuda")
    sink = torch.empty(1, device="cuda")
    buf = (ctypes.c_uint64 * (160 * 2 * S))()
    res = {}
    for i in range(reps):
        if not os.environ.get("NOFLUSH"):
            torch.sum(flush, dim=0, out=sink[0])
        if pair:
            occ.occ_compress(M2, E2, Q2, P2, R2, r=r, ws=ws)
        occ.occ_compress(M, E, Q, P, R, r=r, ws=ws)
        torch.cuda.synchronize()
        assert occ.lib().occ_read_trace(ws.data_ptr(), buf, 160 * 2 * S, None) == 0
        st = occ.occ_read_stats(ws)
        if i < 3:
            continue
        g = st["grid"]
        tr = np.array(buf[: g * 2 * S], dtype=np.float64).reshape(g, 2 * S)
        gt = tr[:, S:]
        ck = tr[:, :S]
        t0 = gt[:, 0].min()
        for name, a, b in SEG:
            d = (gt[:, b] - gt[:, a]) / 1e3
            res.setdefault(name, []).append((np.median(d), d.max()))
            c = (ck[:, b] - ck[:, a]) / 1e3
            res.setdefault(name + " [kclk]", []).append((np.median(c), c.max()))
        res.setdefault("total(max end - min start)", []).append(((gt[:, 11].max() - t0) / 1e3,) * 2)
        res.setdefault("start skew", []).append(((gt[:, 0].max() - t0) / 1e3,) * 2)
    out = {k: {"median_us": round(float(np.median([x[0] for x in v])), 2), "max_us": round(float(np.median([x[1] for x in v])), 2)}
           for k, v in res.items()}
    print(json.dumps({"shape": [n, m, r], "grid": g, "second_pass": st["second_pass"], "kappa": st["kappa_est"], "fallback": st["fallback_columns"], "q_amp": st["q_amp"], "q_fused": st["q_fused"]}))
    for k, v in out.items():
        print(f"  {k:28s} median {v['median_us']:7.2f} us   max {v['max_us']:7.2f} us")


if __name__ == "__main__":
    for spec in sys.argv[1:] or ["4096x1920x16"]:
        run(*map(int, spec.split("x")))
