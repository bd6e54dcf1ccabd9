"""Debug driver: one occ_compress call (plus an occ_decompress of its factors)
on one shape, prints stats and parity.  Shape "n x m x r", or "ot:n x m x r"
for OCC_ORIENT_T.  Used by tools/sanitize.sh under compute-sanitizer."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2301_09830_b200 import occ  # noqa: E402
from workloads import synth  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "128x256x4"
ot = arg.startswith("ot:")
n, m, r = (int(x) for x in arg.split(":")[-1].split("x"))
M = synth.d2_gradlike(n, m, 3)
e = synth.e0(n, m, 4, like=M)
Q0 = synth.q0(n if ot else m, r, 5)
Md, Ed, Qd = (torch.from_numpy(x).cuda() for x in (M, e, Q0))
Pd = torch.empty(m if ot else n, r, device="cuda")
Rd = torch.empty_like(Md)
t = time.time()
ws = occ.occ_compress(Md, Ed, Qd, Pd, Rd, r=r, flags=occ.OCC_ORIENT_T if ot else 0)
out = torch.empty_like(Md)
if ot:
    occ.occ_decompress(Qd, Pd, out)
else:
    occ.occ_decompress(Pd, Qd, out)
torch.cuda.synchronize()
st = occ.occ_read_stats(ws)
o = oracle.compress_step(M, e, Q0, orient_t=ot)
A = M.astype(np.float64) + e
err = np.linalg.norm(Rd.double().cpu().numpy() - o["recon"]) / np.linalg.norm(A)
print(json.dumps({"shape": [n, m, r], "orient_t": ot, "path": st["path"], "recon_rel": err,
                  "decompress_bit_identical": bool(torch.equal(out, Rd)), "sec": time.time() - t}), flush=True)
