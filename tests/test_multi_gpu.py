"""Multi-process tests.

* CPU (gloo, world size 2): the host side of the N > 1 path -- the NCCL
  unique-id bootstrap through torch.distributed and the 2 PP x D DP box
  partition of the host policy (every rank derives the same groups).
* GPU (>= 2 devices): tests/mp_check.py under torchrun -- DP factor
  allreduce, PP factor send/recv, dense and compressed embedding sync, all
  against the fp64 oracle.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, out_path):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2301_09830_b200 import occ, policy
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # unique-id bootstrap: rank 0 asks NCCL for an id, the process group broadcasts it
    import ctypes
    buf = ctypes.create_string_buffer(128)
    if rank == 0:
        assert occ.lib().occ_get_unique_id(buf) == 0
    obj = [bytes(buf.raw)]
    dist.broadcast_object_list(obj, src=0)
    # every rank derives the same 2 PP x D DP partition
    D = 4
    mine = {"dp": policy.dp_group(rank % 2, D), "pp": policy.pp_group(rank % D, D, 2), "fe": policy.fe_group(D, 2)}
    allg = [None] * world
    dist.all_gather_object(allg, (obj[0].hex(), mine))
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allg, f)
    dist.destroy_process_group()


def test_gloo_bootstrap_and_partition(tmp_path):
    import torch.multiprocessing as mp
    from paper_2301_09830_b200 import build as occ_build
    occ_build.build()
    port = _free_port()
    out = str(tmp_path / "g.json")
    mp.spawn(_gloo_worker, args=(2, port, out), nprocs=2, join=True)
    allg = json.load(open(out))
    ids = {a[0] for a in allg}
    assert len(ids) == 1 and len(next(iter(ids))) == 256     # same 128-byte id everywhere
    assert any(c != "0" for c in next(iter(ids)))
    assert allg[0][1]["fe"] == list(range(8))
    assert allg[0][1]["dp"] == [0, 1, 2, 3] and allg[1][1]["dp"] == [4, 5, 6, 7]


@pytest.mark.gpu
def test_multi_gpu_parity():
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "tests", "mp_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    names = {x["check"] for x in lines}
    assert {"dp_local_ef", "dp_global_ef", "pp_send_recv", "pp_ring_link", "emb_dense", "emb_compressed"} <= names, lines
    assert all(x["ok"] for x in lines), lines


@pytest.mark.gpu
@pytest.mark.parametrize("link", [False, True])
def test_threed_integration(link):
    """f2: two iterations of the 2 PP x D DP communication step (tests/threed_check.py)."""
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "threed_check.py")] + (["--link"] if link else [])
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    names = {x["check"] for x in lines}
    assert {"threed_backward_link", "threed_dp_sync_stage0", "threed_rank1_dense", "threed_embedding_sync"} <= names
    assert all(x["ok"] for x in lines), lines
