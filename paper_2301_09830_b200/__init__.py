"""B200-native hot path of Optimus-CC (arXiv 2301.09830): PowerSGD-style
rank-r compression with error feedback for inter-stage activation gradients,
data-parallel gradients and the fused embedding sync.

The compute path is libocc.so (include/occ.h, csrc/); `occ` is its ctypes
binding and `policy` holds the paper's host-side switches (epilogue-only
compression, selective stage compression, fused embedding group, warm-up).
"""
from . import occ, policy  # noqa: F401
from .occ import (occ_compress, occ_decompress, occ_allreduce_factors, occ_send_factors,  # noqa: F401
                  occ_recv_factors, occ_embed_sync, occ_init_q, occ_workspace_bytes, Comm)
