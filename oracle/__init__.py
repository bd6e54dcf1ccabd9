"""CPU float64 oracle for the Optimus-CC hot path.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never
imports it.  See oracle/powersgd.py for the algorithm and its citations.
"""
from .powersgd import (splitmix64, fallback_vector, mgs2, round_to, compress_step,
                       decompress, dp_step, embed_sync_sequential, embed_sync_fused)
from .costmodel import allreduce_cost, c_emb, c_emb_fused, compression_ratio

__all__ = ["splitmix64", "fallback_vector", "mgs2", "round_to", "compress_step",
           "decompress", "dp_step", "embed_sync_sequential", "embed_sync_fused",
           "allreduce_cost", "c_emb", "c_emb_fused", "compression_ratio"]
