"""Host policy switches (§8(a) a10) against hand-derived values."""
import pytest

from paper_2301_09830_b200 import policy as pol


def test_epilogue_mask_two_stages_sixteen_microbatches():
    # reading C10: P=2, M=16 -> only k = 15 is compressed
    got = [k for k in range(16) if pol.epilogue_compressed(k, 16, 2, 1)]
    assert got == [15]


def test_epilogue_mask_four_stages():
    # receiver s-1 has P-s cool-down backwards: stage 3 -> 2: {7}; 2 -> 1: {6,7}; 1 -> 0: {5,6,7}
    M, P = 8, 4
    assert [k for k in range(M) if pol.epilogue_compressed(k, M, P, 3)] == [7]
    assert [k for k in range(M) if pol.epilogue_compressed(k, M, P, 2)] == [6, 7]
    assert [k for k in range(M) if pol.epilogue_compressed(k, M, P, 1)] == [5, 6, 7]
    with pytest.raises(ValueError):
        pol.epilogue_compressed(0, M, P, 0)


def test_selective_stage_set():
    assert pol.sc_stages(4, 0.75) == {0, 1, 2}
    assert pol.sc_stages(2, 0.75) == {0, 1}         # reading C11
    assert pol.sc_stages(4, 0.0) == set()
    assert pol.sc_stages(4, 1.0) == {0, 1, 2, 3}


def test_warmup_and_rank1_bypass():
    p = pol.Policy()
    assert not pol.cb_compressed(p, 29999, 15, 16, 2, 1)
    assert pol.cb_compressed(p, 30000, 15, 16, 2, 1)
    assert not pol.cb_compressed(p, 30000, 14, 16, 2, 1)
    assert not pol.dp_compressed(p, 40000, 0, 4, 1)    # bias / LayerNorm (C16)
    assert pol.dp_compressed(p, 40000, 0, 4, 2)
    assert not pol.dp_compressed(p, 40000, 3, 4, 2)


def test_groups_two_pp_four_dp():
    assert pol.dp_group(0, 4) == [0, 1, 2, 3]
    assert pol.dp_group(1, 4) == [4, 5, 6, 7]
    assert pol.pp_group(2, 4, 2) == [2, 6]
    assert pol.fe_group(4, 2) == list(range(8))
    assert pol.fe_scale(4) == 0.25
    assert pol.is_embedding("language_model.embedding.word_embeddings.weight")
    assert not pol.is_embedding("layers.0.mlp.dense_h_to_4h.weight")


def test_kernel_rank_maps_paper_ranks_to_built_instances():
    p = pol.Policy()
    assert p.kernel_rank(p.cb_rank) == 16          # PAPER.md:773 CB rank is built
    assert p.kernel_rank(p.dp_rank) == 64          # 128 is not built: the largest built rank below it
    assert p.kernel_rank(33) == 32 and p.kernel_rank(4) == 4
    with pytest.raises(ValueError):
        p.kernel_rank(3)
