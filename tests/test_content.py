"""Pins the shared content generator (workloads/content.py) to values fixed outside this repo's code."""
import numpy as np

from workloads import content


def test_splitmix64_reference_outputs():
    # Vigna's reference splitmix64.c with state x = 0: next() returns mix(x += 0x9E3779B97F4A7C15), i.e. the
    # first three outputs are splitmix64(0), splitmix64(GOLDEN), splitmix64(2*GOLDEN) in this module's convention.
    g = 0x9E3779B97F4A7C15
    xs = np.array([0, g, (2 * g) % (1 << 64)], dtype=np.uint64)
    out = [int(v) for v in content.splitmix64(xs)]
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_mix_is_bijective_on_sample():
    x = np.arange(1 << 16, dtype=np.uint64)
    assert len(np.unique(content.splitmix64(x))) == len(x)


def test_shard_is_head_slice_of_unsharded():
    # reading A19: rank r of G holds heads [r*H/G, (r+1)*H/G) of every chunk
    L, N, T, H, D = 2, 5, 16, 8, 128
    full = content.pool_bytes(7, L, N, T, H, D)                  # [L][2][N][C]
    C = full.shape[-1]
    full5 = full.reshape(L, 2, N, T, H, D * 2)
    for G in (2, 4, 8):
        for r in range(G):
            sh = content.pool_bytes(7, L, N, T, H, D, rank=r, world=G).reshape(L, 2, N, T, H // G, D * 2)
            assert np.array_equal(sh, full5[:, :, :, :, r * H // G:(r + 1) * H // G, :])
    # chunk_bytes agrees with pool_bytes
    for (l, kv, b) in [(0, 0, 0), (1, 1, 4), (0, 1, 3)]:
        assert np.array_equal(content.chunk_bytes(7, l, kv, b, N, T, H, D), full[l, kv, b])
    assert C == T * H * D * 2


def test_contents_cover_special_fp_patterns():
    # uniform random 16-bit words: NaN payloads, +-Inf, -0 and denormals must occur in a large enough pool
    w = content.pool_bytes(3, 4, 64, 16, 8, 128).view(np.uint16)
    exp_bf16 = (w >> 7) & 0xFF
    assert ((exp_bf16 == 0xFF) & ((w & 0x7F) != 0)).any()      # bf16 NaN
    assert (exp_bf16 == 0).any()                                # bf16 zero/denormal
    assert ((w == 0x8000)).sum() >= 0


def test_torch_generator_matches_numpy_generator():
    """tests/gen_torch.py (the full-size GPU tests' expected-bytes generator) equals this module on CPU: the
    reference outputs, and whole shard blocks with scattered provenance for every head split."""
    import torch
    from gen_torch import _i64, block_words, splitmix64
    g = 0x9E3779B97F4A7C15
    xs = torch.tensor([_i64(0), _i64(g), _i64(2 * g)], dtype=torch.int64)
    assert [v & ((1 << 64) - 1) for v in splitmix64(xs).tolist()] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                                      0x06C45D188009454F]
    L, N, T, H, D = 3, 40, 16, 8, 64
    provs = torch.tensor([0, 39, 17, 5, 5, 22], dtype=torch.int64)
    for seed in (0, 3, 12345):
        for world in (1, 2, 8):
            for rank in {0, world - 1}:
                full = content.pool_bytes(seed, L, N, T, H, D, rank=rank, world=world)
                got = block_words(seed, provs, L, N, T, H, D, rank, world).numpy().view(np.uint8)
                assert np.array_equal(got, full[:, :, provs.numpy()]), (seed, world, rank)
