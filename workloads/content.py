"""Seeded synthetic KV-cache *content* generator (shared input generator; holds none of the method's arithmetic).

Both sides of the parity contract draw their initial KV bytes from the same counter-based generator:
  * this NumPy module (used by the oracle side and by the tests' expected values), and
  * the CUDA fill kernel in ``paper_2510_18586_b200/csrc/kernels.cu`` (``tc_fill_kv``), an independent
    re-implementation of the same formula.  ``tests/test_content.py`` pins this module to hard-coded
    splitmix64 reference outputs and the GPU tests cross-check the fill kernel against it.

Content model: every 8-byte little-endian word of the *unsharded* KV pool
``[L][2][N][T][H][D]`` (16-bit elements) is ``splitmix64(key(seed, widx))`` where ``widx`` is the word's index in the
unsharded layout.  A head-shard (rank r of G, heads [r*H/G, (r+1)*H/G)) therefore holds exactly the head slice of the
unsharded bytes.  Uniform random bits make bf16/fp16 NaN payloads, +-Inf, -0 and denormals occur, which the bit-copy
path must preserve (SURVEY.md §8(d) "contents").
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
SEED_MUL = np.uint64(0xD1B54A32D192ED03)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Steele/Lea/Flood splitmix64 output function applied to state ``x`` (uint64, wraps mod 2**64)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def word_key(seed: int, widx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return np.asarray(widx, dtype=np.uint64) + np.uint64(seed) * SEED_MUL


def chunk_words(seed: int, layer: int, kv: int, orig_block: int, n_blocks: int, T: int, H: int, D: int,
                rank: int = 0, world: int = 1, elem_bytes: int = 2) -> np.ndarray:
    """uint64 words of one (block, layer, K|V) chunk of the rank's head shard, in local layout [T][H/G][D]."""
    assert (D * elem_bytes) % 8 == 0 and H % world == 0
    wpr = D * elem_bytes // 8            # words per (token, head) row
    hl = H // world
    t = np.arange(T, dtype=np.uint64)[:, None, None]
    h = (np.uint64(rank * hl) + np.arange(hl, dtype=np.uint64))[None, :, None]
    w = np.arange(wpr, dtype=np.uint64)[None, None, :]
    base = np.uint64(((layer * 2 + kv) * n_blocks + orig_block) * T)
    widx = ((base + t) * np.uint64(H) + h) * np.uint64(wpr) + w
    return splitmix64(word_key(seed, widx)).reshape(-1)


def chunk_bytes(seed: int, layer: int, kv: int, orig_block: int, n_blocks: int, T: int, H: int, D: int,
                rank: int = 0, world: int = 1, elem_bytes: int = 2) -> np.ndarray:
    return chunk_words(seed, layer, kv, orig_block, n_blocks, T, H, D, rank, world, elem_bytes).view(np.uint8)


def pool_bytes(seed: int, L: int, n_blocks: int, T: int, H: int, D: int, rank: int = 0, world: int = 1,
               elem_bytes: int = 2) -> np.ndarray:
    """Whole shard pool as uint8[L][2][N][C] (small pools only: the oracle's byte-level input)."""
    assert H % world == 0
    hl = H // world
    wpr = D * elem_bytes // 8
    C = T * hl * D * elem_bytes
    lk = np.arange(L * 2, dtype=np.uint64)[:, None, None, None, None]
    b = np.arange(n_blocks, dtype=np.uint64)[None, :, None, None, None]
    t = np.arange(T, dtype=np.uint64)[None, None, :, None, None]
    h = (np.uint64(rank * hl) + np.arange(hl, dtype=np.uint64))[None, None, None, :, None]
    w = np.arange(wpr, dtype=np.uint64)[None, None, None, None, :]
    widx = (((lk * np.uint64(n_blocks) + b) * np.uint64(T) + t) * np.uint64(H) + h) * np.uint64(wpr) + w
    words = splitmix64(word_key(seed, widx))
    return np.ascontiguousarray(words).view(np.uint8).reshape(L, 2, n_blocks, C)
