"""Test-only third implementation of the seeded content generator (workloads/content.py), in plain torch int64
tensor ops so the full-size parity tests can produce the expected bytes of whole pools on the GPU.

It is not the product path (no kernel of libtokencake.so runs here) and holds none of the method's arithmetic; it is
pinned to workloads/content.py (itself pinned to splitmix64 reference outputs) by tests/test_content.py on CPU and by
tests/test_gpu_fullsize.py on the device before any comparison uses it.  uint64 arithmetic is emulated in int64:
adds and multiplies wrap mod 2**64 identically, and the logical right shift masks off the sign extension.
"""
from __future__ import annotations

import torch

_M64 = (1 << 64) - 1


def _i64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= 1 << 63 else v


GOLDEN = _i64(0x9E3779B97F4A7C15)
M1 = _i64(0xBF58476D1CE4E5B9)
M2 = _i64(0x94D049BB133111EB)
SEED_MUL = 0xD1B54A32D192ED03


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + GOLDEN
    z = (z ^ _srl(z, 30)) * M1
    z = (z ^ _srl(z, 27)) * M2
    return z ^ _srl(z, 31)


def block_words(seed: int, provs: torch.Tensor, L: int, N: int, T: int, H: int, D: int, rank: int = 0,
                world: int = 1) -> torch.Tensor:
    """Expected int64 words of the rank's head shard of blocks whose content is original block provs[i], in the
    pool's layout: [L][2][len(provs)][T * H/G * D * 2 / 8]."""
    dev = provs.device
    hl = H // world
    wpr = D * 2 // 8
    lk = torch.arange(2 * L, dtype=torch.int64, device=dev).view(-1, 1, 1, 1, 1)
    b = provs.to(torch.int64).view(1, -1, 1, 1, 1)
    t = torch.arange(T, dtype=torch.int64, device=dev).view(1, 1, -1, 1, 1)
    h = (rank * hl + torch.arange(hl, dtype=torch.int64, device=dev)).view(1, 1, 1, -1, 1)
    w = torch.arange(wpr, dtype=torch.int64, device=dev).view(1, 1, 1, 1, -1)
    widx = (((lk * N + b) * T + t) * H + h) * wpr + w
    key = widx + _i64(seed * SEED_MUL)
    return splitmix64(key).reshape(L, 2, provs.numel(), T * hl * wpr)
