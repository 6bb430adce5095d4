"""The five BASELINE.json configs as geometry + workload parameters.

Pure data: no method arithmetic.  Sizes: chunk C = T*(H/G)*D*e bytes per (block, layer, K|V); block shard
B = 2*L*C bytes (SURVEY.md §8 header).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class Config:
    name: str
    title: str
    L: int
    H: int
    D: int
    dtype: str                # "fp16" | "bf16" (payload = opaque 16-bit words)
    T: int = 16               # tokens per block (reading A1)
    G: int = 1                # head-shard world size the config is defined for
    N: int = 64               # blocks per GPU pool
    host_frac: float = 0.18   # pinned host slots as a fraction of N ("18.5 %" stalled share; P:674 swap)
    seed: int = 1
    n_agents: int = 1
    classes: tuple = ()       # agent classes (names) for the agents; background class appended
    quotas: tuple = ()        # (class index, fraction of N) reservations (Space Scheduler output, a1)
    bg_fill: float = 0.0      # background requests fill this fraction of N before the steady state
    med_blocks: float = 8     # log-normal median blocks per agent
    sigma: float = 0.0
    clamp: tuple = (1, 1 << 30)
    per_cycle: int = 1        # offloads (and uploads) per scheduling cycle (a8)
    stall_cycles: int = 2     # cycles an agent stays offloaded (FC duration in cycles)
    fill_chunk: int = 1       # decode-like interleaving granularity of the pre-fill
    sweep: tuple = ()         # C5: offload sizes swept
    churn: float = 0.0        # C5: random-free churn pass fraction
    max_blocks_per_agent: int = 4096
    extra: dict = field(default_factory=dict)

    @property
    def elem_bytes(self) -> int:
        return 2

    def chunk_bytes(self, G: int | None = None) -> int:
        G = self.G if G is None else G
        return self.T * (self.H // G) * self.D * self.elem_bytes

    def block_bytes(self, G: int | None = None) -> int:
        return 2 * self.L * self.chunk_bytes(G)

    def host_slots(self) -> int:
        return max(1, int(self.N * self.host_frac))

    def scaled(self, N: int, host_slots: int | None = None, **kw) -> "Config":
        """Same shapes and per-offload sizes on a smaller pool (for host-RAM-bounded oracle runs)."""
        hf = (host_slots / N) if host_slots else self.host_frac
        return replace(self, N=N, host_frac=hf, **kw)


C1 = Config("c1", "tiny pool: 1 layer, 2 KV heads, head_dim 64, 64-block fp16 pool, offload+upload 8 blocks",
            L=1, H=2, D=64, dtype="fp16", N=64, host_frac=0.25, seed=1, n_agents=1, med_blocks=8,
            max_blocks_per_agent=64)
C2 = Config("c2", "Qwen2.5-7B-shaped KV bf16, Code-Writer-style 16 agents stalling/resuming on 1 B200",
            L=28, H=4, D=128, dtype="bf16", N=65536, seed=2, n_agents=16,
            classes=("programmer", "reviewer", "tester"), bg_fill=0.70, med_blocks=48, sigma=0.8,
            clamp=(1, 2048), per_cycle=2, stall_cycles=2, fill_chunk=4)
C3 = Config("c3", "Llama-3-8B-shaped KV bf16, Deep-Research-style 64 agents with Space-Scheduler partitions",
            L=32, H=8, D=128, dtype="bf16", N=32768, seed=3, n_agents=64,
            classes=("planner", "searcher", "summarizer", "writer"), quotas=((0, 0.10), (1, 0.05)),
            bg_fill=0.20, med_blocks=256, sigma=0.6, clamp=(16, 512), per_cycle=8, stall_cycles=1,
            fill_chunk=8, host_frac=0.25)
C4 = Config("c4", "Qwen2.5-32B-shaped KV bf16 head-sharded across 2/4/8 B200, 128 agents",
            L=64, H=8, D=128, dtype="bf16", N=32768, G=8, seed=4, n_agents=128,
            classes=("planner", "searcher", "summarizer", "writer"), quotas=((0, 0.10), (1, 0.05)),
            bg_fill=0.15, med_blocks=128, sigma=0.8, clamp=(1, 2048), per_cycle=16, stall_cycles=1,
            fill_chunk=8, host_frac=0.25)
C5 = Config("c5", "Llama-3-70B-shaped KV bf16 on 8xB200, 256 agents at ~18% of the pool stalled, sweep 1-512",
            L=80, H=8, D=128, dtype="bf16", N=131072, G=8, seed=5, n_agents=256,
            classes=("planner", "searcher", "summarizer", "writer"), quotas=((0, 0.10), (1, 0.05)),
            bg_fill=0.0, med_blocks=445, sigma=0.0, clamp=(1, 512), per_cycle=24, stall_cycles=2, host_frac=0.25,
            fill_chunk=16, sweep=(1, 2, 4, 8, 16, 32, 64, 128, 256, 512), churn=0.10, max_blocks_per_agent=8192)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
