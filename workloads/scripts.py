"""Seeded op-script generator for the five configs (SURVEY.md §8(d) "Concrete synthetic inputs").

An op script is a list of tuples in a *logical* vocabulary; block ids are never written into a script — each replayer
resolves them from its own block table, so the script carries no allocator arithmetic:

  ("reserve", cls, n)                  partition quota (a1)
  ("agent_add", agent, cls)
  ("alloc", agent, n)                  decode growth
  ("offload", agent, sel)              sel = "all" (every on-GPU position, table order) | [positions]
  ("upload", agent)                    the agent's oldest outstanding handle
  ("offload_batch", [(agent, sel), ...])   one cycle's offloads (a8)
  ("upload_batch", [agent, ...])           one cycle's uploads (a8)
  ("sync",)                            drain + retire
  ("agent_free", agent)

The generator keeps only a tiny agent lifecycle (running / stalled) to decide *who* offloads or uploads in a cycle —
the LLM1 => FC => LLM2 pattern of P:348-350 with FC durations counted in scheduling cycles.
"""
from __future__ import annotations

from collections import deque

import numpy as np

from .configs import Config

N_CLASSES = 8          # pool class slots; background requests use class BG_CLASS
BG_CLASS = 7


def agent_sizes(cfg: Config, rng: np.random.Generator) -> list:
    lo, hi = cfg.clamp
    if cfg.sigma > 0:
        x = rng.lognormal(mean=np.log(cfg.med_blocks), sigma=cfg.sigma, size=cfg.n_agents)
    else:
        x = np.full(cfg.n_agents, cfg.med_blocks, dtype=np.float64)
    return [int(min(hi, max(lo, round(v)))) for v in x]


def setup_ops(cfg: Config, rng: np.random.Generator | None = None) -> tuple[list, list, list]:
    """Quotas, agents, background requests and the decode-like interleaved pre-fill.
    Returns (ops, agent_ids, background_ids)."""
    rng = rng if rng is not None else np.random.default_rng(cfg.seed)
    ops: list = []
    for c, frac in cfg.quotas:
        ops.append(("reserve", c, int(frac * cfg.N)))
    ncls = max(1, len(cfg.classes))
    agents = list(range(cfg.n_agents))
    sizes = agent_sizes(cfg, rng)
    for a in agents:
        ops.append(("agent_add", a, a % ncls))
    bg = []
    target = dict(zip(agents, sizes))
    if cfg.bg_fill > 0:
        n_bg = max(1, cfg.n_agents)
        total = int(cfg.bg_fill * cfg.N)
        for i in range(n_bg):
            b = cfg.n_agents + i
            bg.append(b)
            ops.append(("agent_add", b, BG_CLASS))
            target[b] = total // n_bg + (1 if i < total % n_bg else 0)
    # decode-like interleaving: seeded round-robin, each turn grows one request by up to fill_chunk blocks
    have = {k: 0 for k in target}
    order = [k for k in target if target[k] > 0]
    while order:
        rng.shuffle(order)
        nxt = []
        for k in order:
            g = min(cfg.fill_chunk, target[k] - have[k])
            ops.append(("alloc", k, g))
            have[k] += g
            if have[k] < target[k]:
                nxt.append(k)
        order = nxt
    if cfg.churn > 0:
        victims = rng.choice(agents, size=max(1, int(cfg.churn * len(agents))), replace=False)
        for a in victims:
            ops.append(("agent_free", int(a)))
        for a in victims:
            ops.append(("alloc", int(a), target[int(a)]))
    ops.append(("sync",))
    return ops, agents, bg


class CycleGen:
    """Steady-state scheduling cycles: uploads of agents whose FC is over, then offloads of agents entering an FC
    (P:645-647 order), then a sync.  Deterministic given the config seed."""

    def __init__(self, cfg: Config, agents: list, rng: np.random.Generator | None = None, combined: bool = False):
        self.cfg = cfg
        self.combined = combined           # emit one ("cycle", ups, offs) op per cycle (tc_cycle)
        self.rng = rng if rng is not None else np.random.default_rng(cfg.seed + 1000)
        self.running = deque(agents)
        self.stalled: deque = deque()      # (agent, cycle offloaded)
        self.t = 0

    def next_cycle(self) -> list:
        cfg = self.cfg
        ops = []
        due = []
        while self.stalled and self.stalled[0][1] <= self.t - cfg.stall_cycles and len(due) < cfg.per_cycle:
            due.append(self.stalled.popleft()[0])
        off = []
        for _ in range(min(cfg.per_cycle, len(self.running))):
            off.append(self.running.popleft())
        if self.combined and (due or off):
            ops.append(("cycle", due, [(a, "all") for a in off]))
        else:
            if due:
                ops.append(("upload_batch", due))
            if off:
                ops.append(("offload_batch", [(a, "all") for a in off]))
        for a in off:
            self.stalled.append((a, self.t))
        self.running.extend(due)
        ops.append(("sync",))
        self.t += 1
        return ops


def build_script(cfg: Config, n_cycles: int, combined: bool = False) -> list:
    ops, agents, _ = setup_ops(cfg)
    gen = CycleGen(cfg, agents, combined=combined)
    for _ in range(n_cycles):
        ops.extend(gen.next_cycle())
    return ops


def c1_worked_example() -> list:
    """SURVEY.md §8(c) 'Pinned C1 worked example' as a script (agents A=0 class 0, F=1 class 1)."""
    ops = [("agent_add", 0, 0), ("agent_add", 1, 1)]
    for _ in range(8):
        ops += [("alloc", 0, 1), ("alloc", 1, 1)]
    ops += [("offload", 0, "all"), ("alloc", 1, 4), ("sync",), ("alloc", 1, 3), ("upload", 0), ("sync",)]
    return ops


def fuzz_script(seed: int, n_ops: int = 60, n_agents: int = 3, n_classes: int = 2, N: int = 64,
                max_alloc: int = 6, p_err: float = 0.05, gradual: bool = False, retire: bool = False,
                lags: tuple = (1,)) -> list:
    """Random op mix for small pools, including error paths (bad ids, double uploads, over-quota, BUSY frees)."""
    rng = np.random.default_rng(seed)
    ops = [("agent_add", a, a % n_classes) for a in range(n_agents)]
    kinds = ["alloc", "alloc", "offload", "offload_some", "upload", "sync", "reserve", "agent_free",
             "offload_batch", "upload_batch", "cycle"] + (["reserve_begin", "tick", "tick", "reserve_cancel"] if gradual else []) \
        + (["retire", "retire"] if retire else [])
    for _ in range(n_ops):
        k = kinds[rng.integers(len(kinds))]
        a = int(rng.integers(n_agents))
        if k == "alloc":
            ops.append(("alloc", a, int(rng.integers(1, max_alloc + 1))))
        elif k == "offload":
            ops.append(("offload", a, "all"))
        elif k == "offload_some":
            ops.append(("offload", a, sorted(set(int(x) for x in rng.integers(0, 12, size=rng.integers(1, 5))))))
        elif k == "upload":
            ops.append(("upload", a))
        elif k == "sync":
            ops.append(("sync",))
        elif k == "reserve":
            ops.append(("reserve", int(rng.integers(n_classes)), int(rng.integers(0, N // 2))))
        elif k == "agent_free":
            ops.append(("agent_free", a))
        elif k == "offload_batch":
            bs = sorted(set(int(x) for x in rng.integers(n_agents, size=2)))
            ops.append(("offload_batch", [(b, "all") for b in bs]))
        elif k == "upload_batch":
            bs = sorted(set(int(x) for x in rng.integers(n_agents, size=2)))
            ops.append(("upload_batch", bs))
        elif k == "cycle":
            ups = sorted(set(int(x) for x in rng.integers(n_agents, size=int(rng.integers(0, 3)))))
            offs = sorted(set(int(x) for x in rng.integers(n_agents, size=int(rng.integers(0, 3)))))
            ops.append(("cycle", ups, [(b, "all") for b in offs]))
        elif k == "reserve_begin":
            ops.append(("reserve_begin", a, int(rng.integers(1, 4))))
        elif k == "tick":
            ops.append(("tick",))
        elif k == "retire":
            lag = int(lags[rng.integers(len(lags))])
            ops.append(("retire",) if lag == 1 else ("retire", lag))
        else:
            ops.append(("reserve_cancel", a))
        if rng.random() < p_err:
            ops.append(("alloc", 99, 1))              # unknown agent -> E_INVAL on both sides
    ops.append(("sync",))
    return ops
