"""CPU ORACLE for the Space-Scheduler update step — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SPEC.md space_scheduler run against the block pool (oracle/pool.py): on each partition update the
agent types (= the pool's classes) are scored (static + the sum of the dynamic priorities of that type's waiting
requests), the top critical_ratio types are selected, Alg. 2 turns the
pool's own usage — total non-free blocks, and per class the on-GPU blocks its agents hold — into reserve_num, and
the quotas are applied to the pool's partitions at once (lazy shrink; non-critical classes get 0).
critical_inversion(evicted, cause) = the evicted type's last combined score is strictly higher.
Composed of oracle/scheduler.py's functions; class indices are the type keys (ties -> lower index).  Reading
DESIGN.md C3.
"""
from __future__ import annotations

from .pool import ALLOC, E_INVAL, FREE, OraclePool, OracleError
from .scheduler import dynamic_priority, select_critical, update_memory_reservations


class SpaceSchedulerOracle:
    def __init__(self, pool: OraclePool, gpu_usage_high: float = 0.85, gpu_usage_low: float = 0.50,
                 adjustment_step: float = 0.05, reserve_ratio_max: float = 0.40, critical_ratio: float = 0.25,
                 initial_reserve_ratio: float = 0.0):
        self.pool = pool
        self.pp = dict(gpu_usage_high=gpu_usage_high, gpu_usage_low=gpu_usage_low, adjustment_step=adjustment_step,
                       reserve_ratio_max=reserve_ratio_max)
        self.critical_ratio = critical_ratio
        self.ratio = initial_reserve_ratio
        self.scores: dict = {}

    def usage(self) -> tuple:
        """(non-free blocks, {class: on-GPU blocks held by its agents})."""
        p = self.pool
        total = p.N - int((p.blk_state == FREE).sum())
        per = {c: 0 for c in range(p.n_classes)}
        for a, ag in p.agents.items():
            per[ag.cls] += sum(1 for b in ag.table if b >= 0 and p.blk_state[b] == ALLOC)
        return total, per

    def update(self, static_scores, waiting) -> dict:
        """static_scores[c] per class; waiting = [(class, time_wait_ms, tokens_req), ...]."""
        n = self.pool.n_classes
        if len(static_scores) != n or any(not (0 <= c < n) for c, _, _ in waiting):
            raise OracleError(E_INVAL, "one static score per class; waiting classes in range")
        scores = {c: float(static_scores[c]) for c in range(n)}
        for c, tw, tok in waiting:                                       # hybrid score: static + sum dynamic
            scores[c] += dynamic_priority(tw, tok)
        critical = select_critical(scores, self.critical_ratio)
        usage, per = self.usage()
        self.ratio, r_total, reserve = update_memory_reservations(self.ratio, usage, self.pool.N, critical, scores,
                                                                 per, **self.pp)   # Alg. 2
        new = [reserve.get(c, 0) for c in range(n)]
        if sum(new) > self.pool.N:
            raise OracleError(E_INVAL, "reservations exceed the pool")
        self.pool.reserved = list(new)                                   # applied at once; claimed untouched
        self.scores = scores
        return {"reserve": new, "critical": [c in critical for c in range(n)], "ratio": self.ratio,
                "r_total": r_total, "scores": [scores[c] for c in range(n)]}

    def critical_inversion(self, evicted_cls: int, cause_cls: int) -> bool:
        return self.scores.get(evicted_cls, 0.0) > self.scores.get(cause_cls, 0.0)
