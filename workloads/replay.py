"""Replays an op script (workloads/scripts.py vocabulary) against any pool object with the shared op vocabulary:
reserve, agent_add, alloc, offload, upload, offload_batch, upload_batch, sync, agent_free, block_table, stats.

Dispatch only: it resolves logical selections to ids through the pool's *own* block table and keeps, per agent, the
FIFO of handles that pool returned.  It computes nothing of the method.  Errors are any exception carrying
``.status``; they are recorded, never swallowed silently.
"""
from __future__ import annotations

from collections import defaultdict, deque


class Replayer:
    def __init__(self, pool):
        self.pool = pool
        self.handles = defaultdict(deque)     # agent -> outstanding handles, oldest first

    def _ids(self, a, sel):
        try:
            table = self.pool.block_table(a)
        except Exception as e:  # noqa: BLE001 - unknown agent: let the pool op itself report it
            if hasattr(e, "status"):
                return [-1]
            raise
        if sel == "all":
            return [b for b in table if b >= 0]
        return [table[p] if 0 <= p < len(table) else -1 for p in sel]

    def _handle(self, a):
        q = self.handles.get(a)
        return q[0] if q else 0        # 0 = "no handle" -> E_HANDLE on both sides

    def step(self, op):
        """Run one op; returns (status, output)."""
        kind = op[0]
        p = self.pool
        try:
            if kind == "reserve":
                p.reserve(op[1], op[2]); out = None
            elif kind == "agent_add":
                p.agent_add(op[1], op[2]); out = None
            elif kind == "alloc":
                out = list(p.alloc(op[1], op[2]))
            elif kind == "offload":
                h = p.offload(op[1], self._ids(op[1], op[2]))
                self.handles[op[1]].append(h); out = h
            elif kind == "upload":
                h = self._handle(op[1])
                out = list(p.upload(h))
                self.handles[op[1]].popleft()
            elif kind == "offload_batch":
                items = [(a, self._ids(a, sel)) for a, sel in op[1]]
                hs = p.offload_batch(items)
                for (a, _), h in zip(op[1], hs):
                    self.handles[a].append(h)
                out = list(hs)
            elif kind == "upload_batch":
                # distinct agents -> their oldest handles; an agent listed twice takes its next handle
                taken = defaultdict(int)
                hs = []
                for a in op[1]:
                    q = self.handles.get(a, ())
                    hs.append(q[taken[a]] if taken[a] < len(q) else 0)
                    taken[a] += 1
                out = [list(x) for x in p.upload_batch(hs)]
                for a in op[1]:
                    self.handles[a].popleft()
            elif kind in ("cycle", "cycle_r"):   # ("cycle", [upload agents], [(agent, sel), ...])
                # cycle_r: a refused cycle (no host slots / device blocks: nothing changed) is retried after a
                # tc_retire (the previous cycle's transfers return their slots / blocks), then once more after a
                # tc_sync — the caller policy of bench.py's retire-each loop ("the caller retries")
                items = [(a, self._ids(a, sel)) for a, sel in op[2]]       # resolved on pre-cycle tables
                taken = defaultdict(int)
                hs = []
                for a in op[1]:
                    q = self.handles.get(a, ())
                    hs.append(q[taken[a]] if taken[a] < len(q) else 0)
                    taken[a] += 1
                try:
                    news, out_h = p.cycle(hs, items)
                except Exception as e:  # noqa: BLE001
                    if kind != "cycle_r" or getattr(e, "status", None) not in (-2, -3):
                        raise
                    p.retire(1)
                    try:
                        news, out_h = p.cycle(hs, items)
                    except Exception as e2:  # noqa: BLE001
                        if getattr(e2, "status", None) not in (-2, -3):
                            raise
                        p.sync()
                        news, out_h = p.cycle(hs, items)
                for a in op[1]:
                    self.handles[a].popleft()
                for (a, _), h in zip(op[2], out_h):
                    self.handles[a].append(h)
                out = ([list(x) for x in news], list(out_h))
            elif kind == "sync":
                p.sync(); out = None
            elif kind == "retire":             # ("retire",) or ("retire", lag) (readings A8', A8'')
                p.retire(*op[1:]); out = None
            elif kind == "agent_free":
                p.agent_free(op[1]); out = None
            elif kind == "reserve_begin":        # gradual reservation for the agent's oldest handle (NEXT-1)
                p.reserve_begin(self._handle(op[1]), op[2]); out = None
            elif kind == "tick":
                p.reserve_tick(); out = None
            elif kind == "reserve_cancel":
                p.reserve_cancel(self._handle(op[1])); out = None
            else:
                raise ValueError(f"unknown op {op!r}")
            return 0, out
        except Exception as e:  # noqa: BLE001
            if hasattr(e, "status"):
                return int(e.status), None
            raise

    def run(self, ops, on_step=None):
        trace = []
        for i, op in enumerate(ops):
            r = self.step(op)
            trace.append(r)
            if on_step is not None:
                on_step(i, op, r)
        return trace
