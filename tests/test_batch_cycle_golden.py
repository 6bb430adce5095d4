"""Pins of one-cycle batch semantics (readings B1, B5): the hand-derived scenarios of
tests/golden/b1_batch_cycle_examples.json, run on the oracle — whose complete state (payload, block states, owners,
tables, quotas, host free list, pending list, handles, epochs) must be unchanged by every refused batch — and on the
C-ABI library's metadata-only pool (statuses, ids, handles, tables, counters)."""
import json
import os

import numpy as np
import pytest

import paper_2510_18586_b200 as tcb
from oracle import BytesStore, OracleError, OraclePool
from workloads import content

GOLD = os.path.join(os.path.dirname(__file__), "golden", "b1_batch_cycle_examples.json")
G = json.load(open(GOLD))
SCEN = {s["name"]: s for s in G["scenarios"]}


def full_state(p: OraclePool):
    st = p.store
    return (st.pool.copy(), st.host.copy(), p.blk_state.copy(), p.owner.copy(),
            {a: (g.cls, list(g.table)) for a, g in p.agents.items()}, list(p.reserved), list(p.claimed),
            list(p.slot_free), list(p.released_slots), list(p.released_epoch), list(p.peer_free),
            [(c, list(i)) for c, i in p.pending_dev], list(p.pending_epoch), p.epoch,
            {h: (x.agent, x.cls, x.state, list(x.pos), list(x.slots), list(x.resv), list(x.plan), x.ticks)
             for h, x in p.handles.items()}, p.next_handle)


def same(a, b):
    if isinstance(a, np.ndarray):
        return np.array_equal(a, b)
    if isinstance(a, (tuple, list)):
        return len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
    if isinstance(a, dict):
        return a.keys() == b.keys() and all(same(a[k], b[k]) for k in a)
    return a == b


class Oracle:
    def __init__(self, N, S):
        L, H, D, T = 2, 1, 8, 2
        self.pool0 = content.pool_bytes(7, L, N, T, H, D)
        self.p = OraclePool(N, S, n_classes=G["n_classes"], store=BytesStore(self.pool0, S))

    def call(self, op):
        k, args = op[0], op[1:]
        try:
            if k == "alloc":
                return 0, self.p.alloc(args[0], args[1])
            if k == "offload":
                return 0, self.p.offload(args[0], args[1])
            if k == "sync":
                return 0, self.p.sync()
            if k == "offload_batch":
                return 0, self.p.offload_batch([(a, ids) for a, ids in args[0]])
            if k == "upload_batch":
                return 0, self.p.upload_batch(args[0])
            if k == "cycle":
                news, hs = self.p.cycle(args[0], [(a, ids) for a, ids in args[1]])
                return 0, [news, hs]
        except OracleError as e:
            return e.status, None
        raise AssertionError(op)

    def table(self, a):
        return self.p.block_table(a)

    def counts(self):
        s = self.p.stats()
        return {k: s[k] for k in ("free", "alloc", "pending", "host_free")}

    def next_handle(self):
        return self.p.next_handle


class Library:
    def __init__(self, N, S):
        self.c = tcb.Pool(1, 2, 64, 16, "fp16", N, device=-1, host_slots=S, n_classes=G["n_classes"])

    def call(self, op):
        k, args = op[0], op[1:]
        try:
            if k == "alloc":
                return 0, [int(x) for x in self.c.alloc(args[0], args[1])]
            if k == "offload":
                return 0, self.c.offload(args[0], args[1])
            if k == "sync":
                return 0, self.c.sync()
            if k == "offload_batch":
                return 0, self.c.offload_batch([(a, ids) for a, ids in args[0]])
            if k == "upload_batch":
                return 0, [list(map(int, x)) for x in self.c.upload_batch(args[0])]
            if k == "cycle":
                news, hs = self.c.cycle(args[0], [(a, ids) for a, ids in args[1]])
                return 0, [[list(map(int, x)) for x in news], hs]
        except tcb.TcError as e:
            return e.status, None
        raise AssertionError(op)

    def table(self, a):
        return [int(x) for x in self.c.block_table(a)]

    def counts(self):
        s = self.c.stats()
        return {k: s[k] for k in ("free", "alloc", "pending", "host_free")}


def run(sc, impl):
    x = impl(sc["N"], sc["S"])
    for a, c in G["agents"]:
        (x.p.agent_add if isinstance(x, Oracle) else x.c.agent_add)(a, c)
    for st in sc["setup"]:
        k = st[0]
        if k == "alloc":
            assert x.call(st[:3]) == (0, st[3]), st
        elif k == "offload":
            assert x.call(st[:3]) == (0, st[3]), st
        else:
            assert x.call(st) == (0, None), st
    return x


def check_expectations(x, sc, tables_key="expect_tables"):
    for a, t in sc[tables_key].items():
        assert x.table(int(a)) == t, (sc["name"], a)


@pytest.mark.parametrize("name", list(SCEN))
def test_oracle_golden_batch_cycle(name):
    sc = SCEN[name]
    x = run(sc, Oracle)
    before = full_state(x.p)
    st, out = x.call(sc["op"])
    assert st == sc["expect_status"], (name, st)
    assert same(before, full_state(x.p)), f"{name}: a refused batch changed the oracle's state"
    check_expectations(x, sc)
    assert x.counts() == sc["expect_counts"], name
    assert x.next_handle() == sc["expect_next_handle"], name
    for op in sc.get("after", []):
        assert x.call(op[:-2]) == (op[-2], op[-1]), (name, op)
    if "after_tables" in sc:
        check_expectations(x, sc, "after_tables")


@pytest.mark.parametrize("name", list(SCEN))
def test_library_golden_batch_cycle(name):
    sc = SCEN[name]
    x = run(sc, Library)
    before = ({a: x.table(a) for a, _ in G["agents"]}, x.counts(), x.c.stats()["live_handles"])
    st, out = x.call(sc["op"])
    assert st == sc["expect_status"], (name, st)
    assert before == ({a: x.table(a) for a, _ in G["agents"]}, x.counts(), x.c.stats()["live_handles"]), name
    check_expectations(x, sc)
    assert x.counts() == sc["expect_counts"], name
    for op in sc.get("after", []):
        assert x.call(op[:-2]) == (op[-2], op[-1]), (name, op)
    if "after_tables" in sc:
        check_expectations(x, sc, "after_tables")
