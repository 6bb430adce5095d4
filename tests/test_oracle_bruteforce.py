"""Brute force: every op sequence of depth <= 5 over a fixed 15-op alphabet on tiny pools,
oracle vs the independent set-based model in tests/brute_model.py; plus all 2^8 subsets x 2 orders of C1's 8-block
offload.  States already explored at the same remaining depth (identical oracle AND model state) are not
re-expanded: their futures are identical by determinism, so every sequence's behaviour is still covered."""
import copy

import numpy as np
import pytest

from oracle import BytesStore, OracleError, OraclePool
from oracle.pool import OFFLOADED
from workloads import content

from brute_model import Fail, SetModel

A, B = 0, 1
ALPHABET = ([("alloc", a, n) for a in (A, B) for n in (1, 2)]
            + [("offload", a, sel) for a in (A, B) for sel in ("all", "first")]
            + [("upload", w) for w in ("oldest", "newest")]
            + [("sync",)] + [("reserve", 0, n) for n in (0, 2)] + [("agent_free", a) for a in (A, B)])
assert len(ALPHABET) == 15
# NEXT-1 gradual reservation: begin a 2-tick reservation for the oldest live handle; one scheduling tick
ALPHABET_R = ALPHABET + [("reserve_begin", 2), ("tick",)]
# reading A8': retire without draining (only what was enqueued before the previous retire / sync point)
ALPHABET_RT = ALPHABET + [("retire",)]
# reading A8'': retire against the lag-th previous point (lag 2), and the refused lag 0
ALPHABET_RL = ALPHABET + [("retire",), ("retire", 2), ("retire", 0)]
# readings B1 / B5: one cycle's batches — two agents' offloads, an overlapping pair (INVAL at item 2),
# all live uploads, a duplicate upload (HANDLE), uploads-then-offloads cycles, and a cycle whose offload names the
# lowest free block for the uploaded agent (the block its own upload takes: B5)
ALPHABET_B = ALPHABET + [("offload_batch", ((A, "all"), (B, "all"))), ("offload_batch", ((A, "first"), (A, "all"))),
                         ("upload_batch", "all"), ("upload_batch", "dup"), ("cycle", (B, "all")),
                         ("cycle", (A, "first")), ("cycle_b5",)]


def sel_ids(table, sel):
    on = [b for b in table if b >= 0]
    return on if sel == "all" else on[:1]


def live_handles(live):
    return sorted(live)


def batch_args(op, tab, live, free, owner):
    """The concrete arguments of a batch op, from the pre-op state (identical on both sides): tab(a) = agent a's
    table, live = live handles ascending, free = free block ids ascending, owner(h) = the agent of handle h."""
    k = op[0]
    if k == "offload_batch":
        return [(a, sel_ids(tab(a), sel)) for a, sel in op[1]]
    if k == "upload_batch":
        if not live:
            return [0]
        return live if op[1] == "all" else [live[0], live[0]]
    if k == "cycle":
        a, sel = op[1]
        return live[:1], [(a, sel_ids(tab(a), sel))]
    if k == "cycle_b5":
        return live[:1], [(owner(live[0]) if live else A, free[:1] or [0])]
    raise AssertionError(op)


def run_oracle(p: OraclePool, op):
    try:
        k = op[0]
        if k in ("offload_batch", "upload_batch", "cycle", "cycle_b5"):
            live = live_handles(h for h, x in p.handles.items() if x.state == OFFLOADED)
            free = [b for b in range(len(p.blk_state)) if p.blk_state[b] == 0]
            args = batch_args(op, p.block_table, live, free, lambda h: p.handles[h].agent)
            if k == "offload_batch":
                return 0, p.offload_batch(args)
            if k == "upload_batch":
                return 0, p.upload_batch(args)
            return 0, p.cycle(*args)
        if k == "alloc":
            return 0, p.alloc(op[1], op[2])
        if k == "offload":
            return 0, p.offload(op[1], sel_ids(p.block_table(op[1]), op[2]))
        if k == "upload":
            live = sorted(h for h, x in p.handles.items() if x.state == OFFLOADED)
            h = (live[0] if op[1] == "oldest" else live[-1]) if live else 0
            return 0, p.upload(h)
        if k == "sync":
            return 0, p.sync()
        if k == "reserve":
            return 0, p.reserve(op[1], op[2])
        if k == "agent_free":
            return 0, p.agent_free(op[1])
        if k == "reserve_begin":
            live = sorted(h for h, x in p.handles.items() if x.state == OFFLOADED)
            return 0, p.reserve_begin(live[0] if live else 0, op[1])
        if k == "tick":
            return 0, p.reserve_tick()
        if k == "retire":
            return 0, p.retire(*op[1:])
    except OracleError as e:
        return e.status, None
    raise AssertionError(op)


def run_model(m: SetModel, op):
    try:
        k = op[0]
        if k in ("offload_batch", "upload_batch", "cycle", "cycle_b5"):
            live = live_handles(m.live)
            args = batch_args(op, lambda a: m.tab[a], live, sorted(m.free), lambda h: m.live[h][0])
            if k == "offload_batch":
                return 0, m.offload_batch(args)
            if k == "upload_batch":
                return 0, m.upload_batch(args)
            return 0, m.cycle(*args)
        if k == "alloc":
            return 0, m.alloc(op[1], op[2])
        if k == "offload":
            return 0, m.offload(op[1], sel_ids(m.tab[op[1]], op[2]))
        if k == "upload":
            live = sorted(m.live)
            h = (live[0] if op[1] == "oldest" else live[-1]) if live else 0
            return 0, m.upload(h)
        if k == "sync":
            return 0, m.sync()
        if k == "reserve":
            return 0, m.reserve(op[1], op[2])
        if k == "agent_free":
            return 0, m.agent_free(op[1])
        if k == "reserve_begin":
            live = sorted(m.live)
            return 0, m.begin(live[0] if live else 0, op[1])
        if k == "tick":
            return 0, m.tick()
        if k == "retire":
            return 0, m.retire(*op[1:])
    except Fail as e:
        return e.status, None
    raise AssertionError(op)


def compare(p: OraclePool, m: SetModel, pool0, where):
    s = p.stats()
    assert (s["free"], s["alloc"], s["pending"]) == m.counts(), where
    assert s["reserved_blocks"] == sum(len(v) for v in m.rsv.values()), where
    assert {h: list(x.resv) for h, x in p.handles.items() if x.state == OFFLOADED and x.resv} == \
        {h: v for h, v in m.rsv.items() if v}, where
    assert p.block_table(A) == m.tab[A] and p.block_table(B) == m.tab[B], where
    assert p.reserved == m.res and p.claimed == m.clm, where
    assert p.slot_free == m.stack and p.released_slots == m.back and p.peer_free == m.pstack, where
    live = {h: (x.agent, x.pos, x.slots) for h, x in p.handles.items() if x.state == OFFLOADED}
    assert live == {h: (v[0], v[2], v[3]) for h, v in m.live.items()}, where
    # payload: every physical block holds the original bytes of the model's provenance; live slots likewise
    for b in range(m.N):
        assert np.array_equal(p.store.pool[:, :, b], pool0[:, :, m.prov[b]]), (where, b)
    for h, (_, _, _, slots) in m.live.items():
        for sl in slots:
            assert np.array_equal(p.store.host[sl], pool0[:, :, m.hprov[sl]]), (where, sl)


def key(p: OraclePool, m: SetModel):
    return (p.blk_state.tobytes(), p.owner.tobytes(), p.store.pool.tobytes(), p.store.host.tobytes(),
            tuple(tuple(g.table) for g in p.agents.values()), tuple(p.reserved), tuple(p.claimed),
            tuple(p.slot_free), tuple(p.peer_free), tuple(p.released_slots),
            tuple(map(tuple, (x[1] for x in p.pending_dev))),
            tuple((h, x.state, tuple(x.pos), tuple(x.slots)) for h, x in p.handles.items()), p.next_handle,
            tuple(sorted(m.free)), tuple(sorted(m.prov.items())), tuple(sorted(m.hprov.items())),
            tuple(m.stack), tuple(m.pstack), tuple(m.back), tuple(m.back_ep), m.ep, tuple(sorted(m.live)),
            tuple(p.pending_epoch), tuple(p.released_epoch), p.epoch,
            tuple((h, tuple(x.plan), x.ticks, tuple(x.resv)) for h, x in p.handles.items()),
            tuple(sorted((h, tuple(v[0]), v[1]) for h, v in m.rplan.items())),
            tuple(sorted((h, tuple(v)) for h, v in m.rsv.items())))


def explore(N, S, depth, alphabet=ALPHABET, P=0, seen_status=None):
    pool0 = content.pool_bytes(9, 1, N, 1, 1, 8)          # C = 16 bytes per chunk
    p = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S + P), n_peer_slots=P)
    m = SetModel(N, S, P=P)
    for a, c in ((A, 0), (B, 1)):
        p.agent_add(a, c)
        m.add(a, c)
    seen = set()
    nodes = [0]

    def dfs(p, m, d, path):
        if d == 0:
            return
        k = (d, key(p, m))
        if k in seen:
            return
        seen.add(k)
        for op in alphabet:
            p2, m2 = copy.deepcopy(p), copy.deepcopy(m)
            ro, rm = run_oracle(p2, op), run_model(m2, op)
            nodes[0] += 1
            where = path + [op]
            assert ro == rm, (where, ro, rm)
            if seen_status is not None:
                seen_status.add((op[0], ro[0]))
            compare(p2, m2, pool0, where)
            dfs(p2, m2, d - 1, where)

    dfs(p, m, depth, [])
    return nodes[0], len(seen)


@pytest.mark.parametrize("N,S,depth", [(4, 3, 5), (6, 4, 5), (5, 2, 6)])
def test_bruteforce_vs_set_model(N, S, depth):
    n, states = explore(N, S, depth)
    assert n > 1000 and states > 100


@pytest.mark.parametrize("N,S,depth", [(4, 3, 5), (6, 4, 5)])
def test_bruteforce_gradual_reservation(N, S, depth):
    n, states = explore(N, S, depth, ALPHABET_R)
    assert n > 1000 and states > 100


@pytest.mark.slow
@pytest.mark.skipif(not __import__("os").environ.get("TC_DEEP"), reason="depth-7 sweep (~3 min): TC_DEEP=1 runs it")
def test_bruteforce_vs_set_model_deep():
    explore(6, 4, 7)


def test_c1_offload_all_subsets_both_orders():
    """All 2^8 subsets x 2 orders of C1's 8-block offload, each followed by upload: round trip + ids."""
    N, S = 64, 16
    pool0 = content.pool_bytes(1, 1, N, 16, 2, 64)
    for mask in range(1, 256):
        for rev in (False, True):
            p = OraclePool(N, S, store=BytesStore(pool0, S))
            p.agent_add(0, 0); p.agent_add(1, 1)
            for _ in range(8):
                p.alloc(0, 1); p.alloc(1, 1)
            tab = p.block_table(0)
            pos = [i for i in range(8) if mask >> i & 1]
            if rev:
                pos = pos[::-1]
            ids = [tab[i] for i in pos]
            h = p.offload(0, ids)
            p.sync()
            new = p.upload(h)
            # lowest free ids first, assigned in i order (A7): freed ids are exactly `ids`, plus 16.. upward
            expect = sorted(set(range(16, N)) | set(ids))[:len(ids)]
            assert new == expect
            for i, b in zip(ids, new):
                assert np.array_equal(p.store.pool[:, :, b], pool0[:, :, i])
            t2 = p.block_table(0)
            for q, b in zip(pos, new):
                assert t2[q] == b
            assert all(t2[i] == tab[i] for i in range(8) if i not in pos)


@pytest.mark.parametrize("N,S,P,depth", [(4, 2, 1, 5), (5, 2, 2, 5), (6, 3, 2, 5)])
def test_bruteforce_peer_tier(N, S, P, depth):
    """NEXT-2 peer tier (reading C1): offloads land in the peer slots when the whole offload fits, else in the
    host buffer, else NOHOST; slots return to their own tier at sync."""
    nodes, states = explore(N, S, depth, P=P)
    assert nodes > 1000 and states > 100


@pytest.mark.parametrize("N,S,depth", [(4, 3, 5), (5, 2, 5)])
def test_bruteforce_retire(N, S, depth):
    """Every sequence over the 15-op alphabet plus `retire` (A8': retire only what was enqueued before the previous
    retire / sync point) against the set model with its own epochs."""
    nodes, states = explore(N, S, depth, alphabet=ALPHABET_RT)
    assert nodes > 1000 and states > 100


@pytest.mark.parametrize("N,S,depth", [(4, 3, 5), (5, 2, 5)])
def test_bruteforce_retire_lag(N, S, depth):
    """Every sequence over the 15-op alphabet plus retire with lag 1, 2 and the refused 0 (reading A8'': retire only
    what was enqueued before the lag-th previous retirement point) against the set model with its own epochs."""
    nodes, states = explore(N, S, depth, alphabet=ALPHABET_RL)
    assert nodes > 1000 and states > 100


@pytest.mark.parametrize("N,S,depth", [(4, 3, 5), (5, 2, 5), (6, 4, 4)])
def test_bruteforce_batches_and_cycles(N, S, depth):
    """Every sequence over the 15-op alphabet plus seven batch / cycle ops (readings B1, B5: all-or-nothing, first
    failing item's status, uploads before offloads, no offload of a block the cycle's own uploads allocate) against
    the set model's validate-then-apply batches; payload, tables, counters, slot lists and handles after every op."""
    seen = set()
    nodes, states = explore(N, S, depth, alphabet=ALPHABET_B, seen_status=seen)
    assert nodes > 1000 and states > 100
    # the batch paths' outcomes all occur: success, INVAL (overlap / B5 / empty), HANDLE (duplicate), NOBLOCKS / NOHOST
    for st in ((("offload_batch", 0), ("offload_batch", -1), ("upload_batch", 0), ("upload_batch", -4),
                ("cycle", 0), ("cycle", -1), ("cycle_b5", -1))):
        assert st in seen, st
    assert {("offload_batch", -3), ("cycle", -3), ("upload_batch", -2), ("cycle", -2)} & seen


@pytest.mark.parametrize("N,S,P,depth", [(5, 2, 2, 5)])
def test_bruteforce_batches_peer_tier(N, S, P, depth):
    """The batch / cycle alphabet with a peer tier: per-item tier choice inside a batch (NEXT-2, reading C1)."""
    nodes, states = explore(N, S, depth, alphabet=ALPHABET_B, P=P)
    assert nodes > 1000 and states > 100
