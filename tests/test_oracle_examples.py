"""Oracle pins: SPEC worked examples, the hand-derived C1 worked example and quota pin (tests/golden/)."""
import json
import os

import numpy as np

from oracle import (ALLOC, E_BUSY, E_HANDLE, E_INVAL, E_NOBLOCKS, E_NOHOST, FREE, PENDING, BytesStore, OracleError,
                    OraclePool, ProvStore)
from workloads import content
from workloads.replay import Replayer
from workloads.scripts import c1_worked_example

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def status_of(fn, *a):
    try:
        fn(*a)
    except OracleError as e:
        return e.status
    return 0


def full_state(p: OraclePool):
    st = p.store
    pay = (st.pool.copy(), st.host.copy()) if isinstance(st, BytesStore) else (st.prov.copy(), st.host_prov.copy())
    return (pay, p.blk_state.copy(), p.owner.copy(), {a: (g.cls, list(g.table)) for a, g in p.agents.items()},
            list(p.reserved), list(p.claimed), list(p.slot_free), list(p.released_slots),
            [(c, list(i)) for c, i in p.pending_dev],
            {h: (x.agent, x.state, list(x.pos), list(x.slots)) for h, x in p.handles.items()}, p.next_handle)


def same(a, b):
    if isinstance(a, np.ndarray):
        return np.array_equal(a, b)
    if isinstance(a, (tuple, list)):
        return len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
    return a == b


# ------------------------------------------------------------------------------------------- SPEC examples
def test_spec_allocate_examples():
    g = gold("spec_block_memory_examples.json")
    e = g["allocate_free10_req4"]
    p = OraclePool(e["N"], 4); p.agent_add(0, 1)
    p.alloc(0, e["request"])
    assert p.stats()["free"] == e["expect_free"]

    e = g["allocate_noncritical_headroom0"]
    p = OraclePool(e["N"], 4); p.reserve(0, e["reserve_c0"]); p.agent_add(0, 1)
    before = full_state(p)
    assert status_of(p.alloc, 0, e["noncritical_request"]) == E_NOBLOCKS
    assert same(before, full_state(p))                       # "pool unchanged"

    e = g["allocate_critical_from_reservation"]
    p = OraclePool(e["N"], 4); p.reserve(0, e["reserve_c0"]); p.agent_add(0, 0)
    p.alloc(0, e["request"])
    assert p.claimed[0] == e["expect_claimed"]


def test_spec_free_reservation_first():
    e = gold("spec_block_memory_examples.json")["free_reservation_first"]
    # via agent_free: X holds 3, Y holds 2 (all claimed against class 0's reservation of 8)
    p = OraclePool(16, 4); p.reserve(0, e["reserved"]); p.agent_add(0, 0); p.agent_add(1, 0)
    p.alloc(0, 3); p.alloc(1, 2)
    assert p.claimed[0] == e["claimed_before"]
    p.agent_free(0)
    assert p.claimed[0] == e["expect_claimed"]
    # via offload retirement (S:141 + reading A10)
    p = OraclePool(16, 8); p.reserve(0, e["reserved"]); p.agent_add(0, 0)
    p.alloc(0, 5)
    p.offload(0, p.block_table(0)[:3])
    assert p.claimed[0] == 5                       # not yet: pending until sync
    p.sync()
    assert p.claimed[0] == e["expect_claimed"]


def test_spec_zero_blocks_is_error():
    p = OraclePool(8, 4); p.agent_add(0, 0); p.alloc(0, 2)
    assert status_of(p.alloc, 0, 0) == E_INVAL
    assert status_of(p.offload, 0, []) == E_INVAL


def test_spec_offload_buffer_first_and_exhausted():
    g = gold("spec_block_memory_examples.json")
    e = g["offload_buffer_first"]
    p = OraclePool(128, e["host_free_list"]); p.agent_add(0, 0); p.alloc(0, e["offload"])
    p.offload(0, p.block_table(0))
    s = p.stats()
    assert s["host_free"] == e["expect_free_list"] and s["host_used"] == e["expect_in_use"]

    p = OraclePool(16, 4, store=BytesStore(content.pool_bytes(1, 1, 16, 16, 2, 64), 4)); p.agent_add(0, 0)
    p.alloc(0, 5)
    before = full_state(p)
    assert status_of(p.offload, 0, p.block_table(0)) == E_NOHOST
    assert same(before, full_state(p))


def test_spec_upload_stall_and_retry():
    p = OraclePool(8, 8, store=BytesStore(content.pool_bytes(2, 1, 8, 16, 2, 64), 8))
    p.agent_add(0, 0); p.agent_add(1, 1)
    p.alloc(0, 4)
    orig = p.store.pool[:, :, p.block_table(0)].copy()
    h = p.offload(0, p.block_table(0)); p.sync()
    p.alloc(1, 8)                                            # no free blocks left
    before = full_state(p)
    assert status_of(p.upload, h) == E_NOBLOCKS              # upload stalls
    assert same(before, full_state(p))                       # handle stays valid, nothing changed
    p.agent_free(1)
    new = p.upload(h)
    assert np.array_equal(p.store.pool[:, :, new], orig)
    assert status_of(p.upload, h) == E_HANDLE                # single use


# ------------------------------------------------------------------------------------------- C1 pins
def test_c1_worked_example_golden():
    g = gold("c1_worked_example.json")
    N = g["N"]
    pool0 = content.pool_bytes(1, 1, N, 16, 2, 64)
    p = OraclePool(N, 16, store=BytesStore(pool0, 16))
    A, F = g["agents"]["A"]["id"], g["agents"]["F"]["id"]
    ops = c1_worked_example()
    r = Replayer(p)
    outs = []
    for op in ops:
        st, out = r.step(op)
        assert st == 0, op
        outs.append(out)
        if op == ("offload", A, "all"):
            assert p.block_table(A) == g["table_A_after_offload"]
            assert p.block_table(F) == g["after_interleaved_alloc"]["F"]
    assert outs[-5] == g["alloc_F_4_while_pending"]
    assert outs[-3] == g["alloc_F_3_after_sync"]
    assert outs[-2] == g["upload_new_ids"]
    assert p.block_table(A) == g["upload_new_ids"]
    s = p.stats()
    assert {k: s[k] for k in ("free", "alloc", "pending")} == g["final_counts"]
    for dst, src in g["final_bytes_provenance"].items():
        assert np.array_equal(p.store.pool[:, :, int(dst)], pool0[:, :, src])


def test_c1_interleaved_alloc_prefix():
    g = gold("c1_worked_example.json")
    p = OraclePool(64, 16); p.agent_add(0, 0); p.agent_add(1, 1)
    for _ in range(8):
        p.alloc(0, 1); p.alloc(1, 1)
    assert p.block_table(0) == g["after_interleaved_alloc"]["A"]
    assert p.block_table(1) == g["after_interleaved_alloc"]["F"]


def test_c1_quota_pin():
    g = gold("c1_quota_pin.json")
    p = OraclePool(g["N"], 16)
    ids = {"A": 0, "F": 1}
    p.agent_add(0, 0); p.agent_add(1, 1)
    for s in g["steps"]:
        if s["op"] == "reserve":
            p.reserve(s["cls"], s["n"])
        elif "expect_status" in s:
            assert status_of(p.alloc, ids[s["agent"]], s["n"]) == E_NOBLOCKS
        else:
            assert p.alloc(ids[s["agent"]], s["n"]) == s["expect_ids"]
            if "expect_claimed0" in s:
                assert p.claimed[0] == s["expect_claimed0"]


def test_error_paths_leave_state_unchanged():
    p = OraclePool(16, 4, store=BytesStore(content.pool_bytes(5, 1, 16, 16, 2, 64), 4))
    p.agent_add(0, 0); p.agent_add(1, 0)
    p.alloc(0, 3); p.alloc(1, 2)
    t0 = p.block_table(0)
    h = p.offload(0, t0[:2])
    cases = [
        (p.offload, 0, [t0[2], t0[2]]),           # duplicate ids
        (p.offload, 0, [t0[0]]),                  # pending (already offloaded) block
        (p.offload, 1, [t0[2]]),                  # block of another agent
        (p.offload, 0, [99]),                     # out of range
        (p.offload, 7, [t0[2]]),                  # unknown agent
        (p.upload, h + 5),                        # unknown handle
        (p.agent_free, 0),                        # BUSY: agent 0 has an offloaded handle
        (p.reserve, 0, 17),                       # sum of reservations > N
        (p.reserve, 9, 1),                        # unknown class
        (p.agent_add, 1, 0),                      # duplicate agent
        (p.alloc, 1, 0),
    ]
    expect = [E_INVAL, E_INVAL, E_INVAL, E_INVAL, E_INVAL, E_HANDLE, E_BUSY, E_INVAL, E_INVAL, E_INVAL, E_INVAL]
    for (fn, *args), st in zip(cases, expect):
        before = full_state(p)
        assert status_of(fn, *args) == st, (fn.__name__, args)
        assert same(before, full_state(p)), (fn.__name__, args)


def test_block_states_and_location_flags():
    p = OraclePool(8, 8); p.agent_add(0, 0); p.alloc(0, 3)
    t = p.block_table(0)
    p.offload(0, [t[1]])
    assert p.blk_state[t[1]] == PENDING and p.block_table(0)[1] == -1
    assert p.blk_state[t[0]] == ALLOC
    p.sync()
    assert p.blk_state[t[1]] == FREE


# ------------------------------------------------------------------------------------------- NEXT-1 gradual reservation
def _offloaded(N, n, S=None, cls=0):
    p = OraclePool(N, S or max(n, 1))
    p.agent_add(0, cls); p.agent_add(1, 1)
    p.alloc(0, n)
    h = p.offload(0, p.block_table(0))
    p.sync()
    return p, h


def test_spec_gradual_reservation_chunks():
    g = gold("spec_gradual_reservation.json")
    for key in ("even_split", "largest_first"):
        e = g[key]
        p, h = _offloaded(256, e["n"])
        p.reserve_begin(h, e["cycles"])
        got = []
        for _ in range(e["cycles"]):
            before = p.reserve_info(h)[0]
            p.reserve_tick()
            got.append(p.reserve_info(h)[0] - before)
        assert got == e["expect_chunks"], key
        assert p.reserve_info(h) == (e["n"], e["n"])


def test_spec_gradual_reservation_total_shortfall_then_stall():
    p, h = _offloaded(16, 8)
    p.alloc(1, 16)                                    # device_free = 0 at every tick
    p.reserve_begin(h, 4)
    for _ in range(4):
        p.reserve_tick()
    assert p.reserve_info(h) == (0, 8)                # readiness 0 at the deadline
    assert status_of(p.upload, h) == E_NOBLOCKS       # falls back to the stall path


def test_spec_reservation_covers_demand():
    e = gold("spec_gradual_reservation.json")["reservation_covers_demand"]
    n = e["n"]
    p, h = _offloaded(2 * n, n)
    p.reserve_begin(h, 4)
    for _ in range(4):
        p.reserve_tick()
    p.alloc(1, p.stats()["free"])                     # now device_free = 0
    assert p.stats()["free"] == 0
    new = p.upload(h)                                 # no allocation stall
    assert len(new) == n and p.stats()["reserved_blocks"] == 0


def test_gradual_reservation_shortfall_carries_and_cancel():
    p, h = _offloaded(32, 12)
    p.alloc(1, 18)                                    # free = 2 (12 pending retired -> 14 free; 18 taken... )
    free0 = p.stats()["free"]
    p.reserve_begin(h, 3)                             # chunks 4/4/4
    p.reserve_tick()
    assert p.reserve_info(h)[0] == min(4, free0)
    p.agent_free(1)                                   # blocks come back: the shortfall carries
    p.reserve_tick()
    assert p.reserve_info(h)[0] == 8
    before = p.stats()
    p.reserve_cancel(h)
    after = p.stats()
    assert after["free"] == before["free"] + 8 and after["reserved_blocks"] == 0
    assert p.upload(h) == list(range(12))             # plain lowest-free upload after the cancel


def test_next2_peer_tier_worked_example():
    """NEXT-2 peer tier (reading C1) — tests/golden/next2_peer_tier.json, hand-derived."""
    g = gold("next2_peer_tier.json")
    N, S, P = g["N"], g["S"], g["P"]
    pool0 = content.pool_bytes(5, 2, N, 16, 1, 8)
    p = OraclePool(N, S, store=BytesStore(pool0, S + P), n_peer_slots=P)
    p.agent_add(0, 0)
    p.agent_add(1, 1)
    codes = {"NOHOST": E_NOHOST}
    for st in g["steps"]:
        if st["op"] == "alloc":
            assert p.alloc(st["agent"], st["n"]) == st["expect"]
        elif st["op"] == "offload":
            if "expect_status" in st:
                before = full_state(p)
                assert status_of(p.offload, st["agent"], st["ids"]) == codes[st["expect_status"]]
                assert same(before, full_state(p))
                continue
            h = p.offload(st["agent"], st["ids"])
            assert p.handles[h].slots == st["expect_slots"], st
        elif st["op"] == "upload":
            assert p.upload(st["handle"]) == st["expect"]
        elif st["op"] == "sync":
            p.sync()
            assert p.stats()["free"] == st["expect_free_blocks"]
        s = p.stats()
        if "expect_peer_free" in st:
            assert s["peer_free"] == st["expect_peer_free"] and s["host_free"] == st["expect_host_free"], st
    for new, orig in zip((13, 14, 15), (0, 1, 2)):
        assert np.array_equal(p.store.pool[:, :, new], pool0[:, :, orig])
    s = p.stats()
    assert s["peer_used"] == 4 and s["host_used"] == 6          # peer: handle 3 (slot 11) + the last offload


def test_peer_tier_slot_conservation():
    """With P = 0 the peer tier never engages (every slot id < S); with P > 0 a random script conserves slots per
    tier after every op (per tier)."""
    from workloads.scripts import fuzz_script
    N, S = 40, 12
    for P in (0, 6):
        pool0 = content.pool_bytes(11, 2, N, 16, 1, 8)
        p = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S + P), n_peer_slots=P)
        r = Replayer(p)
        for op in fuzz_script(21, n_ops=120, n_agents=3, n_classes=2, N=N, max_alloc=5):
            r.step(op)
            s = p.stats()
            assert s["host_free"] + s["host_used"] + sum(1 for x in p.released_slots if x < S) == S
            assert s["peer_free"] + s["peer_used"] + sum(1 for x in p.released_slots if x >= S) == P
            if P == 0:
                assert all(x < S for h in p.handles.values() for x in h.slots)
        if P:
            assert any(x >= S for h in p.handles.values() for x in h.slots)


def test_retire_without_drain_example():
    """Reading A8': tests/golden/a8_retire_example.json, hand-derived."""
    g = gold("a8_retire_example.json")
    p = OraclePool(g["N"], g["S"], store=ProvStore(g["N"], g["S"]))
    p.agent_add(0, 0)
    p.agent_add(1, 0)
    for st in g["steps"]:
        if st["op"] == "alloc":
            assert p.alloc(st["agent"], st["n"]) == st["expect"]
        elif st["op"] == "offload":
            p.offload(st["agent"], st["ids"])
        elif st["op"] == "upload":
            assert p.upload(st["handle"]) == st["expect"]
        elif st["op"] == "retire":
            p.retire()
        elif st["op"] == "sync":
            p.sync()
        s = p.stats()
        if "expect_free" in st:
            assert (s["free"], s["pending"]) == (st["expect_free"], st["expect_pending"]), st
        if "expect_host_free" in st:
            assert s["host_free"] == st["expect_host_free"], st


def test_retire_lag_example():
    """Reading A8'': tests/golden/a8_retire_lag_example.json, hand-derived (retire against the lag-th
    previous retirement point; lag 0 refused with no change)."""
    g = gold("a8_retire_lag_example.json")
    p = OraclePool(g["N"], g["S"], store=ProvStore(g["N"], g["S"]))
    for a in range(3):
        p.agent_add(a, 0)
    for st in g["steps"]:
        try:
            if st["op"] == "alloc":
                assert p.alloc(st["agent"], st["n"]) == st["expect"]
            elif st["op"] == "offload":
                p.offload(st["agent"], st["ids"])
            elif st["op"] == "upload":
                assert p.upload(st["handle"]) == st["expect"]
            elif st["op"] == "retire":
                p.retire(st.get("lag", 1))
            elif st["op"] == "sync":
                p.sync()
            assert "expect_error" not in st, st
        except OracleError as e:
            assert st.get("expect_error") == "INVAL" and e.status == E_INVAL, st
        s = p.stats()
        if "expect_free" in st:
            assert (s["free"], s["pending"]) == (st["expect_free"], st["expect_pending"]), st
        if "expect_host_free" in st:
            assert s["host_free"] == st["expect_host_free"], st
