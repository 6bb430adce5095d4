"""Oracle pins by invariants, closed forms (round-trip identity) and library-routine
reductions (numpy.take / fancy-index assignment), over seeded random scripts."""
import numpy as np
import pytest

from oracle import ALLOC, FREE, PENDING, RESERVED, BytesStore, OraclePool, ProvStore
from oracle.pool import OFFLOADED
from workloads import content
from workloads.configs import C2, C3
from workloads.replay import Replayer
from workloads.scripts import build_script, fuzz_script

GEOM = dict(L=2, T=4, H=2, D=8)          # C = 4*2*8*2 = 128 bytes


def make(N, S, seed, ncls=2):
    pool0 = content.pool_bytes(seed, GEOM["L"], N, GEOM["T"], GEOM["H"], GEOM["D"])
    return OraclePool(N, S, n_classes=ncls, store=BytesStore(pool0, S)), pool0


def check_invariants(p: OraclePool, prev_sound: bool) -> bool:
    N, S = p.N, p.S
    st = p.blk_state
    # conservation |FREE| + |ALLOC| + |PENDING| = N
    assert (st == FREE).sum() + (st == ALLOC).sum() + (st == PENDING).sum() + (st == RESERVED).sum() == N
    # gradually reserved blocks are exactly the live handles' claim lists
    assert set(np.flatnonzero(st == RESERVED).tolist()) == {b for h in p.handles.values() for b in h.resv}
    # host conservation: slots in use by live handles + released-not-returned + free list = S
    live = [s for h in p.handles.values() if h.state == OFFLOADED for s in h.slots]
    assert len(live) + len(p.released_slots) + len(p.slot_free) == S
    assert len(set(live) | set(p.released_slots) | set(p.slot_free)) == S
    # ownership: table <-> owner bijection; table entries are ALLOC blocks of that agent; -1 iff on host
    seen = set()
    for a, ag in p.agents.items():
        for pos, b in enumerate(ag.table):
            if b >= 0:
                assert st[b] == ALLOC and tuple(p.owner[b]) == (a, pos)
                assert b not in seen
                seen.add(b)
    assert seen == set(np.flatnonzero(st == ALLOC).tolist())
    host_pos = {(h.agent, q) for h in p.handles.values() if h.state == OFFLOADED for q in h.pos}
    minus = {(a, q) for a, ag in p.agents.items() for q, b in enumerate(ag.table) if b < 0}
    assert host_pos == minus
    # pending blocks are exactly the retired-at-sync list
    assert set(np.flatnonzero(st == PENDING).tolist()) == {b for _, ids in p.pending_dev for b in ids}
    # reservation soundness: free >= sum of unclaimed reservations and claimed <= reserved
    unc = sum(max(0, r - c) for r, c in zip(p.reserved, p.claimed))
    sound = (st == FREE).sum() >= unc and all(c <= r for r, c in zip(p.reserved, p.claimed))
    return sound


@pytest.mark.parametrize("seed", range(40))
def test_invariants_and_round_trip_on_fuzz(seed):
    N, S = 24, 10
    p, pool0 = make(N, S, seed)
    r = Replayer(p)
    ops = fuzz_script(seed, n_ops=120, n_agents=3, n_classes=2, N=N, gradual=seed % 2 == 1)
    snap_at_offload = {}           # handle -> bytes of its blocks at offload time, [n][L][2][C]
    sound = True
    for op in ops:
        hbefore = p.next_handle
        live_before = {h for h, x in p.handles.items() if x.state == OFFLOADED}
        pool_before = p.store.pool.copy()
        state_before = whole_state(p)
        st, out = r.step(op)
        if st != 0:                                    # strong guarantee: a refused op changes nothing at all
            assert states_equal(state_before, whole_state(p)), op
        if st == 0 and op[0] in ("offload", "offload_batch", "cycle"):
            for h in range(hbefore, p.next_handle):
                hd = p.handles[h]
                # the gathered slots hold exactly the source blocks' bytes as they were before the offload
                snap_at_offload[h] = np.stack([p.store.host[s].copy() for s in hd.slots])
        if st == 0 and op[0] in ("upload", "upload_batch", "cycle"):
            done = sorted(h for h in live_before if p.handles[h].state != OFFLOADED)
            news = [out] if op[0] == "upload" else (out[0] if op[0] == "cycle" else out)
            assert len(done) == len(news)
            touched = set()
            for h in done:
                hd = p.handles[h]
                new = [p.agents[hd.agent].table[q] for q in hd.pos]
                assert new in news
                # round-trip identity: pool[:, :, new[i]] == x_i (closed form) ...
                assert np.array_equal(p.store.pool[:, :, new].transpose(2, 0, 1, 3), snap_at_offload[h])
                touched |= set(new)
            # ... and everything else untouched
            mask = np.ones(N, bool)
            mask[list(touched)] = False
            assert np.array_equal(p.store.pool[:, :, mask], pool_before[:, :, mask])
        if st != 0 or op[0] in ("offload", "offload_batch", "sync", "alloc", "reserve", "agent_free"):
            assert np.array_equal(p.store.pool, pool_before)        # only uploads write the pool
        now_sound = check_invariants(p, sound)
        if sound and op[0] != "reserve":
            assert now_sound, op                       # selects preserve soundness (reading A9)
        sound = now_sound


def whole_state(p: OraclePool):
    """Every field of the oracle's state (S:132 / S:169 / S:178 'pool unchanged' is checked against all of it)."""
    import copy
    return (p.store.pool.copy(), p.store.host.copy(), p.blk_state.copy(), p.owner.copy(),
            {a: (g.cls, list(g.table)) for a, g in p.agents.items()}, list(p.reserved), list(p.claimed),
            list(p.slot_free), list(p.peer_free), list(p.released_slots), list(p.released_epoch),
            copy.deepcopy(p.pending_dev), list(p.pending_epoch), p.epoch, p.next_handle,
            {h: (x.agent, x.cls, x.state, list(x.pos), list(x.slots), list(x.resv), list(x.plan), x.ticks)
             for h, x in p.handles.items()})


def states_equal(a, b):
    if isinstance(a, np.ndarray):
        return np.array_equal(a, b)
    if isinstance(a, (tuple, list)):
        return len(a) == len(b) and all(states_equal(x, y) for x, y in zip(a, b))
    if isinstance(a, dict):
        return a.keys() == b.keys() and all(states_equal(a[k], b[k]) for k in a)
    return a == b


def test_round_trip_identity_explicit():
    N, S = 32, 16
    p, pool0 = make(N, S, 11)
    p.agent_add(0, 0); p.agent_add(1, 1)
    for _ in range(6):
        p.alloc(0, 2); p.alloc(1, 1)
    ids = p.block_table(0)[::2]
    x = p.store.pool[:, :, ids].copy()
    other = p.store.pool.copy()
    h = p.offload(0, ids)
    p.alloc(1, 3)
    new = p.upload(h)
    assert np.array_equal(p.store.pool[:, :, new], x)
    keep = np.ones(N, bool); keep[new] = False
    assert np.array_equal(p.store.pool[:, :, keep], other[:, :, keep])


@pytest.mark.parametrize("seed", range(10))
def test_gather_scatter_equal_numpy_routines(seed):
    rng = np.random.default_rng(seed)
    N, S = 40, 20
    p, pool0 = make(N, S, seed)
    p.agent_add(0, 0)
    p.alloc(0, 30)
    tab = p.block_table(0)
    ids = [tab[i] for i in rng.choice(30, size=int(rng.integers(1, 16)), replace=False)]
    h = p.offload(0, ids)
    slots = p.handles[h].slots
    # gather: host slots == np.take(pool, ids, axis=2) moved to [n][L][2][C]
    expect = np.take(pool0, ids, axis=2).transpose(2, 0, 1, 3)
    assert np.array_equal(p.store.host[slots], expect)
    p.sync()
    staged = p.store.host[slots].copy()
    ref = p.store.pool.copy()
    new = p.upload(h)
    ref[:, :, new] = staged.transpose(1, 2, 0, 3)          # scatter == fancy-index assignment
    assert np.array_equal(p.store.pool, ref)


def test_buffer_reuse_repeating_cycle():
    """after warm-up, a repeating offload/upload cycle of fixed size takes all host blocks from the free
    list — the set of slots used stops growing."""
    p = OraclePool(64, 32)
    p.agent_add(0, 0); p.alloc(0, 10)
    used = []
    for _ in range(6):
        h = p.offload(0, p.block_table(0)[:7])
        used.append(frozenset(p.handles[h].slots))
        p.upload(h)
        p.sync()
    assert all(u == used[0] for u in used[1:])
    assert len(set().union(*used)) == 7


@pytest.mark.parametrize("seed", range(12))
def test_prov_store_equals_byte_store(seed):
    N, S = 24, 10
    pool0 = content.pool_bytes(seed, GEOM["L"], N, GEOM["T"], GEOM["H"], GEOM["D"])
    pb = OraclePool(N, S, store=BytesStore(pool0, S))
    pp = OraclePool(N, S, store=ProvStore(N, S))
    ops = fuzz_script(seed + 100, n_ops=100, n_agents=3, N=N)
    tb = Replayer(pb).run(ops)
    tp = Replayer(pp).run(ops)
    assert tb == tp
    for b in range(N):
        assert np.array_equal(pb.store.pool[:, :, b], pool0[:, :, pp.store.prov[b]])


@pytest.mark.parametrize("cfg", [C2, C3])
def test_workload_scripts_replay_cleanly_scaled(cfg):
    """The C2/C3 generators produce scripts whose every op succeeds (scaled N, same per-agent sizes); ProvStore
    and BytesStore agree on them."""
    small = cfg.scaled(N=4096, n_agents=cfg.n_agents) if cfg is C2 else cfg.scaled(N=8192, n_agents=16, per_cycle=2)
    ops = build_script(small, 8)
    pp = OraclePool(small.N, small.host_slots(), store=ProvStore(small.N, small.host_slots()))
    tr = Replayer(pp).run(ops)
    assert all(s == 0 for s, _ in tr), [op for op, (s, _) in zip(ops, tr) if s][:3]
    assert pp.stats()["pending"] == 0
