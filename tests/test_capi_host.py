"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/tokencake.h declares, and its host
logic (allocator, partitions, host-slot buffer, handles, tables, batch semantics, error statuses) replays every
script identically to the oracle.  Uses metadata-only pools (device = -1): bookkeeping without KV storage — no data
is produced or compared here (that is the -m gpu parity suite)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2510_18586_b200 as tcb
from oracle import OraclePool, ProvStore
from workloads.configs import CONFIGS
from workloads.replay import Replayer
from workloads.scripts import N_CLASSES, build_script, c1_worked_example, fuzz_script

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tokencake.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(tcb.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 29
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(tcb.SYMBOLS)


def test_strerror_and_status_codes():
    for st in (0, -1, -2, -3, -4, -5, -6, -7, -8):
        assert tcb.lib.tc_strerror(st)
    assert tcb.lib.tc_strerror(0).decode() == "ok"


def meta_pool(N, S, ncls=N_CLASSES, max_bpa=4096, L=1, H=2, D=64, P=0):
    return tcb.Pool(L, H, D, 16, "fp16", N, device=-1, host_slots=S, n_classes=ncls, max_agents=1024,
                    max_blocks_per_agent=max_bpa, peer_slots=P)


def stats_view(s):
    return {k: s[k] for k in ("free", "alloc", "pending", "reserved_blocks", "host_free", "host_used", "peer_free",
                              "peer_used", "reserved", "claimed")}


def replay_both(ops, N, S, ncls=N_CLASSES, max_bpa=4096, P=0):
    o = OraclePool(N, S, n_classes=ncls, max_agents=1024, max_blocks_per_agent=max_bpa, store=ProvStore(N, S + P),
                   n_peer_slots=P)
    c = meta_pool(N, S, ncls, max_bpa, P=P)
    ro, rc = Replayer(o), Replayer(c)
    for i, op in enumerate(ops):
        a, b = ro.step(op), rc.step(op)
        assert a == b, (i, op, a, b)
        if op[0] in ("sync", "retire", "upload_batch", "offload_batch"):
            assert stats_view(o.stats()) == stats_view(c.stats()), (i, op)
    for ag in o.agents:
        assert o.block_table(ag) == c.block_table(ag)
    assert stats_view(o.stats()) == stats_view(c.stats())
    return o, c


def test_c1_worked_example_through_capi():
    o, c = replay_both(c1_worked_example(), 64, 16)
    assert c.block_table(0) == [6, 8, 10, 12, 14, 20, 21, 22]
    s = c.stats()
    assert (s["free"], s["alloc"], s["pending"]) == (41, 23, 0)


@pytest.mark.parametrize("seed", range(60))
def test_fuzz_scripts_match_oracle(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.choice([8, 24, 64]))
    S = int(rng.choice([4, 10, 32]))
    ops = fuzz_script(seed, n_ops=150, n_agents=3, n_classes=2, N=N, max_alloc=int(rng.choice([2, 6, 12])),
                      gradual=seed % 2 == 1)
    replay_both(ops, N, S, ncls=2, max_bpa=int(rng.choice([8, 4096])))


@pytest.mark.parametrize("seed", range(30))
def test_fuzz_scripts_with_peer_tier_match_oracle(seed):
    """NEXT-2 peer tier (reading C1): tier placement, per-tier slot counts and refusals identical to the oracle."""
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.choice([16, 40]))
    S, P = int(rng.choice([3, 8])), int(rng.choice([2, 5, 12]))
    ops = fuzz_script(500 + seed, n_ops=150, n_agents=3, n_classes=2, N=N, max_alloc=int(rng.choice([2, 6])),
                      gradual=seed % 3 == 0)
    replay_both(ops, N, S, ncls=2, P=P)


def test_peer_tier_worked_example_through_capi():
    """tests/golden/next2_peer_tier.json through the C ABI (metadata-only pool): placement and counters."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "next2_peer_tier.json")))
    c = meta_pool(g["N"], g["S"], P=g["P"])
    c.agent_add(0, 0)
    c.agent_add(1, 1)
    for st in g["steps"]:
        if st["op"] == "alloc":
            assert list(c.alloc(st["agent"], st["n"])) == st["expect"]
        elif st["op"] == "offload":
            if "expect_status" in st:
                with pytest.raises(tcb.TcError) as e:
                    c.offload(st["agent"], st["ids"])
                assert e.value.status == tcb.E_NOHOST
                continue
            c.offload(st["agent"], st["ids"])
        elif st["op"] == "upload":
            assert list(c.upload(st["handle"])) == st["expect"]
        elif st["op"] == "sync":
            c.sync()
        s = c.stats()
        if "expect_peer_free" in st:
            assert (s["peer_free"], s["host_free"]) == (st["expect_peer_free"], st["expect_host_free"]), st
    assert (c.stats()["peer_used"], c.stats()["host_used"]) == (4, 6)


def test_peer_tier_rejected_with_unbuffered_ablation():
    with pytest.raises(tcb.TcError) as e:
        tcb.Pool(1, 2, 64, 16, "fp16", 8, device=-1, host_slots=4, peer_slots=2, unbuffered=True)
    assert e.value.status == tcb.E_INVAL


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_scripts_match_oracle_full_size(name):
    """Full-size (N, agents, sizes) scripts of every config: identical ids, handles, tables and counters."""
    cfg = CONFIGS[name]
    cycles = 6 if name != "c1" else 4
    ops = build_script(cfg, cycles) if name != "c1" else c1_worked_example() + fuzz_script(1, 80)
    replay_both(ops, cfg.N, cfg.host_slots(), max_bpa=cfg.max_blocks_per_agent)


def test_batch_all_or_nothing_and_first_failure_status():
    c = meta_pool(16, 6, ncls=2)
    c.agent_add(0, 0); c.agent_add(1, 1)
    c.alloc(0, 4); c.alloc(1, 4)
    before = (c.block_table(0), c.block_table(1), stats_view(c.stats()))
    # item 0 needs 4 slots, item 1 needs 4 more: cumulative NOHOST at item 1 -> nothing offloaded
    with pytest.raises(tcb.TcError) as e:
        c.offload_batch([(0, c.block_table(0)), (1, c.block_table(1))])
    assert e.value.status == tcb.E_NOHOST
    assert before == (c.block_table(0), c.block_table(1), stats_view(c.stats()))
    # item 0 NOHOST? no: item 0 invalid (block of agent 1) -> INVAL even though item 1 would be NOHOST
    with pytest.raises(tcb.TcError) as e:
        c.offload_batch([(0, c.block_table(1)[:1]), (1, c.block_table(1))])
    assert e.value.status == tcb.E_INVAL
    h = c.offload_batch([(0, c.block_table(0)[:2]), (1, c.block_table(1)[:2])])
    assert h == [1, 2]
    with pytest.raises(tcb.TcError) as e:
        c.upload_batch([1, 1])
    assert e.value.status == tcb.E_HANDLE
    assert c.upload_batch([2, 1]) == [[8, 9], [10, 11]]


def test_metadata_only_pool_refuses_data_ops():
    c = meta_pool(8, 4)
    with pytest.raises(tcb.TcError) as e:
        c.fill(1)
    assert e.value.status == tcb.E_NODEV
    with pytest.raises(tcb.TcError) as e:
        c.kv_ptr()
    assert e.value.status == tcb.E_NODEV


def test_create_rejects_bad_geometry():
    for kw in (dict(L=0), dict(H=3), dict(D=2)):
        args = dict(L=1, H=2, D=64)
        args.update(kw)
        with pytest.raises(tcb.TcError) as e:
            tcb.Pool(args["L"], args["H"], args["D"], 16, "fp16", 8, device=-1, shard_world=2 if kw.get("H") else 1)
        assert e.value.status == tcb.E_INVAL


def test_randomized_safety_suite_1e5_events_with_invariant_checks(monkeypatch):
    """S:606 randomized safety suite: 10^5 events (20 scripts x 5000 ops, peer tier and gradual reservation on) through
    the C ABI with TC_CHECK=1 — the library re-derives every SPEC invariant after each mutating call and aborts on a
    violation — while matching the oracle's statuses, ids and tables op by op."""
    monkeypatch.setenv("TC_CHECK", "1")
    total = 0
    for seed in range(20):
        rng = np.random.default_rng(seed)
        N, S, P = 48, int(rng.choice([4, 12])), int(rng.choice([0, 6]))
        ops = fuzz_script(9000 + seed, n_ops=5000, n_agents=4, n_classes=2, N=N, max_alloc=6, gradual=seed % 2 == 0)
        o = OraclePool(N, S, n_classes=2, max_agents=1024, store=ProvStore(N, S + P), n_peer_slots=P)
        c = meta_pool(N, S, ncls=2, P=P)
        ro, rc = Replayer(o), Replayer(c)
        for i, op in enumerate(ops):
            assert ro.step(op) == rc.step(op), (seed, i, op)
        assert stats_view(o.stats()) == stats_view(c.stats())
        total += len(ops)
    assert total >= 100_000


def test_per_call_trace_records():
    """tc_trace (SURVEY.md §5 tracing; SPEC S:298 offload_done / upload_done with block counts): one record per handle
    per offload / upload, in call order, with monotone host timestamps; a metadata-only pool stamps completion at
    enqueue.  tc_trace(0) stops recording; bad arguments -> INVAL."""
    c = meta_pool(32, 8)
    c.trace(16)
    c.agent_add(0, 0)
    c.agent_add(1, 1)
    a = c.alloc(0, 3)
    b = c.alloc(1, 2)
    hs = c.offload_batch([(0, list(a)), (1, list(b))])
    c.sync()
    c.upload_batch(hs)
    c.sync()
    recs = c.trace_read()
    assert [(r["op"], r["agent"], r["handle"], r["blocks"]) for r in recs] == \
        [("offload", 0, hs[0], 3), ("offload", 1, hs[1], 2), ("upload", 0, hs[0], 3), ("upload", 1, hs[1], 2)]
    for r in recs:
        assert r["bytes"] == r["blocks"] * c.block_bytes
        assert r["t_call_ns"] <= r["t_enqueued_ns"] == r["t_done_ns"]
    assert c.trace_read() == []
    c.trace(0)
    h = c.offload(0, c.block_table(0))
    assert c.trace_read() == [] and h
    with pytest.raises(tcb.TcError) as e:
        c.trace(-1)
    assert e.value.status == tcb.E_INVAL


def test_header_is_plain_c_and_demo_runs(tmp_path):
    """The boundary is a C ABI: include/tokencake.h compiles as strict C11 (-pedantic -Werror) and
    examples/c_abi_demo.c, linked against libtokencake.so, drives offload / upload / block-table remap on a
    metadata-only pool."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    exe = tmp_path / "c_abi_demo"
    libdir = os.path.dirname(tcb.LIB_PATH)
    r = subprocess.run([gcc, "-std=c11", "-pedantic", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", libdir, "-ltokencake",
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("ok: 48 blocks")


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_scripts_with_retire_match_oracle(seed, monkeypatch):
    """Reading A8' through the C ABI: scripts mixing tc_retire (retire only what was enqueued before the previous
    retirement point) with syncs, cycles, gradual reservations and the peer tier; TC_CHECK on."""
    monkeypatch.setenv("TC_CHECK", "1")
    rng = np.random.default_rng(2000 + seed)
    N, S, P = int(rng.choice([24, 64])), int(rng.choice([6, 16])), int(rng.choice([0, 4]))
    ops = fuzz_script(700 + seed, n_ops=200, n_agents=3, n_classes=2, N=N, max_alloc=6, gradual=seed % 2 == 0,
                      retire=True)
    replay_both(ops, N, S, ncls=2, P=P)


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_scripts_with_retire_lag_match_oracle(seed, monkeypatch):
    """Reading A8'' through the C ABI: tc_retire_lag with lags 1-3 and the refused 0, mixed with syncs, cycles,
    gradual reservations and the peer tier; TC_CHECK on."""
    monkeypatch.setenv("TC_CHECK", "1")
    rng = np.random.default_rng(3000 + seed)
    N, S, P = int(rng.choice([24, 64])), int(rng.choice([6, 16])), int(rng.choice([0, 4]))
    ops = fuzz_script(900 + seed, n_ops=200, n_agents=3, n_classes=2, N=N, max_alloc=6, gradual=seed % 2 == 0,
                      retire=True, lags=(0, 1, 2, 2, 3))
    replay_both(ops, N, S, ncls=2, P=P)


@pytest.mark.parametrize("name,lag", [("c2", 3), ("c3", 2)])
def test_config_scripts_retire_lag_match_oracle(name, lag):
    """bench.py's retire-each loop with a lag (tc_retire_lag), full size, metadata-only pool vs the oracle."""
    cfg = CONFIGS[name]
    ops = build_script(cfg, 8, combined=True)
    n_setup = next(i for i, op in enumerate(ops) if op[0] == "cycle")
    ops = ops[:n_setup] + [("retire", lag) if op[0] == "sync" else ("cycle_r",) + op[1:] if op[0] == "cycle" else op
                           for op in ops[n_setup:]] + [("sync",)]
    replay_both(ops, cfg.N, cfg.host_slots(), max_bpa=cfg.max_blocks_per_agent)


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_config_scripts_retire_each_match_oracle(name):
    """bench.py's default loop at full size: tc_cycle + tc_retire per cycle, a refused cycle retried once after a
    tc_sync (cycle_r) — identical statuses, ids, handles, tables and counters to the oracle (metadata-only pool)."""
    cfg = CONFIGS[name]
    ops = build_script(cfg, 8, combined=True)
    n_setup = next(i for i, op in enumerate(ops) if op[0] == "cycle")
    ops = ops[:n_setup] + [("retire",) if op[0] == "sync" else ("cycle_r",) + op[1:] if op[0] == "cycle" else op
                           for op in ops[n_setup:]] + [("sync",)]
    o, c = replay_both(ops, cfg.N, cfg.host_slots(), max_bpa=cfg.max_blocks_per_agent)


@pytest.mark.parametrize("name,lag", [("c3", 2), ("c4", 1), ("c5", 1), ("c2", 4)])
def test_retire_ladder_loop_matches_oracle(name, lag):
    """bench.py's retire-each loop with the refusal ladder (a refused tc_cycle is retried after tc_retire, then after
    tc_sync) at full size: identical statuses, ids, handles, tables and counters on the library and the oracle, and
    the ladder is actually exercised for the configs whose host buffers cannot carry the lag."""
    cfg = CONFIGS[name]
    ops = build_script(cfg, 12, combined=True)
    n_setup = next(i for i, op in enumerate(ops) if op[0] == "cycle")
    rt = ("retire",) if lag == 1 else ("retire", lag)
    ops = ops[:n_setup] + [rt if op[0] == "sync" else ("cycle_r",) + op[1:] if op[0] == "cycle" else op
                           for op in ops[n_setup:]] + [("sync",)]
    o = OraclePool(cfg.N, cfg.host_slots(), max_agents=1024, max_blocks_per_agent=cfg.max_blocks_per_agent,
                   store=ProvStore(cfg.N, cfg.host_slots()))
    c = meta_pool(cfg.N, cfg.host_slots(), max_bpa=cfg.max_blocks_per_agent)
    calls = {"retire": 0}
    orig = c.retire

    def counting_retire(k=1):
        calls["retire"] += 1
        return orig(k)
    c.retire = counting_retire
    ro, rc = Replayer(o), Replayer(c)
    for i, op in enumerate(ops):
        a, b = ro.step(op), rc.step(op)
        assert a == b, (name, i, op)
        assert a[0] == 0, (name, i, op)
    n_retire_ops = sum(1 for op in ops if op[0] == "retire")
    if name in ("c3", "c4", "c5"):
        assert calls["retire"] > n_retire_ops            # some cycles were refused and took the ladder
    assert stats_view(o.stats()) == stats_view(c.stats())
