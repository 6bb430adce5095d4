"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, byte for byte, on the same seeded inputs.

* small pools (C1 and fuzz scripts, several geometries with ragged chunk counts): the whole device pool, every live
  handle's pinned host image, every block table (host mirror and device table) and all counters are compared
  after every sync, in both transfer modes (DIRECT mapped-host kernels, STAGED device ring + copy engine);
* full BASELINE sizes: tests/test_gpu_fullsize.py;
* the synthetic-content fill kernel against workloads/content.py; the device tier against numpy.take.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2510_18586_b200 as tcb  # noqa: E402
from oracle import BytesStore, OraclePool  # noqa: E402
from oracle.pool import OFFLOADED  # noqa: E402
from workloads import content  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402
from workloads.replay import Replayer  # noqa: E402
from workloads.scripts import N_CLASSES, build_script, c1_worked_example, fuzz_script  # noqa: E402

MODES = {"direct": (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 0), "staged": (tcb.XFER_STAGED, tcb.XFER_STAGED, 0),
         "mixed": (tcb.XFER_DIRECT, tcb.XFER_STAGED, 0), "direct_tma": (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 1),
         "staged_tma": (tcb.XFER_STAGED, tcb.XFER_STAGED, 1), "direct_tile": (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 2),
         "staged_tile": (tcb.XFER_STAGED, tcb.XFER_STAGED, 2), "staged_tma4": (tcb.XFER_STAGED, tcb.XFER_STAGED, 3),
         "mixed_rev": (tcb.XFER_STAGED, tcb.XFER_DIRECT, 2), "copy": (tcb.XFER_COPY, tcb.XFER_COPY, 0),
         "copy_staged": (tcb.XFER_COPY, tcb.XFER_STAGED, 3), "staged_copy": (tcb.XFER_STAGED, tcb.XFER_COPY, 3),
         "auto": (tcb.XFER_AUTO, tcb.XFER_AUTO, 3), "direct_tma4": (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 3),
         "direct_default": (tcb.XFER_DIRECT, tcb.XFER_DIRECT, None),
         "direct_tile8": (tcb.XFER_DIRECT, tcb.XFER_DIRECT, 4), "staged_tile8": (tcb.XFER_STAGED, tcb.XFER_STAGED, 4)}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dev_pool(L, H, D, N, S, mode="direct", ncls=N_CLASSES, max_bpa=4096, seed=1, rank=0, world=1, staging=0,
             dtype="bf16", T=16, P=0, peer_dev=0):
    d2h, h2d, variant = MODES[mode]
    p = tcb.Pool(L, H, D, T, dtype, N, device=0, shard_rank=rank, shard_world=world, host_slots=S, n_classes=ncls,
                 max_agents=1024, max_blocks_per_agent=max_bpa, xfer_d2h=d2h, xfer_h2d=h2d, staging_bytes=staging,
                 peer_device=peer_dev if P else -1, peer_slots=P)
    if variant is not None:                 # None: the library's default launch configuration per path
        for path in range(3):
            p.set_launch_config(path, 0, 256, variant)
    p.fill(seed)
    return p


def compare_full(o: OraclePool, c: tcb.Pool, where=""):
    kv = c.kv_tensor().cpu().numpy()
    assert np.array_equal(kv, o.store.pool), f"pool bytes differ {where}"
    for a in o.agents:
        assert o.block_table(a) == c.block_table(a), (where, a)
    tab = c.table_tensor().cpu().numpy()
    for a, ag in o.agents.items():
        assert tab[a, :len(ag.table)].tolist() == ag.table, (where, a)
    so, sc = o.stats(), c.stats()
    for k in ("free", "alloc", "pending", "reserved_blocks", "host_free", "host_used", "peer_free", "peer_used",
              "reserved", "claimed"):
        assert so[k] == sc[k], (where, k)


def compare_live_host(o: OraclePool, c: tcb.Pool, where=""):
    for h, hd in o.handles.items():
        if hd.state != OFFLOADED:
            continue
        c.wait(h)
        for i, s in enumerate(hd.slots):
            assert np.array_equal(c.handle_host_bytes(h, i), o.store.host[s]), (where, h, i)


def run_script(ops, L, H, D, N, S, mode, ncls=N_CLASSES, max_bpa=4096, seed=1, staging=0, T=16, P=0, peer_dev=0):
    pool0 = content.pool_bytes(seed, L, N, T, H, D)
    o = OraclePool(N, S, n_classes=ncls, max_agents=1024, max_blocks_per_agent=max_bpa,
                   store=BytesStore(pool0, S + P), n_peer_slots=P)
    c = dev_pool(L, H, D, N, S, mode, ncls, max_bpa, seed, staging=staging, T=T, P=P, peer_dev=peer_dev)
    assert np.array_equal(c.kv_tensor().cpu().numpy(), pool0), "fill kernel != content generator"
    ro, rc = Replayer(o), Replayer(c)
    for i, op in enumerate(ops):
        a, b = ro.step(op), rc.step(op)
        assert a == b, (i, op, a, b)
        if op[0] in ("offload", "offload_batch") and a[0] == 0:
            compare_live_host(o, c, f"op {i}")
        if op[0] == "sync":
            compare_full(o, c, f"op {i}")
    c.sync()
    compare_full(o, c, "end")
    return o, c


@pytest.mark.parametrize("mode", list(MODES))
def test_c1_worked_example_bytes(mode):
    o, c = run_script(c1_worked_example(), 1, 2, 64, 64, 16, mode)
    assert c.block_table(0) == [6, 8, 10, 12, 14, 20, 21, 22]


GEOMS = [  # (L, H, D, N, S, T): ragged chunk counts vs CTA ranges, 4 KiB .. 32 KiB chunks
    (1, 2, 64, 64, 16, 16),
    (3, 2, 64, 50, 20, 16),
    (5, 4, 128, 40, 24, 16),
    (2, 8, 128, 33, 12, 16),
    (7, 1, 8, 29, 9, 3),      # C = 48 B: sub-warp chunks (ragged tail inside a chunk)
]


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_fuzz_scripts_bytes(mode, gi):
    L, H, D, N, S, T = GEOMS[gi]
    for seed in range(3):
        ops = fuzz_script(seed + 10 * gi, n_ops=90, n_agents=3, n_classes=2, N=N, gradual=seed == 2)
        run_script(ops, L, H, D, N, S, mode, ncls=2, seed=seed + 1, staging=(3 * 2 * L * T * H * D * 2), T=T)


def test_fill_kernel_matches_generator_sharded():
    L, H, D, N = 3, 8, 128, 20
    full = content.pool_bytes(5, L, N, 16, H, D)
    for world in (1, 2, 4, 8):
        for rank in range(world):
            c = dev_pool(L, H, D, N, 4, rank=rank, world=world, seed=5)
            got = c.kv_tensor().cpu().numpy().reshape(L, 2, N, 16, H // world, D * 2)
            exp = full.reshape(L, 2, N, 16, H, D * 2)[:, :, :, :, rank * H // world:(rank + 1) * H // world]
            assert np.array_equal(got, exp), (world, rank)
            c.close()


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_device_tier_equals_numpy_take(variant):
    L, H, D, N = 4, 4, 128, 64
    c = dev_pool(L, H, D, N, 4, seed=9, mode="direct")
    c.set_launch_config(2, 0, 256, variant)
    pool0 = content.pool_bytes(9, L, N, 16, H, D)
    rng = np.random.default_rng(0)
    ids = rng.choice(N, size=23, replace=False).astype(np.int32)
    dst = torch.empty(23 * c.block_bytes, dtype=torch.uint8, device="cuda:0")
    c.gather_dev(ids, dst.data_ptr())
    torch.cuda.synchronize()
    got = dst.cpu().numpy().reshape(23, L, 2, c.chunk_bytes)
    assert np.array_equal(got, np.take(pool0, ids, axis=2).transpose(2, 0, 1, 3))
    tgt = rng.choice(N, size=23, replace=False).astype(np.int32)
    c.scatter_dev(dst.data_ptr(), tgt)
    torch.cuda.synchronize()
    ref = pool0.copy()
    ref[:, :, tgt] = got.transpose(1, 2, 0, 3)
    assert np.array_equal(c.kv_tensor().cpu().numpy(), ref)


def test_special_bit_patterns_survive_round_trip():
    """NaN payloads, +-Inf, -0, denormals: the path is a bit copy (A14)."""
    L, H, D, N = 1, 2, 64, 16
    c = dev_pool(L, H, D, N, 8)
    pat = np.array([0x7FC1, 0xFFFF, 0x7F80, 0xFF80, 0x8000, 0x0001, 0x8001, 0x7FBF], dtype=np.uint16)
    words = np.resize(pat, c.kv_tensor().numel() // 2)
    c.kv_tensor().copy_(torch.from_numpy(words.view(np.uint8).reshape(c.kv_tensor().shape)))
    before = c.kv_tensor().cpu().numpy().copy()
    c.agent_add(0, 0); c.agent_add(1, 0)
    ids = c.alloc(0, 6)
    c.alloc(1, 2)
    h = c.offload(0, ids)
    c.sync()
    c.alloc(1, 3)
    new = c.upload(h)
    c.sync()
    after = c.kv_tensor().cpu().numpy()
    assert np.array_equal(after[:, :, new], before[:, :, ids])


# full BASELINE sizes: tests/test_gpu_fullsize.py (whole pool + every live host image, exhaustive)


@pytest.mark.parametrize("head_kib,piece_kib", [(0, 2), (1, 2), (3, 1024), (64, 64), (4096, 1024)])
def test_staged_piece_plans_bytes(monkeypatch, head_kib, piece_kib):
    """Staged pipelining with several pieces per batch: small head/tail pieces, multi-block pieces, a head covering
    the whole batch, and batches above one launch's by-value descriptor capacity; B = 1 KiB blocks."""
    monkeypatch.setenv("TC_HEAD_KIB", str(head_kib))
    monkeypatch.setenv("TC_PIECE_KIB", str(piece_kib))
    L, H, D, T, N, S = 1, 1, 64, 4, 600, 400
    for seed in range(3):
        ops = fuzz_script(seed + 77, n_ops=60, n_agents=3, n_classes=2, N=N, max_alloc=150)
        run_script(ops, L, H, D, N, S, "staged", ncls=2, seed=seed + 3, T=T)


def test_unbuffered_ablation_bytes():
    """The Fig. 11 ablation mode (per-offload cudaHostAlloc, no CPU block buffer) moves the same bytes."""
    L, H, D, N, S = 2, 2, 64, 48, 4
    pool0 = content.pool_bytes(4, L, N, 16, H, D)
    o = OraclePool(N, 64, n_classes=2, store=BytesStore(pool0, 64))
    c = tcb.Pool(L, H, D, 16, "bf16", N, device=0, host_slots=S, n_classes=2, unbuffered=True)
    c.fill(4)
    ops = fuzz_script(5, n_ops=80, n_agents=3, n_classes=2, N=N)
    ro, rc = Replayer(o), Replayer(c)
    for i, op in enumerate(ops):
        a, b = ro.step(op), rc.step(op)
        assert a == b, (i, op, a, b)
    c.sync()
    assert np.array_equal(c.kv_tensor().cpu().numpy(), o.store.pool)


@pytest.mark.parametrize("mode", ["direct", "staged", "staged_tile", "direct_tma", "copy"])
def test_batches_above_one_launch_capacity(monkeypatch, mode):
    """A batch of more blocks than one launch's by-value descriptor capacity (2040) is split over several launches:
    offload + upload of 4100 blocks (and a device-tier gather of 4100) against the oracle / numpy."""
    monkeypatch.setenv("TC_PIECE_KIB", "64")        # staged: 2048-block pieces, each above one launch's capacity
    L, H, D, T, N, S = 1, 1, 8, 2, 5000, 4200
    ops = [("agent_add", 0, 0), ("alloc", 0, 4100), ("offload", 0, "all"), ("sync",), ("upload", 0), ("sync",)]
    pool0 = content.pool_bytes(3, L, N, T, H, D)
    o = OraclePool(N, S, max_blocks_per_agent=8192, store=BytesStore(pool0, S))
    c = dev_pool(L, H, D, N, S, mode, max_bpa=8192, seed=3, T=T)
    ro, rc = Replayer(o), Replayer(c)
    for op in ops:
        a, b = ro.step(op), rc.step(op)
        assert a == b and a[0] == 0, op
    c.sync()
    compare_full(o, c, "after 4100-block round trip")
    ids = np.random.default_rng(1).choice(N, size=4100, replace=False).astype(np.int32)
    dst = torch.empty(4100 * c.block_bytes, dtype=torch.uint8, device="cuda:0")
    c.gather_dev(ids, dst.data_ptr())
    torch.cuda.synchronize()
    exp = np.take(o.store.pool, ids, axis=2).transpose(2, 0, 1, 3)
    assert np.array_equal(dst.cpu().numpy().reshape(exp.shape), exp)


@pytest.mark.parametrize("mode", ["staged", "direct", "copy", "staged_tile"])
@pytest.mark.parametrize("gi", [0, 2, 4])
def test_peer_tier_fuzz_bytes(mode, gi):
    """NEXT-2 peer tier (reading C1) with the peer slab on this same GPU (the single-GPU stand-in for a neighbour's
    HBM): tier placement, peer-slot images, pool bytes, tables and counters against the oracle after every sync; the
    host-tier part of each batch still takes `mode`'s path."""
    L, H, D, N, S, T = GEOMS[gi]
    for seed in range(2):
        ops = fuzz_script(seed + 31 * gi, n_ops=90, n_agents=3, n_classes=N_CLASSES, N=N, max_alloc=6)
        o, c = run_script(ops, L, H, D, N, S, mode, seed=seed + 5, T=T, P=max(2, S // 2))
        assert c.stats()["peer_slots"] == max(2, S // 2)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="NEXT-2 across GPUs needs a second GPU (the peer slab in its HBM, reached over NVLink)")
@pytest.mark.parametrize("mode", ["staged", "direct"])
def test_peer_tier_on_second_gpu(mode):
    """NEXT-2 peer tier (reading C1) with the peer slab in GPU 1's HBM: offloads gather straight into the
    neighbour's memory over NVLink (peer access), uploads scatter back from it; pool bytes, peer / host images,
    tables and counters against the oracle after every sync, for fuzz scripts and C2-shaped tc_cycle batches."""
    for gi in (0, 2):
        L, H, D, N, S, T = GEOMS[gi]
        for seed in range(2):
            ops = fuzz_script(seed + 71 * gi, n_ops=90, n_agents=3, n_classes=N_CLASSES, N=N, max_alloc=6)
            o, c = run_script(ops, L, H, D, N, S, mode, seed=seed + 5, T=T, P=max(2, S // 2), peer_dev=1)
            c.close()
    cfg = CONFIGS["c2"].scaled(N=512, host_slots=160, bg_fill=0.3)
    o, c = run_script(build_script(cfg, 10, combined=True), cfg.L, cfg.H, cfg.D, cfg.N, cfg.host_slots(), mode,
                      seed=2, P=96, peer_dev=1)
    assert any(x >= cfg.host_slots() for h in o.handles.values() for x in h.slots)
    c.close()


def test_peer_tier_cycles_mixed_tiers():
    """tc_cycle batches whose offloads split across both tiers (peer slots fill up mid-batch), over C2-shaped
    blocks: bytes and tables against the oracle."""
    cfg = CONFIGS["c2"].scaled(N=512, host_slots=160, bg_fill=0.3)
    ops = build_script(cfg, 10, combined=True)
    L, H, D = cfg.L, cfg.H, cfg.D
    o, c = run_script(ops, L, H, D, cfg.N, cfg.host_slots(), "staged", seed=2, P=96)
    assert any(x >= cfg.host_slots() for h in o.handles.values() for x in h.slots)


def test_c1_many_seeds_auto():
    """C1 geometry, 1000 seeded fuzz scripts through the default AUTO path (staged, with the
    small-batch direct kernel), a tiny staging buffer so ring reuse engages: pool bytes, tables and counters equal
    the oracle's at the end of every script."""
    L, H, D, T, N, S = 1, 2, 64, 16, 64, 16
    for seed in range(1000):
        ops = fuzz_script(seed + 5000, n_ops=40, n_agents=2, n_classes=2, N=N, max_alloc=8, gradual=seed % 4 == 0)
        pool0 = content.pool_bytes(seed, L, N, T, H, D)
        o = OraclePool(N, S, n_classes=2, max_agents=1024, max_blocks_per_agent=4096, store=BytesStore(pool0, S))
        c = tcb.Pool(L, H, D, T, "fp16", N, device=0, host_slots=S, n_classes=2, staging_bytes=4 * 8192)
        c.fill(seed)
        ro, rc = Replayer(o), Replayer(c)
        for i, op in enumerate(ops):
            a, b = ro.step(op), rc.step(op)
            assert a == b, (seed, i, op, a, b)
        c.sync()
        o.sync()
        compare_full(o, c, f"seed {seed}")
        c.close()


def test_head_shards_concatenate_to_unsharded_run():
    """SURVEY.md §4 item 6 (sharding without 8 GPUs): G = 4 head-shard pools and one unsharded pool on this GPU run
    the same script; the shards' pools, concatenated along the head axis, equal the unsharded pool byte for byte,
    and all tables agree (the multi-GPU layout is correct by construction)."""
    L, H, D, T, N, S, G = 3, 8, 64, 16, 48, 24, 4
    ops = fuzz_script(77, n_ops=120, n_agents=3, n_classes=2, N=N, max_alloc=6)
    pools = []
    for r, w in [(0, 1)] + [(r, G) for r in range(G)]:
        c = tcb.Pool(L, H, D, T, "bf16", N, device=0, shard_rank=r, shard_world=w, host_slots=S, n_classes=2)
        c.fill(13)
        tr = Replayer(c).run(ops)
        c.sync()
        pools.append((c, tr))
    full = pools[0][0].kv_tensor().cpu().numpy().reshape(L, 2, N, T, H, D * 2)
    shards = [p.kv_tensor().cpu().numpy().reshape(L, 2, N, T, H // G, D * 2) for p, _ in pools[1:]]
    assert np.array_equal(np.concatenate(shards, axis=4), full)
    for p, tr in pools[1:]:
        assert tr == pools[0][1]
        for a in range(3):
            assert p.block_table(a) == pools[0][0].block_table(a)
    for p, _ in pools:
        p.close()


def test_per_call_trace_completion_stamps():
    """On the GPU the trace's t_done comes from a host callback behind the batch's work: after tc_sync every record
    has t_call <= t_enqueued <= t_done."""
    L, H, D, N, S = 2, 2, 64, 64, 32
    c = dev_pool(L, H, D, N, S, "staged")
    c.trace(64)
    r = Replayer(c)
    r.run(fuzz_script(3, n_ops=60, n_agents=3, n_classes=2, N=N, max_alloc=6))
    c.sync()
    recs = c.trace_read()
    assert recs and {x["op"] for x in recs} == {"offload", "upload"}
    for x in recs:
        assert 0 < x["t_call_ns"] <= x["t_enqueued_ns"] <= x["t_done_ns"], x
    c.close()


def test_c_abi_demo_on_device(tmp_path):
    """examples/c_abi_demo.c (plain C, no Python in the loop) on cuda:0: real KV bytes moved through the C ABI."""
    import os
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(tcb.LIB_PATH)
    exe = tmp_path / "c_abi_demo"
    r = subprocess.run([gcc, "-std=c11", "-I", os.path.join(root, "include"), os.path.join(root, "examples",
                        "c_abi_demo.c"), "-L", libdir, "-ltokencake", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe), "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("ok: 48 blocks")


def test_calibrate_keeps_pool_and_sets_auto():
    """tc_calibrate times the four {DIRECT, STAGED} cycle combinations on this box; the pool's bytes, tables and
    counters are unchanged afterwards, AUTO directions take the chosen modes, and a later script still matches the
    oracle byte for byte."""
    L, H, D, N, S = 4, 4, 128, 96, 64
    pool0 = content.pool_bytes(21, L, N, 16, H, D)
    c = tcb.Pool(L, H, D, 16, "bf16", N, device=0, host_slots=S, n_classes=2)
    c.fill(21)
    before = c.stats()
    cal = c.calibrate(8 << 20)
    assert cal["probe_bytes"] > 0 and all(v > 0 for v in cal["gbs"].values())
    # the measured small-batch crossover: a whole number of blocks (0 = DIRECT never faster), at most 64 blocks
    for v in cal["direct_max_bytes"].values():
        assert v % c.block_bytes == 0 and 0 <= v <= 64 * c.block_bytes
    assert np.array_equal(c.kv_tensor().cpu().numpy(), pool0)
    after = c.stats()
    assert {k: before[k] for k in ("free", "alloc", "host_free", "host_used")} == \
        {k: after[k] for k in ("free", "alloc", "host_free", "host_used")}
    names = {tcb.XFER_DIRECT: "direct", tcb.XFER_STAGED: "staged"}
    assert (names[after["xfer_d2h"]], names[after["xfer_h2d"]]) == (cal["d2h"], cal["h2d"])
    o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S))
    ro, rc = Replayer(o), Replayer(c)
    for op in fuzz_script(8, n_ops=80, n_agents=3, n_classes=2, N=N, max_alloc=8):
        assert ro.step(op) == rc.step(op), op
    c.sync()
    o.sync()
    compare_full(o, c, "after calibrate")
    c.close()


def test_xfer_model_calibrates_from_measured_transfers():
    """NEXT-3's T_transfer comes from this pool's own measured transfers (tc_xfer_model_measure): after offloads and
    uploads of 1..64 blocks the fitted line has a per-block cost between a 10 and a 100 GB/s link and a small
    non-negative fixed cost, and it predicts a 64-block round trip within 35 % of the measured one."""
    import time
    from paper_2510_18586_b200 import sched
    L, H, D, N, S = 28, 4, 128, 512, 256                    # C2-shaped 896 KiB blocks
    c = tcb.Pool(L, H, D, 16, "bf16", N, device=0, host_slots=S, n_classes=2, xfer_d2h=tcb.XFER_STAGED,
                 xfer_h2d=tcb.XFER_STAGED)
    c.fill(5)
    c.timing(1)
    c.agent_add(0, 0)
    c.alloc(0, 64)
    for n in (1, 4, 16, 64, 1, 4, 16, 64):
        h = c.offload(0, c.block_table(0)[:n])
        c.sync()
        c.upload(h)
        c.sync()
    m = sched.xfer_model_measure(c)
    B = c.block_bytes
    for k in ("offload_ms_per_block", "upload_ms_per_block"):
        assert B / 100e9 * 1e3 < m[k] < B / 10e9 * 1e3, m
    assert 0.0 <= m["fixed_ms"] < 0.5, m
    t0 = time.perf_counter()
    h = c.offload(0, c.block_table(0))
    c.wait(h)
    c.sync()
    c.upload(h)
    c.wait(h)
    wall_ms = (time.perf_counter() - t0) * 1e3
    c.sync()
    pred = sched.transfer_ms(64, m["offload_ms_per_block"], m["upload_ms_per_block"], m["fixed_ms"])
    assert 0.65 * wall_ms < pred < 1.35 * wall_ms, (pred, wall_ms, m)
    c.close()


def test_time_scheduler_runtime_bytes():
    """The native Time Scheduler (tc_ts_*) driving a device pool through a random event stream, against the oracle
    event machine on a byte-level pool: identical decisions and handles, and after the stream the KV bytes, tables
    and counters match exactly."""
    from oracle.time_scheduler import TimeSchedulerOracle
    from paper_2510_18586_b200 import sched
    L, H, D, N, S = 2, 2, 64, 160, 48
    rng = np.random.default_rng(4)
    pool0 = content.pool_bytes(6, L, N, 16, H, D)
    o = OraclePool(N, S, n_classes=2, store=BytesStore(pool0, S))
    c = dev_pool(L, H, D, N, S, "staged", ncls=2, seed=6)
    for a in range(5):
        n = int(rng.integers(2, 20))
        o.agent_add(a, a % 2)
        c.agent_add(a, a % 2)
        assert o.alloc(a, n) == list(c.alloc(a, n))
    prm = dict(v_tokens_per_s=4000.0, tick_ms=5.0, reserve_cycles=2, lead_ms=10.0, cold_start_ms=60.0)
    model = {"offload_ms_per_block": 0.1, "upload_ms_per_block": 0.1, "fixed_ms": 0.0}
    to = TimeSchedulerOracle(o, offload_ms_per_block=0.1, upload_ms_per_block=0.1, **prm)
    tc = sched.TimeScheduler(c, model=model, **prm)
    now = 0.0
    for _ in range(300):
        now += float(rng.integers(1, 12))
        a = int(rng.integers(0, 5))
        if a in to.stalled():
            if rng.random() < 0.4:
                assert to.call_finish(a, now) == tc.call_finish(a, now)
        else:
            w = [float(x) for x in rng.integers(1, 300, size=2)]
            x, y = to.call_start(a, 0, now, waiting=w), tc.call_start(a, 0, now, waiting=w)
            assert (x["offload"], x["handle"]) == (y["offload"], y["handle"])
        assert to.tick(now) == tc.tick(now)
        if rng.random() < 0.2:
            o.sync()
            c.sync()
    for a in list(to.stalled()):
        assert to.call_finish(a, now + 1000.0) == tc.call_finish(a, now + 1000.0)
    o.sync()
    c.sync()
    compare_full(o, c, "after the time-scheduler stream")
    tc.close()
    c.close()


@pytest.mark.parametrize("mode,P", [("auto", 0), ("staged_tile", 0), ("direct", 0), ("staged", 6)])
def test_long_random_stream_with_invariant_checks(monkeypatch, mode, P):
    """Stress: 8,000 random ops (gradual reservation on, uploads issued before their offloads finished, ring reuse
    through a 3-block staging buffer) on one pool with TC_CHECK=1 (SPEC invariants re-derived after every call);
    the whole pool, every table and every counter equal the oracle's at every sync."""
    monkeypatch.setenv("TC_CHECK", "1")
    L, H, D, N, S, T = 3, 2, 64, 50, 20, 16
    ops = fuzz_script(4242 + P, n_ops=8000, n_agents=4, n_classes=2, N=N, max_alloc=6, gradual=True)
    run_script(ops, L, H, D, N, S, mode, ncls=2, seed=9, staging=3 * 2 * L * T * H * D * 2, T=T, P=P)


@pytest.mark.parametrize("mode", ["auto", "staged", "direct", "staged_tile"])
def test_retire_without_drain_bytes(mode):
    """Reading A8' on the GPU: tc_retire returns last epoch's blocks and slots while this epoch's transfers are
    still streaming; the next transfers reuse them.  Whole pool, host images, tables and counters equal the oracle
    after every sync, on scripts that retire often and sync rarely."""
    L, H, D, N, S, T = 4, 4, 128, 40, 24, 16
    for seed in range(3):
        ops = [op for op in fuzz_script(seed + 90, n_ops=150, n_agents=3, n_classes=2, N=N, max_alloc=6,
                                        gradual=True, retire=True) if op[0] != "sync" or seed == 0]
        ops.append(("sync",))
        run_script(ops, L, H, D, N, S, mode, ncls=2, seed=seed + 11, T=T)


@pytest.mark.parametrize("halves", ["0", "1"])
def test_staging_halves_on_off_bytes(halves, monkeypatch):
    """The staged path with and without the cross-batch staging halves (TC_STAGING_HALVES, read at pool creation):
    a 5-block staging buffer mixes half-buffer batches (1-2 blocks, alternating halves), whole-buffer batches and ring
    batches in one script; whole pool, host images, tables and counters equal the oracle after every sync."""
    monkeypatch.setenv("TC_STAGING_HALVES", halves)
    L, H, D, N, S, T = 4, 4, 128, 48, 32, 16
    for seed in range(3):
        ops = fuzz_script(seed + 290, n_ops=160, n_agents=4, n_classes=2, N=N, max_alloc=7, retire=True,
                          lags=(1, 2, 3))
        run_script(ops, L, H, D, N, S, "staged", ncls=2, seed=seed + 31, staging=5 * 2 * L * T * H * D * 2, T=T)


@pytest.mark.parametrize("mode", ["auto", "staged"])
def test_retire_lag_bytes(mode):
    """Reading A8'' on the GPU: tc_retire_lag with lags 1-3 (and the refused 0) on scripts that retire often and sync
    rarely; whole pool, host images, tables and counters equal the oracle after every sync."""
    L, H, D, N, S, T = 4, 4, 128, 40, 24, 16
    for seed in range(3):
        ops = [op for op in fuzz_script(seed + 190, n_ops=150, n_agents=3, n_classes=2, N=N, max_alloc=6,
                                        gradual=True, retire=True, lags=(0, 1, 2, 3, 3))
               if op[0] != "sync" or seed == 0]
        ops.append(("sync",))
        run_script(ops, L, H, D, N, S, mode, ncls=2, seed=seed + 21, T=T)


def test_retire_keeps_this_epochs_transfer_running():
    """tc_retire does not wait for work enqueued after the previous retirement point: with a large offload in
    flight, retire() leaves its blocks pending (and normally returns while it still streams); a second retire
    then returns them."""
    L, H, D, N, S = 28, 4, 128, 1024, 512             # C2-shaped blocks; 400 blocks ~ 360 MB ~ 7 ms over PCIe
    c = tcb.Pool(L, H, D, 16, "bf16", N, device=0, host_slots=S, xfer_d2h=tcb.XFER_STAGED, xfer_h2d=tcb.XFER_STAGED)
    c.fill(3)
    c.agent_add(0, 0)
    c.alloc(0, 400)
    c.retire()                                        # a retirement point before the offload
    h = c.offload(0, c.block_table(0))
    c.retire()                                        # must not drain the offload enqueued after the last point
    busy = not c.query(h)                             # normally still streaming (~7 ms over PCIe)
    assert c.stats()["pending"] == 400                # not retired either way: enqueued after the previous point
    print("offload still in flight after retire():", busy)
    c.retire()
    assert c.stats()["pending"] == 0 and c.stats()["free"] == N
    c.close()
