"""Full-size parity (SURVEY.md §8(c) "Oracle-at-scale"): the BASELINE configs C2-C5 at their full pool
sizes, in bench.py's launch configuration (AUTO transfer modes, tc_cycle per scheduling cycle, the retirement rule
bench.py picks for the config), replayed on the GPU pool and on the oracle's provenance store.  At the end:

* every block table (host mirror and device table) and every counter equal the oracle's;
* the WHOLE device pool, streamed in pieces of at most 1 GiB, equals the content generator evaluated at the oracle's
  provenance (prov[b] = the original block whose bytes physical block b must hold) — every chunk of every block an
  upload wrote, and every other block untouched;
* every live handle's host image (each offloaded block shard in its pinned slot, read through tc_handle_host) equals
  the generator at the oracle's host provenance for that handle's block.

The expected bytes come from tests/gen_torch.py (torch int64 ops, no libtokencake kernel), pinned first against
workloads/content.py on sampled chunks of the same pool geometry.
"""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2510_18586_b200 as tcb  # noqa: E402
from gen_torch import block_words  # noqa: E402
from oracle import OraclePool, ProvStore  # noqa: E402
from oracle.pool import OFFLOADED  # noqa: E402
from workloads import content  # noqa: E402
from workloads.configs import CONFIGS  # noqa: E402
from workloads.replay import Replayer  # noqa: E402
from workloads.scripts import build_script  # noqa: E402

PIECE = 1 << 30


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def pin_generator(cfg, rank, world, provs):
    """gen_torch on the device == workloads/content.py on a few chunks of this geometry (before trusting it)."""
    got = block_words(cfg.seed, torch.tensor(provs, device="cuda:0"), cfg.L, cfg.N, cfg.T, cfg.H, cfg.D, rank,
                      world).cpu().numpy().view(np.uint8)
    for i, b in enumerate(provs):
        for l, kv in ((0, 0), (cfg.L - 1, 1), (cfg.L // 2, 0)):
            exp = content.chunk_bytes(cfg.seed, l, kv, int(b), cfg.N, cfg.T, cfg.H, cfg.D, rank=rank, world=world)
            assert np.array_equal(got[l, kv, i], exp), (cfg.name, b, l, kv)


def compare_whole_pool(c, cfg, prov, rank, world):
    kv64 = c.kv_tensor().view(torch.int64)                 # [L][2][N][C/8]
    B = c.block_bytes
    step = max(1, PIECE // B)
    prov_d = torch.from_numpy(np.asarray(prov, dtype=np.int64)).cuda()
    for b0 in range(0, cfg.N, step):
        b1 = min(cfg.N, b0 + step)
        exp = block_words(cfg.seed, prov_d[b0:b1], cfg.L, cfg.N, cfg.T, cfg.H, cfg.D, rank, world)
        if not torch.equal(kv64[:, :, b0:b1], exp):
            bad = (kv64[:, :, b0:b1] != exp).any(dim=3).nonzero()[:5].tolist()
            raise AssertionError(f"{cfg.name} G={world} r={rank}: pool bytes differ in blocks [{b0}, {b1}): "
                                 f"(layer, kv, block-b0) {bad}")
        del exp
    torch.cuda.synchronize()


def compare_live_host_images(c, o, cfg, rank, world):
    """Every block of every live handle: the library's pinned slot image vs the generator at the oracle's host
    provenance of the same (handle, i)."""
    B = c.block_bytes
    items = [(h, i, int(o.store.host_prov[s])) for h, hd in o.handles.items() if hd.state == OFFLOADED
             for i, s in enumerate(hd.slots)]
    assert items, "no live handle at the end of the script"
    step = max(1, PIECE // B)
    ptr = ctypes.c_void_p()
    for k0 in range(0, len(items), step):
        chunk = items[k0:k0 + step]
        got = torch.empty((len(chunk), B), dtype=torch.uint8, device="cuda:0")
        for j, (h, i, _) in enumerate(chunk):
            c.wait(h)
            assert tcb.lib.tc_handle_host(c._h, h, i, ctypes.byref(ptr)) == 0
            host = torch.frombuffer((ctypes.c_uint8 * B).from_address(ptr.value), dtype=torch.uint8)
            got[j].copy_(host)
        exp = block_words(cfg.seed, torch.tensor([p for _, _, p in chunk], device="cuda:0"), cfg.L, cfg.N, cfg.T,
                          cfg.H, cfg.D, rank, world)               # [L][2][n][Cw]
        exp = exp.permute(2, 0, 1, 3).reshape(len(chunk), -1)      # host slot layout [L][2][C] per block
        if not torch.equal(got.view(torch.int64).view(len(chunk), -1), exp):
            bad = [chunk[j][:2] for j in (got.view(torch.int64).view(len(chunk), -1) != exp).any(1).nonzero()
                   .flatten()[:5].tolist()]
            raise AssertionError(f"{cfg.name} G={world} r={rank}: host images differ for (handle, i) {bad}")
    return len(items)


def run_full(name, world, rank, lag, cycles):
    torch.cuda.empty_cache()
    cfg = CONFIGS[name]
    S = cfg.host_slots()
    ops = build_script(cfg, cycles, combined=True)
    n_setup = next(i for i, op in enumerate(ops) if op[0] == "cycle")
    if lag:                                # bench.py's retire-each loop: tc_cycle (retried once after a sync if
        rt = ("retire",) if lag == 1 else ("retire", lag)          # refused) + tc_retire_lag(lag)
        ops = ops[:n_setup] + [rt if op[0] == "sync" else ("cycle_r",) + op[1:] if op[0] == "cycle" else op
                               for op in ops[n_setup:]]
    ops.append(("sync",))
    o = OraclePool(cfg.N, S, max_agents=1024, max_blocks_per_agent=cfg.max_blocks_per_agent,
                   store=ProvStore(cfg.N, S))
    c = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, cfg.N, device=0, shard_rank=rank, shard_world=world,
                 host_slots=S, max_agents=1024, max_blocks_per_agent=cfg.max_blocks_per_agent)
    c.fill(cfg.seed)
    pin_generator(cfg, rank, world, [0, cfg.N - 1, cfg.N // 3])
    ro, rc = Replayer(o), Replayer(c)
    moved = 0
    for i, op in enumerate(ops):
        a, b = ro.step(op), rc.step(op)
        assert a == b, (name, i, op)
        assert a[0] == 0, (name, i, op)
        if op[0] in ("cycle", "cycle_r") and a[1]:
            moved += sum(len(x) for x in a[1][0])
    c.sync()
    o.sync()
    assert moved > 0
    tab = c.table_tensor().cpu().numpy()
    for ag_id, ag in o.agents.items():
        assert c.block_table(ag_id) == ag.table, (name, ag_id)
        assert tab[ag_id, :len(ag.table)].tolist() == ag.table, (name, ag_id)
    so, sc = o.stats(), c.stats()
    for k in ("free", "alloc", "pending", "host_free", "host_used", "reserved", "claimed"):
        assert so[k] == sc[k], (name, k)
    assert (o.store.prov != np.arange(cfg.N)).any()           # uploads really moved content around
    compare_whole_pool(c, cfg, o.store.prov, rank, world)
    n_img = compare_live_host_images(c, o, cfg, rank, world)
    c.close()
    return moved, n_img


# (config, head shards G, rank, retire lag (0 = drained with tc_sync every cycle), cycles).  bench.py's loop is
# retire-each with the retire ladder for every config (lag 4 C2, 1 otherwise); two drained cases keep that loop covered.
# C3 runs the driver's default bench length (priming + 5 warm-up + 20 timed cycles) and more.
CASES = [("c2", 1, 0, 4, 40), ("c3", 1, 0, 1, 30), ("c4", 1, 0, 1, 8), ("c4", 2, 0, 1, 8), ("c4", 2, 1, 0, 8),
         ("c4", 4, 0, 1, 8), ("c4", 4, 3, 1, 8), ("c4", 8, 0, 1, 8), ("c4", 8, 7, 0, 8), ("c5", 8, 0, 1, 8),
         ("c5", 8, 7, 1, 8)]


@pytest.mark.parametrize("name,world,rank,lag,cycles", CASES)
def test_full_size_whole_pool_and_host_images(name, world, rank, lag, cycles):
    moved, n_img = run_full(name, world, rank, lag, cycles)
    print(f"{name} G={world} rank={rank} lag={lag}: {moved} blocks uploaded, {n_img} live host images checked")
