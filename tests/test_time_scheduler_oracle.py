"""Pins of the Time-Scheduler event machine oracle (oracle/time_scheduler.py) to SPEC.md time_scheduler's worked
examples and its invariants, on a byte-less pool."""
import numpy as np
import pytest

from oracle import OraclePool, ProvStore
from oracle.pool import E_INVAL, E_NOHOST, OFFLOADED, UPLOADED
from oracle.time_scheduler import TimeSchedulerOracle

SPEC_MODEL = dict(offload_ms_per_block=30.0 / 4096, upload_ms_per_block=30.0 / 4096)   # 60 ms / 4096 RT


def machine(n_blocks=4096, slots=4096, N=9000, **kw):
    pool = OraclePool(N, slots, store=ProvStore(N, slots))
    pool.agent_add(0, 0)
    pool.alloc(0, n_blocks)
    params = dict(SPEC_MODEL, v_tokens_per_s=2000.0, lead_ms=100.0, tick_ms=10.0, reserve_cycles=4)
    params.update(kw)
    return pool, TimeSchedulerOracle(pool, **params)


def test_plan_example_s267_and_offload_example_s259():
    """call_start at t=0 with t_final = 5000 (hint, no history), upload 30 ms, lead 100 ms -> upload_start 4970,
    reservation deadline 4870; T_fc 5000, T_transfer 60, v 2000 tok/s -> N_capacity 9880, an 8000-token
    waiting request -> offload, matched."""
    pool, ts = machine()
    d = ts.call_start(0, label=1, now=0.0, t_req=5000.0, waiting=[8000.0])
    assert d["offload"] and d["match"] == 0 and d["status"] == 0
    assert d["t_fc"] == pytest.approx(5000.0) and d["t_transfer"] == pytest.approx(60.0)
    assert d["upload_start"] == pytest.approx(4970.0)
    assert d["reservation_start"] == pytest.approx(4870.0 - 4 * 10.0)
    assert pool.block_table(0) == [-1] * 4096 and pool.handles[d["handle"]].state == OFFLOADED


def test_retain_example_s258():
    """T_fc = 100 ms, 4096 blocks (T_transfer 60 ms), v = 1000 tok/s -> 40-token capacity; smallest waiting request
    4000 tokens -> retain; the call's finish resumes at once with the blocks still on the GPU."""
    pool, ts = machine(v_tokens_per_s=1000.0)
    d = ts.call_start(0, 1, 0.0, t_req=100.0, waiting=[4000.0])
    assert not d["offload"] and d["handle"] == 0
    assert ts.call_finish(0, 100.0) == 0
    assert all(b >= 0 for b in pool.block_table(0))


def test_empty_queue_retains():
    pool, ts = machine()
    assert not ts.call_start(0, 1, 0.0, t_req=5000.0, waiting=[])["offload"]


def test_early_finish_uploads_immediately():
    """Finish at t = 3000 < upload_start 4970: immediate upload; the handle is returned to wait on."""
    pool, ts = machine()
    d = ts.call_start(0, 1, 0.0, t_req=5000.0, waiting=[8000.0])
    for t in range(10, 3000, 10):
        assert ts.tick(float(t)) == 0
    h = ts.call_finish(0, 3000.0)
    assert h == d["handle"] and pool.handles[h].state == UPLOADED
    assert all(b >= 0 for b in pool.block_table(0))


def test_on_time_finish_finds_the_upload_issued_with_its_reservation():
    """Ticks: the gradual reservation starts reserve_cycles ticks before its deadline and holds all 4096 blocks by
    then; the upload is issued at upload_start (4970) from the reserved blocks; the finish at the predicted time
    adds no upload of its own."""
    pool, ts = machine()
    d = ts.call_start(0, 1, 0.0, t_req=5000.0, waiting=[8000.0])
    h = d["handle"]
    issued_at = None
    for t in range(10, 5001, 10):
        if ts.tick(float(t)) and issued_at is None:
            issued_at = t
        if t == 4870:
            assert len(pool.handles[h].resv) == 4096          # fully reserved by the deadline
    assert issued_at == 4970
    assert pool.handles[h].state == UPLOADED
    assert ts.call_finish(0, 5000.0) == h


def test_nohost_refusal_retains():
    pool, ts = machine(slots=100)
    d = ts.call_start(0, 1, 0.0, t_req=5000.0, waiting=[8000.0])
    assert not d["offload"] and d["status"] == E_NOHOST
    assert all(b >= 0 for b in pool.block_table(0))
    assert ts.call_finish(0, 5000.0) == 0


def test_ewma_feedback_and_convergence():
    """First observation sets t_hist; feeding a constant duration drives the forecast to it."""
    pool, ts = machine(n_blocks=8, cold_start_ms=100.0)
    ts.call_start(0, 7, 0.0, waiting=[1.0])
    ts.call_finish(0, 800.0)
    assert ts.forecast(0, 7) == (800.0, 1)
    now = 1000.0
    for _ in range(12):
        ts.call_start(0, 7, now, waiting=[1.0])
        for t in np.arange(now + 10, now + 300, 10):
            ts.tick(float(t))
        ts.call_finish(0, now + 300.0)
        now += 1000.0
    t_hist, n = ts.forecast(0, 7)
    assert n == 13 and abs(t_hist - 300.0) < 500.0 * 0.5 ** 12 + 1e-9


def test_errors():
    pool, ts = machine(n_blocks=4)
    with pytest.raises(Exception) as e:
        ts.call_finish(0, 1.0)
    assert e.value.status == E_INVAL
    ts.call_start(0, 1, 0.0, waiting=[1.0])
    with pytest.raises(Exception) as e:
        ts.call_start(0, 1, 1.0)
    assert e.value.status == E_INVAL
    with pytest.raises(Exception) as e:
        ts.call_start(5, 1, 1.0)
    assert e.value.status == E_INVAL


@pytest.mark.parametrize("seed", range(6))
def test_safety_random_event_streams(seed):
    """a request never resumes while any of its blocks are host-resident with no upload issued — after every
    call_finish the agent's table is all on-GPU ids (the returned handle's upload has been issued)."""
    rng = np.random.default_rng(seed)
    N, S = 400, 120
    pool = OraclePool(N, S, n_classes=2, store=ProvStore(N, S))
    for a in range(6):
        pool.agent_add(a, a % 2)
        pool.alloc(a, int(rng.integers(1, 40)))
    ts = TimeSchedulerOracle(pool, v_tokens_per_s=5000.0, offload_ms_per_block=0.2, upload_ms_per_block=0.2,
                             tick_ms=5.0, reserve_cycles=3, lead_ms=20.0)
    now = 0.0
    for _ in range(600):
        now += float(rng.integers(1, 20))
        a = int(rng.integers(0, 6))
        if a in ts.stalled():
            if rng.random() < 0.3:
                ts.call_finish(a, now)
                assert all(b >= 0 for b in pool.block_table(a))
        else:
            ts.call_start(a, int(rng.integers(0, 3)), now, waiting=list(rng.integers(1, 400, size=3)))
        ts.tick(now)
        if rng.random() < 0.2:
            pool.sync()
