"""The native Time Scheduler (tc_ts_* in csrc/sched.cpp) against the oracle event machine
(oracle/time_scheduler.py): identical decisions, plans, handles, upload ticks, forecasts, pool tables and counters on
random event streams (metadata-only pools, CPU), the SPEC worked examples through the C ABI, and TC_CHECK's
invariants after every event."""
import numpy as np
import pytest

import paper_2510_18586_b200 as tcb
from oracle import OracleError, OraclePool, ProvStore
from oracle.time_scheduler import TimeSchedulerOracle
from paper_2510_18586_b200 import sched

KEYS = ("offload", "match", "status", "t_fc", "t_transfer", "upload_start", "reservation_start", "handle")


def both(N, S, agents, params, ncls=2):
    o = OraclePool(N, S, n_classes=ncls, store=ProvStore(N, S))
    c = tcb.Pool(1, 2, 64, 16, "fp16", N, device=-1, host_slots=S, n_classes=ncls, max_blocks_per_agent=8192)
    for a, (cls, n) in agents.items():
        o.agent_add(a, cls)
        c.agent_add(a, cls)
        assert o.alloc(a, n) == list(c.alloc(a, n))
    model = {"offload_ms_per_block": params["offload_ms_per_block"],
             "upload_ms_per_block": params["upload_ms_per_block"], "fixed_ms": params.get("fixed_ms", 0.0)}
    rest = {k: v for k, v in params.items() if k not in model}
    return o, c, TimeSchedulerOracle(o, **params), sched.TimeScheduler(c, model=model, **rest)


def run(fn, *a, **kw):
    try:
        return 0, fn(*a, **kw)
    except (OracleError, tcb.TcError) as e:
        return e.status, None


def same_decision(x, y):
    assert x[0] == y[0], (x, y)
    if x[0] == 0:
        for k in KEYS:
            assert x[1][k] == pytest.approx(y[1][k], rel=1e-12, abs=1e-9), (k, x, y)


def test_spec_examples_through_capi():
    params = dict(offload_ms_per_block=30.0 / 4096, upload_ms_per_block=30.0 / 4096, v_tokens_per_s=2000.0,
                  lead_ms=100.0, tick_ms=10.0, reserve_cycles=4)
    o, c, to, tc = both(9000, 4096, {0: (0, 4096)}, params)
    d = tc.call_start(0, 1, 0.0, t_req=5000.0, waiting=[8000.0])
    assert d["offload"] and d["upload_start"] == pytest.approx(4970.0) and d["t_transfer"] == pytest.approx(60.0)
    issued = [t for t in range(10, 5001, 10) if tc.tick(float(t))]
    assert issued == [4970]
    assert tc.call_finish(0, 5000.0) == d["handle"]
    assert tc.forecast(0, 1) == (5000.0, 1)
    assert all(b >= 0 for b in c.block_table(0))
    d = tc.call_start(0, 1, 6000.0, t_req=None, waiting=[8000.0])
    assert d["t_fc"] == pytest.approx(5000.0)                    # history, no hint -> t_hist
    h = tc.call_finish(0, 7000.0)                                  # early: immediate upload
    assert h == d["handle"] and all(b >= 0 for b in c.block_table(0))
    with pytest.raises(tcb.TcError) as e:
        tc.call_finish(0, 8000.0)
    assert e.value.status == tcb.E_INVAL


@pytest.mark.parametrize("seed", range(12))
def test_random_event_streams_match_oracle(seed, monkeypatch):
    monkeypatch.setenv("TC_CHECK", "1")
    rng = np.random.default_rng(seed)
    N, S = 500, int(rng.choice([60, 200]))
    agents = {a: (a % 2, int(rng.integers(1, 50))) for a in range(8)}
    params = dict(offload_ms_per_block=float(rng.choice([0.05, 0.3])), upload_ms_per_block=0.2,
                  fixed_ms=float(rng.choice([0.0, 1.5])), v_tokens_per_s=float(rng.choice([500, 5000])),
                  tick_ms=5.0, reserve_cycles=int(rng.choice([0, 3])), lead_ms=20.0, cold_start_ms=50.0,
                  alpha=float(rng.choice([0.3, 0.5])), beta=0.5)
    o, c, to, tc = both(N, S, agents, params)
    now = 0.0
    for step in range(800):
        now += float(rng.integers(1, 15))
        a = int(rng.integers(0, 9))                       # agent 8 does not exist: INVAL on both sides
        r = rng.random()
        if r < 0.45:
            lab = int(rng.integers(0, 3))
            t_req = None if rng.random() < 0.5 else float(rng.integers(10, 400))
            w = list(map(float, rng.integers(1, 600, size=int(rng.integers(0, 4)))))
            same_decision(run(to.call_start, a, lab, now, t_req, w), run(tc.call_start, a, lab, now, t_req, w))
        elif r < 0.75:
            x, y = run(to.call_finish, a, now), run(tc.call_finish, a, now)
            assert x == y, (step, x, y)
        else:
            assert run(to.tick, now) == run(tc.tick, now), step
        if rng.random() < 0.15:
            o.sync()
            c.sync()
        for ag in agents:
            assert o.block_table(ag) == c.block_table(ag), (step, ag)
        so, sc = o.stats(), c.stats()
        for k in ("free", "alloc", "pending", "reserved_blocks", "host_free", "host_used"):
            assert so[k] == sc[k], (step, k)
    for cls in (0, 1):
        for lab in range(3):
            x, y = to.forecast(cls, lab), tc.forecast(cls, lab)
            assert x[1] == y[1] and (x[0] is None or x[0] == pytest.approx(y[0]))
