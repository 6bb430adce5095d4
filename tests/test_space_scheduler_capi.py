"""The native Space-Scheduler update (tc_ss_* in csrc/sched.cpp) against oracle/space_scheduler.py: identical scores,
critical sets, Phase-1 ratios and quotas on random pools and waiting queues, and identical allocator behaviour
(statuses, ids, counters) under the quotas it applied; the SPEC worked examples through the C ABI."""
import numpy as np
import pytest

import paper_2510_18586_b200 as tcb
from oracle import OraclePool, ProvStore
from oracle.space_scheduler import SpaceSchedulerOracle
from paper_2510_18586_b200 import sched
from workloads.replay import Replayer
from workloads.scripts import fuzz_script


def test_spec_examples_through_capi():
    p = tcb.Pool(1, 2, 64, 16, "fp16", 1000, device=-1, host_slots=8, n_classes=4)
    for a, (c, k) in enumerate([(0, 100), (1, 100), (3, 700)]):
        p.agent_add(a, c)
        p.alloc(a, k)
    ss = sched.SpaceScheduler(p, critical_ratio=0.5, initial_reserve_ratio=0.10)
    out = ss.update([3.0, 1.0, 0.0, 0.0])
    assert out["ratio"] == pytest.approx(0.15) and out["reserve"] == [63, 26, 0, 0]
    assert p.stats()["reserved"] == [63, 26, 0, 0]
    assert ss.critical_inversion(0, 1) and not ss.critical_inversion(2, 3)
    with pytest.raises(tcb.TcError):
        ss.update([0.0] * 4, [(7, 1.0, 5.0)])


@pytest.mark.parametrize("seed", range(15))
def test_random_updates_match_oracle(seed):
    rng = np.random.default_rng(seed)
    N, S, ncls = int(rng.choice([64, 200])), 32, 4
    o = OraclePool(N, S, n_classes=ncls, store=ProvStore(N, S))
    c = tcb.Pool(1, 2, 64, 16, "fp16", N, device=-1, host_slots=S, n_classes=ncls)
    kw = dict(critical_ratio=float(rng.choice([0.25, 0.5, 1.0])), initial_reserve_ratio=float(rng.choice([0, 0.2])),
              gpu_usage_high=0.6, gpu_usage_low=0.3, adjustment_step=0.1)
    so, sc = SpaceSchedulerOracle(o, **kw), sched.SpaceScheduler(c, **kw)
    ro, rc = Replayer(o), Replayer(c)
    ops = fuzz_script(300 + seed, n_ops=240, n_agents=5, n_classes=ncls, N=N, max_alloc=8)
    for i, op in enumerate(ops):
        if op[0] == "reserve":
            continue                                      # quotas come from the Space Scheduler here
        assert ro.step(op) == rc.step(op), (i, op)
        if i % 20 == 0:
            st = list(map(float, rng.integers(0, 10, size=ncls)))
            w = [(int(rng.integers(0, ncls)), float(rng.integers(0, 500)), float(rng.integers(1, 4000)))
                 for _ in range(int(rng.integers(0, 6)))]
            a, b = so.update(st, w), sc.update(st, w)
            assert a["reserve"] == b["reserve"] and a["critical"] == b["critical"], (i, a, b)
            assert a["ratio"] == pytest.approx(b["ratio"]) and a["scores"] == pytest.approx(b["scores"])
            x, y = o.stats(), c.stats()
            assert x["reserved"] == y["reserved"] and x["claimed"] == y["claimed"]
