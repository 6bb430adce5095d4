"""Pins of the Space-Scheduler update oracle (oracle/space_scheduler.py) to SPEC.md space_scheduler's worked
examples and invariants, on a byte-less pool whose own usage drives Alg. 2."""
import pytest

from oracle import OraclePool, ProvStore
from oracle.space_scheduler import SpaceSchedulerOracle


def pool_with_usage(total, per_class, n_classes=4, N=1000):
    p = OraclePool(N, 8, n_classes=n_classes, store=ProvStore(N, 8))
    a = 0
    for c, k in per_class.items():
        p.agent_add(a, c)
        if k:
            p.alloc(a, k)
        a += 1
    rest = total - sum(per_class.values())
    if rest:
        p.agent_add(a, n_classes - 1)
        p.alloc(a, rest)
    return p


def test_phase1_and_phase2_examples_s356_s357():
    """total 1000, usage 900 >= 0.85, prior ratio 0.10 -> 0.15, R_total 150; critical X (score 3, usage
    100) and Y (score 1, usage 100) -> X 63, Y 26 blocks."""
    p = pool_with_usage(900, {0: 100, 1: 100})
    ss = SpaceSchedulerOracle(p, critical_ratio=0.5, initial_reserve_ratio=0.10)
    out = ss.update([3.0, 1.0, 0.0, 0.0], [])
    assert out["ratio"] == pytest.approx(0.15) and out["r_total"] == pytest.approx(150.0)
    assert out["critical"] == [True, True, False, False]
    assert out["reserve"] == [63, 26, 0, 0]
    assert p.reserved == [63, 26, 0, 0]


def test_phase1_low_usage_example_s358():
    p = pool_with_usage(400, {0: 0})
    ss = SpaceSchedulerOracle(p, initial_reserve_ratio=0.10)
    assert ss.update([1.0, 0.0, 0.0, 0.0], [])["ratio"] == pytest.approx(0.05)


def test_hysteresis_clamp_and_dynamic_score():
    p = pool_with_usage(700, {0: 50})
    ss = SpaceSchedulerOracle(p, initial_reserve_ratio=0.2)
    assert ss.update([0.0] * 4, [])["ratio"] == pytest.approx(0.2)        # 0.5 < 0.7 < 0.85: unchanged
    p2 = pool_with_usage(950, {0: 10})
    ss2 = SpaceSchedulerOracle(p2, initial_reserve_ratio=0.38)
    for _ in range(5):
        r = ss2.update([0.0] * 4, [])["ratio"]
        assert 0.0 <= r <= 0.40                                           # clamp
    out = ss2.update([0.0, 0.0, 0.0, 1.0], [(2, 2.0, 2 * 2.718281828459045 ** 2)])
    assert out["scores"][2] == pytest.approx(4.0)                         # 2 * ln(e^2)
    assert out["critical"] == [False, False, True, False]                 # dynamic score 4 beats static 1


def test_critical_inversion_s362():
    p = pool_with_usage(100, {0: 10})
    ss = SpaceSchedulerOracle(p, critical_ratio=0.5)
    ss.update([10.0, 2.0, 2.0, 1.0], [])
    assert ss.critical_inversion(0, 1) is True
    assert ss.critical_inversion(1, 2) is False                          # equal scores
    assert ss.critical_inversion(3, 1) is False


def test_argmax_invariance_and_budget():
    p = pool_with_usage(900, {0: 300, 1: 200, 2: 100})
    a = SpaceSchedulerOracle(p, critical_ratio=0.75, initial_reserve_ratio=0.3).update([5.0, 3.0, 1.0, 0.5], [])
    q = pool_with_usage(900, {0: 300, 1: 200, 2: 100})
    b = SpaceSchedulerOracle(q, critical_ratio=0.75, initial_reserve_ratio=0.3).update([50.0, 30.0, 10.0, 5.0], [])
    assert a["critical"] == b["critical"]
    assert sum(a["reserve"]) <= a["r_total"] + sum(a["critical"])
