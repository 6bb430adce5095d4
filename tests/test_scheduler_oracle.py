"""Pins of the decision-layer oracle (oracle/scheduler.py, NEXT-3 / NEXT-4) to SPEC.md worked examples and to the
closed-form properties SPEC lists."""
import math

import numpy as np
import pytest

from oracle import scheduler as S


# --------------------------------------------------------------------------- NEXT-3: Eq. 1, EWMA, Alg. 1, upload plan
def test_eq1_examples():
    assert S.predict_fc_duration(4000, 3, 999, t_req=2000, alpha=0.5) == pytest.approx(3000)
    assert S.predict_fc_duration(None, 0, 999, t_req=500) == 500
    assert S.predict_fc_duration(2000, 1, 999, t_req=1000, alpha=0.3) == pytest.approx(1700)
    assert S.predict_fc_duration(None, 0, 3000) == 3000                                        # cold start
    assert S.predict_fc_duration(800, 2, 3000) == 800                                          # history, no hint


def test_eq1_boundaries():
    # alpha = 1 returns the hint exactly, alpha = 0 returns t_hist exactly
    assert S.predict_fc_duration(123.0, 4, 0, t_req=77.0, alpha=1.0) == 77.0
    assert S.predict_fc_duration(123.0, 4, 0, t_req=77.0, alpha=0.0) == 123.0


def test_ewma_examples_and_convergence():
    t, n = S.record_fc_observation(None, 0, 800)
    assert (t, n) == (800.0, 1)
    t, n = S.record_fc_observation(800, 1, 1200, beta=0.5)
    assert t == pytest.approx(1000)
    t, n = S.record_fc_observation(1000, 2, 1000, beta=0.5)                                    # S:257 fixed point
    assert t == pytest.approx(1000)
    with pytest.raises(ValueError):
        S.record_fc_observation(1000, 2, 0)
    # geometric convergence with ratio (1 - beta)
    t, n, beta, d = 0.0, 1, 0.3, 500.0
    for k in range(1, 30):
        t, n = S.record_fc_observation(t, n, d, beta=beta)
        assert abs(t - d) == pytest.approx(d * (1 - beta) ** k, rel=1e-9)


def test_transfer_time_linear():
    per = 30.0 / 4096                                                                          # SPEC default
    assert S.transfer_time(4096, per, per) == pytest.approx(60.0)
    assert S.transfer_time(0, per, per) == 0.0
    assert S.transfer_time(2048, per, per) == pytest.approx(30.0)


def test_alg1_examples():
    per = 30.0 / 4096
    # T_fc=100, n=4096 -> T_transfer=60, window 40 ms, 1000 tok/s -> 40 tokens; smallest waiting 4000 -> retain
    d = S.should_offload(4096, 100.0, S.transfer_time(4096, per, per), 1000.0, [4000, 5000])
    assert d["offload"] is False and d["n_capacity"] == pytest.approx(40.0)
    d = S.should_offload(4096, 5000.0, 60.0, 2000.0, [12000, 8000, 9000])
    assert d["offload"] is True and d["n_capacity"] == pytest.approx(9880.0) and d["match"] == 2
    assert S.should_offload(10, 5000.0, 60.0, 2000.0, [])["offload"] is False                  # S:264 empty queue
    d = S.should_offload(10, 50.0, 60.0, 2000.0, [1])                                          # stall too short
    assert d["offload"] is False and d["t_window"] == 0.0


@pytest.mark.parametrize("seed", range(20))
def test_alg1_properties(seed):
    rng = np.random.default_rng(seed)
    for _ in range(200):
        t_fc, t_tr = rng.uniform(0, 1000, size=2)
        v = rng.uniform(1, 5000)
        q = list(rng.integers(1, 5000, size=rng.integers(0, 6)))
        d = S.should_offload(5, t_fc, t_tr, v, q)
        if t_fc <= t_tr:
            assert d["offload"] is False
        if d["offload"]:
            assert q[d["match"]] <= d["n_capacity"]
            assert all(x > d["n_capacity"] or x <= q[d["match"]] for x in q)                    # best fit


def test_predictive_upload_plan_examples():
    p = S.plan_predictive_upload(0.0, 5000.0, upload_ms=30.0, offload_ms=30.0, lead_ms=100.0)
    assert (p["immediate"], p["upload_start"], p["reservation_deadline"]) == (False, 4970.0, 4870.0)
    p = S.plan_predictive_upload(0.0, 50.0, upload_ms=30.0, offload_ms=30.0)
    assert p["immediate"] is True


# --------------------------------------------------------------------------- NEXT-4: priorities, Alg. 2
def test_dynamic_priority_examples():
    assert S.dynamic_priority(2.0, 2 * math.e ** 2) == pytest.approx(4.0)
    assert S.dynamic_priority(0.0, 100.0) == 0.0
    assert S.dynamic_priority(50.0, 10.0) == 0.0                                               # S:326 ratio clamp
    assert S.static_priority(0.5, 3, 4) == 6.0


def test_select_critical_examples():
    assert len(S.select_critical({"a": 1, "b": 2, "c": 3, "d": 4}, 0.25)) == 1
    assert S.select_critical({"a": 1, "b": 2, "c": 3, "d": 4}, 0.25) == ["d"]
    assert S.select_critical({"a": 1, "b": 2}, 1.0) == ["a", "b"]
    assert S.select_critical({"A": 5, "B": 5, "C": 1}, 0.34) == ["A"]                          # S:344 tie-break
    assert S.select_critical({}, 0.5) == []
    # argmax invariance under positive scaling
    sc = {"x": 3.0, "y": 1.0, "z": 2.0, "w": 0.5}
    assert S.select_critical(sc, 0.5) == S.select_critical({k: 7.5 * v for k, v in sc.items()}, 0.5)


def test_alg2_examples():
    r, R, _ = S.update_memory_reservations(0.10, 900, 1000, [], {}, {})
    assert r == pytest.approx(0.15) and R == pytest.approx(150.0)
    r, R, res = S.update_memory_reservations(0.10, 900, 1000, ["X", "Y"], {"X": 3.0, "Y": 1.0},
                                             {"X": 100, "Y": 100})
    assert R == pytest.approx(150.0) and res == {"X": 63, "Y": 26}
    r, _, _ = S.update_memory_reservations(0.10, 400, 1000, [], {}, {})
    assert r == pytest.approx(0.05)


@pytest.mark.parametrize("seed", range(10))
def test_alg2_properties(seed):
    rng = np.random.default_rng(seed)
    r = 0.1
    for _ in range(300):
        tot = int(rng.integers(100, 100000))
        usage = int(rng.integers(0, tot + 1))
        before = r
        types = ["t%d" % i for i in range(int(rng.integers(0, 5)))]
        scores = {t: float(rng.uniform(0.01, 10)) for t in types}
        tu = {t: int(rng.integers(0, tot // 2 + 1)) for t in types}
        r, R, res = S.update_memory_reservations(r, usage, tot, types, scores, tu)
        assert 0.0 <= r <= 0.40 + 1e-12                                                         # S:380 clamp
        if 0.50 < usage / tot < 0.85:
            assert r == before                                                                  # S:378 hysteresis
        assert sum(res.values()) <= R + 1e-9                                                    # S:379 budget
