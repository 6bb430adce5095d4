"""The C-ABI decision layers (csrc/sched.cpp via paper_2510_18586_b200.sched) against the pinned oracle
(oracle/scheduler.py) on seeded random inputs: discrete decisions (offload?, match, critical set, reserve_num) must
agree exactly; fp64 values to 1e-12 relative (same formulas, same operation order)."""
import numpy as np
import pytest

import paper_2510_18586_b200 as tcb
from oracle import scheduler as O
from paper_2510_18586_b200 import sched as C

REL = 1e-12


@pytest.mark.parametrize("seed", range(10))
def test_eq1_ewma_parity(seed):
    rng = np.random.default_rng(seed)
    for _ in range(500):
        n_obs = int(rng.integers(0, 3))
        t_hist = None if n_obs == 0 else float(rng.uniform(1, 1e5))
        hint = None if rng.random() < 0.3 else float(rng.uniform(1, 1e5))
        alpha = float(rng.uniform(0, 1))
        cold = float(rng.uniform(1, 1e4))
        assert C.fc_predict(t_hist, n_obs, cold, hint, alpha) == pytest.approx(
            O.predict_fc_duration(t_hist, n_obs, cold, hint, alpha), rel=REL)
        obs, beta = float(rng.uniform(1, 1e5)), float(rng.uniform(0, 1))
        a, b = C.fc_observe(t_hist, n_obs, obs, beta), O.record_fc_observation(t_hist, n_obs, obs, beta)
        assert a[1] == b[1] and a[0] == pytest.approx(b[0], rel=REL)
    with pytest.raises(tcb.TcError):
        C.fc_observe(1.0, 1, 0.0)


@pytest.mark.parametrize("seed", range(10))
def test_alg1_parity(seed):
    rng = np.random.default_rng(100 + seed)
    for _ in range(500):
        n = int(rng.integers(0, 5000))
        off, up = float(rng.uniform(0, 0.05)), float(rng.uniform(0, 0.05))
        tt = C.transfer_ms(n, off, up)
        assert tt == pytest.approx(O.transfer_time(n, off, up), rel=REL, abs=0)
        t_fc = float(rng.uniform(0, 300))
        v = float(rng.uniform(1, 5000))
        q = [float(x) for x in rng.integers(1, 2000, size=int(rng.integers(0, 8)))]
        a, b = C.should_offload(n, t_fc, tt, v, q), O.should_offload(n, t_fc, tt, v, q)
        assert (a["offload"], a["match"]) == (b["offload"], b["match"])
        assert a["n_capacity"] == pytest.approx(b["n_capacity"], rel=REL, abs=1e-12)
        cs, tf, ul, ol = (float(x) for x in rng.uniform(0, 1000, size=4))
        pa, pb = C.plan_upload(cs, tf, ul, ol, 100.0), O.plan_predictive_upload(cs, tf, ul, ol, 100.0)
        assert pa["immediate"] == pb["immediate"]
        for k in ("upload_start", "reservation_deadline", "predicted_finish"):
            assert pa[k] == pytest.approx(pb[k], rel=REL, abs=1e-9)


def test_spec_examples_through_capi():
    assert C.fc_predict(4000, 3, 0, 2000, 0.5) == pytest.approx(3000)
    d = C.should_offload(4096, 5000.0, 60.0, 2000.0, [12000, 8000, 9000])
    assert d["offload"] and d["n_capacity"] == pytest.approx(9880.0) and d["match"] == 2
    r, R, res = C.update_reservations(0.10, 900, 1000, ["X", "Y"], {"X": 3.0, "Y": 1.0}, {"X": 100, "Y": 100})
    assert r == pytest.approx(0.15) and R == pytest.approx(150.0) and res == {"X": 63, "Y": 26}
    assert C.select_critical({"A": 5, "B": 5, "C": 1}, 0.34) == ["A"]
    assert C.dynamic_priority(2.0, 2 * np.e ** 2) == pytest.approx(4.0)


@pytest.mark.parametrize("seed", range(10))
def test_space_parity(seed):
    rng = np.random.default_rng(200 + seed)
    r_o = r_c = float(rng.uniform(0, 0.4))
    for _ in range(300):
        k = int(rng.integers(1, 7))
        names = ["type%d" % i for i in range(k)]
        scores = {n: float(rng.choice([rng.uniform(0, 10), 1.0])) for n in names}
        ratio = float(rng.uniform(0.05, 1.0))
        crit_o, crit_c = O.select_critical(scores, ratio), C.select_critical(scores, ratio)
        assert crit_o == crit_c
        tot = int(rng.integers(100, 200000))
        usage = int(rng.integers(0, tot + 1))
        tu = {n: int(rng.integers(0, tot // 2 + 1)) for n in names}
        a = O.update_memory_reservations(r_o, usage, tot, crit_o, scores, tu)
        b = C.update_reservations(r_c, usage, tot, crit_c, scores, tu)
        assert a[0] == pytest.approx(b[0], rel=REL, abs=1e-15) and a[2] == b[2]
        r_o, r_c = a[0], b[0]
        tw, tok = float(rng.uniform(0, 1e4)), float(rng.uniform(1, 1e5))
        assert C.dynamic_priority(tw, tok) == pytest.approx(O.dynamic_priority(tw, tok), rel=REL, abs=1e-12)
        d, od = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        assert C.static_priority(0.7, d, od) == pytest.approx(O.static_priority(0.7, d, od), rel=REL)


def test_apply_reservations_feeds_partition_rule():
    p = tcb.Pool(1, 2, 64, 16, "fp16", 64, device=-1, host_slots=8, n_classes=4)
    C.apply_reservations(p, {0: 10, 1: 5})
    assert p.stats()["reserved"][:2] == [10, 5]
    with pytest.raises(tcb.TcError):
        C.apply_reservations(p, {0: 50, 1: 20})            # sum > N: rejected, nothing changes
    assert p.stats()["reserved"][:2] == [10, 5]
    p.agent_add(0, 2)
    with pytest.raises(tcb.TcError) as e:
        p.alloc(0, 50)                                      # headroom = 64 - 15
    assert e.value.status == tcb.E_NOBLOCKS
    assert len(p.alloc(0, 49)) == 49
