"""ctypes binding of the decision layers around the hot path (include/tokencake.h NEXT-3 / NEXT-4 sections).

Marshalling only; the arithmetic runs in libtokencake.so (csrc/sched.cpp).
  NEXT-3 Time Scheduler: Eq. 1 forecast + EWMA, transfer-cost model (calibrated from a pool's measured transfers),
         Alg. 1 ShouldOffload, predictive-upload plan.
  NEXT-4 Space Scheduler: static / dynamic priority, critical selection, Alg. 2 reservations, applied to a pool.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import TcError, _ptr, lib

D, I32, I64, P = ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p


class FcStat(ctypes.Structure):
    _fields_ = [("t_hist", D), ("n_obs", I64), ("cold_start", D)]


class XferModel(ctypes.Structure):
    _fields_ = [("offload_ms_per_block", D), ("upload_ms_per_block", D), ("fixed_ms", D)]


class OffloadDecision(ctypes.Structure):
    _fields_ = [("offload", I32), ("match", I32), ("t_transfer", D), ("t_window", D), ("n_capacity", D)]


class UploadPlan(ctypes.Structure):
    _fields_ = [("immediate", I32), ("upload_start", D), ("reservation_deadline", D), ("predicted_finish", D)]


class PartitionParams(ctypes.Structure):
    _fields_ = [("gpu_usage_high", D), ("gpu_usage_low", D), ("adjustment_step", D), ("reserve_ratio_max", D)]


_SIG = {
    "tc_fc_predict": (D, [ctypes.POINTER(FcStat), D, D]),
    "tc_fc_observe": (I32, [ctypes.POINTER(FcStat), D, D]),
    "tc_transfer_ms": (D, [ctypes.POINTER(XferModel), I64]),
    "tc_xfer_model_measure": (I32, [P, ctypes.POINTER(XferModel)]),
    "tc_should_offload": (I32, [I64, D, D, D, ctypes.POINTER(D), I64, ctypes.POINTER(OffloadDecision)]),
    "tc_plan_upload": (I32, [D, D, D, D, D, ctypes.POINTER(UploadPlan)]),
    "tc_static_priority": (D, [D, I32, I32]),
    "tc_dynamic_priority": (D, [D, D]),
    "tc_select_critical": (I32, [I32, ctypes.POINTER(D), D, ctypes.POINTER(ctypes.c_uint8)]),
    "tc_update_reservations": (I32, [ctypes.POINTER(PartitionParams), ctypes.POINTER(D), I64, I64, I32,
                                     ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(D), ctypes.POINTER(I64),
                                     ctypes.POINTER(D), ctypes.POINTER(I64)]),
    "tc_apply_reservations": (I32, [P, I32, ctypes.POINTER(I32), ctypes.POINTER(I64)]),
}


class TsParams(ctypes.Structure):
    _fields_ = [("alpha", D), ("beta", D), ("cold_start_ms", D), ("lead_ms", D), ("tick_ms", D),
                ("reserve_cycles", I32), ("v_tokens_per_s", D), ("model", XferModel)]


class TsDecision(ctypes.Structure):
    _fields_ = [("offload", I32), ("match", I32), ("status", I32), ("t_fc", D), ("t_transfer", D),
                ("upload_start", D), ("reservation_start", D), ("handle", ctypes.c_uint64)]


class SsParams(ctypes.Structure):
    _fields_ = [("partition", PartitionParams), ("critical_ratio", D), ("initial_reserve_ratio", D)]


_SIG.update({
    "tc_ss_params_init": (None, [ctypes.POINTER(SsParams)]),
    "tc_ss_create": (I32, [P, ctypes.POINTER(SsParams), ctypes.POINTER(P)]),
    "tc_ss_destroy": (None, [P]),
    "tc_ss_update": (I32, [P, ctypes.POINTER(D), I64, ctypes.POINTER(I32), ctypes.POINTER(D), ctypes.POINTER(D),
                           ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(D),
                           ctypes.POINTER(D)]),
    "tc_ss_critical_inversion": (I32, [P, I32, I32, ctypes.POINTER(I32)]),
    "tc_ts_params_init": (None, [ctypes.POINTER(TsParams)]),
    "tc_ts_create": (I32, [P, ctypes.POINTER(TsParams), ctypes.POINTER(P)]),
    "tc_ts_destroy": (None, [P]),
    "tc_ts_call_start": (I32, [P, I32, I32, D, D, ctypes.POINTER(D), I64, ctypes.POINTER(TsDecision)]),
    "tc_ts_tick": (I32, [P, D, ctypes.POINTER(I32)]),
    "tc_ts_call_finish": (I32, [P, I32, D, ctypes.POINTER(ctypes.c_uint64)]),
    "tc_ts_forecast": (I32, [P, I32, I32, ctypes.POINTER(D), ctypes.POINTER(I64)]),
})
for _n, (_r, _a) in _SIG.items():
    _f = getattr(lib, _n)
    _f.restype, _f.argtypes = _r, _a


def _check(st):
    if st != 0:
        raise TcError(st, lib.tc_strerror(st).decode())


# ------------------------------------------------------------------------------------------------ NEXT-3
def fc_predict(t_hist, n_obs, cold_start, t_req=None, alpha=0.5) -> float:
    s = FcStat(0.0 if t_hist is None else t_hist, n_obs, cold_start)
    return lib.tc_fc_predict(ctypes.byref(s), -1.0 if t_req is None else float(t_req), alpha)


def fc_observe(t_hist, n_obs, observed, beta=0.5) -> tuple:
    s = FcStat(0.0 if t_hist is None else t_hist, n_obs, 0.0)
    _check(lib.tc_fc_observe(ctypes.byref(s), observed, beta))
    return s.t_hist, s.n_obs


def transfer_ms(n_blocks, offload_ms_per_block, upload_ms_per_block, fixed_ms=0.0) -> float:
    m = XferModel(offload_ms_per_block, upload_ms_per_block, fixed_ms)
    return lib.tc_transfer_ms(ctypes.byref(m), n_blocks)


def xfer_model_measure(pool) -> dict:
    m = XferModel()
    _check(lib.tc_xfer_model_measure(pool._h, ctypes.byref(m)))
    return {"offload_ms_per_block": m.offload_ms_per_block, "upload_ms_per_block": m.upload_ms_per_block,
            "fixed_ms": m.fixed_ms}


def should_offload(n_blocks, t_fc, t_transfer, v_tok_s, waiting_tokens) -> dict:
    w = np.ascontiguousarray(np.asarray(waiting_tokens, dtype=np.float64).reshape(-1))
    out = OffloadDecision()
    _check(lib.tc_should_offload(n_blocks, t_fc, t_transfer, v_tok_s, _ptr(w, D) if w.size else None, w.size,
                                 ctypes.byref(out)))
    return {"offload": bool(out.offload), "match": out.match, "t_transfer": out.t_transfer,
            "t_window": out.t_window, "n_capacity": out.n_capacity}


def plan_upload(call_start, t_final, upload_ms, offload_ms, lead_ms=100.0) -> dict:
    out = UploadPlan()
    _check(lib.tc_plan_upload(call_start, t_final, upload_ms, offload_ms, lead_ms, ctypes.byref(out)))
    return {"immediate": bool(out.immediate), "upload_start": out.upload_start,
            "reservation_deadline": out.reservation_deadline, "predicted_finish": out.predicted_finish}


# ------------------------------------------------------------------------------------------------ NEXT-3 runtime
class TimeScheduler:
    """The Time Scheduler as an event machine over a Pool (tc_ts_*): call_start / tick / call_finish with the
    engine's clock in ms.  Keyword parameters as tc_ts_params (model = dict of xfer_model_measure's keys)."""

    def __init__(self, pool, **kw):
        prm = TsParams()
        lib.tc_ts_params_init(ctypes.byref(prm))
        model = kw.pop("model", None)
        for k, v in kw.items():
            setattr(prm, k, v)
        if model is not None:
            prm.model = XferModel(model["offload_ms_per_block"], model["upload_ms_per_block"],
                                  model.get("fixed_ms", 0.0))
        h = ctypes.c_void_p()
        _check(lib.tc_ts_create(pool._h, ctypes.byref(prm), ctypes.byref(h)))
        self._h, self.pool = h, pool

    def close(self):
        if getattr(self, "_h", None):
            lib.tc_ts_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def call_start(self, agent: int, label: int, now: float, t_req=None, waiting=()) -> dict:
        w = np.ascontiguousarray(np.asarray(list(waiting), dtype=np.float64).reshape(-1))
        out = TsDecision()
        _check(lib.tc_ts_call_start(self._h, agent, label, now, -1.0 if t_req is None else float(t_req),
                                    _ptr(w, D) if w.size else None, w.size, ctypes.byref(out)))
        return {"offload": bool(out.offload), "match": out.match, "status": out.status, "t_fc": out.t_fc,
                "t_transfer": out.t_transfer, "upload_start": out.upload_start,
                "reservation_start": out.reservation_start, "handle": out.handle}

    def tick(self, now: float) -> int:
        n = ctypes.c_int32()
        _check(lib.tc_ts_tick(self._h, now, ctypes.byref(n)))
        return n.value

    def call_finish(self, agent: int, now: float) -> int:
        h = ctypes.c_uint64()
        _check(lib.tc_ts_call_finish(self._h, agent, now, ctypes.byref(h)))
        return h.value

    def forecast(self, agent_class: int, label: int) -> tuple:
        t, n = ctypes.c_double(), ctypes.c_int64()
        _check(lib.tc_ts_forecast(self._h, agent_class, label, ctypes.byref(t), ctypes.byref(n)))
        return (t.value if n.value else None), n.value


# ------------------------------------------------------------------------------------------------ NEXT-4
def static_priority(w, depth, out_degree) -> float:
    return lib.tc_static_priority(w, depth, out_degree)


def dynamic_priority(time_wait_ms, tokens_req) -> float:
    return lib.tc_dynamic_priority(time_wait_ms, tokens_req)


def select_critical(scores: dict, ratio: float) -> list:
    """scores keyed by type name; the library breaks ties by index, so names are passed in sorted order."""
    names = sorted(scores)
    sc = np.asarray([scores[n] for n in names], dtype=np.float64)
    crit = np.zeros(max(len(names), 1), dtype=np.uint8)
    _check(lib.tc_select_critical(len(names), _ptr(sc, D) if len(names) else None, ratio,
                                  _ptr(crit, ctypes.c_uint8)))
    return [n for n, c in zip(names, crit) if c]


def update_reservations(total_reserve_ratio, usage, tot_blks, critical, scores, type_usage,
                        gpu_usage_high=0.85, gpu_usage_low=0.50, adjustment_step=0.05, reserve_ratio_max=0.40):
    names = sorted(scores) if scores else sorted(critical)
    crit = np.asarray([1 if n in critical else 0 for n in names], dtype=np.uint8)
    sc = np.asarray([scores.get(n, 0.0) for n in names], dtype=np.float64)
    tu = np.asarray([type_usage.get(n, 0) for n in names], dtype=np.int64)
    res = np.zeros(max(len(names), 1), dtype=np.int64)
    pp = PartitionParams(gpu_usage_high, gpu_usage_low, adjustment_step, reserve_ratio_max)
    r = ctypes.c_double(total_reserve_ratio)
    R = ctypes.c_double()
    k = len(names)
    _check(lib.tc_update_reservations(ctypes.byref(pp), ctypes.byref(r), usage, tot_blks, k,
                                      _ptr(crit, ctypes.c_uint8) if k else None, _ptr(sc, D) if k else None,
                                      _ptr(tu, I64) if k else None, ctypes.byref(R), _ptr(res, I64) if k else None))
    return r.value, R.value, {n: int(v) for n, v, c in zip(names, res, crit) if c}


def apply_reservations(pool, quotas: dict):
    cls = np.asarray(list(quotas.keys()), dtype=np.int32)
    num = np.asarray(list(quotas.values()), dtype=np.int64)
    _check(lib.tc_apply_reservations(pool._h, len(cls), _ptr(cls, I32), _ptr(num, I64)))


# ------------------------------------------------------------------------------------------------ NEXT-4 runtime
class SpaceScheduler:
    """One Space-Scheduler partition update per call over a Pool (tc_ss_*): the pool's classes are the agent types,
    Alg. 2 reads the pool's own usage, the quotas are applied to the pool."""

    def __init__(self, pool, critical_ratio=0.25, initial_reserve_ratio=0.0, gpu_usage_high=0.85,
                 gpu_usage_low=0.50, adjustment_step=0.05, reserve_ratio_max=0.40):
        prm = SsParams(PartitionParams(gpu_usage_high, gpu_usage_low, adjustment_step, reserve_ratio_max),
                       critical_ratio, initial_reserve_ratio)
        h = ctypes.c_void_p()
        _check(lib.tc_ss_create(pool._h, ctypes.byref(prm), ctypes.byref(h)))
        self._h, self.pool, self.n = h, pool, pool.stats()["n_classes"]

    def close(self):
        if getattr(self, "_h", None):
            lib.tc_ss_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def update(self, static_scores, waiting=()) -> dict:
        """static_scores: one per class; waiting: [(class, time_wait_ms, tokens_req), ...]."""
        st = np.ascontiguousarray(np.asarray(static_scores, dtype=np.float64).reshape(-1))
        if st.size != self.n:
            raise TcError(-1, "one static score per class")
        w = list(waiting)
        wc = np.ascontiguousarray(np.asarray([x[0] for x in w], dtype=np.int32))
        wt = np.ascontiguousarray(np.asarray([x[1] for x in w], dtype=np.float64))
        wk = np.ascontiguousarray(np.asarray([x[2] for x in w], dtype=np.float64))
        res = np.zeros(self.n, dtype=np.int64)
        crit = np.zeros(self.n, dtype=np.uint8)
        sc = np.zeros(self.n, dtype=np.float64)
        ratio = ctypes.c_double()
        _check(lib.tc_ss_update(self._h, _ptr(st, D), len(w), _ptr(wc, I32) if w else None,
                                _ptr(wt, D) if w else None, _ptr(wk, D) if w else None, _ptr(res, I64),
                                _ptr(crit, ctypes.c_uint8), _ptr(sc, D), ctypes.byref(ratio)))
        return {"reserve": [int(x) for x in res], "critical": [bool(x) for x in crit], "ratio": ratio.value,
                "scores": [float(x) for x in sc]}

    def critical_inversion(self, evicted_cls: int, cause_cls: int) -> bool:
        r = ctypes.c_int32()
        _check(lib.tc_ss_critical_inversion(self._h, evicted_cls, cause_cls, ctypes.byref(r)))
        return bool(r.value)
