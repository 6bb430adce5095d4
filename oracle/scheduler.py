"""CPU ORACLE for the decision layers around the hot path — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

NEXT-3  Time Scheduler (§4.1-4.2): Eq. 1 FC-duration forecast with an EWMA history, the linear
        transfer-cost model, Alg. 1 ShouldOffload and the predictive-upload plan (P:388,
        P:492-495).  Readings where the paper is silent follow SPEC.md time_scheduler: alpha/beta, the
        best-fit rule, token demand, the reservation lead, the immediate-upload fallback.
NEXT-4  Space Scheduler (§5): hybrid priority, critical-agent selection and Alg. 2
        UpdateMemoryReservations.  Readings follow SPEC.md space_scheduler: thresholds,
        natural log with the ratio clamped at 1, sum as the "combined" operator, proportional renormalisation when
        the final ratios sum above 1, floor rounding, lexical tie-break.

Plain fp64 Python, written in the paper's order and notation.  Pinned by the SPEC worked examples in
tests/test_scheduler_oracle.py.
"""
from __future__ import annotations

import math

# ------------------------------------------------------------------------------------------------- NEXT-3


def predict_fc_duration(t_hist, n_obs: int, cold_start: float, t_req=None, alpha: float = 0.5) -> float:
    """Eq. 1: t_final = alpha * t_req + (1 - alpha) * t_hist.  Before the first observation the
    cold-start estimate from static analysis is used, or the developer hint if given."""
    if n_obs == 0:
        return float(t_req) if t_req is not None else float(cold_start)
    if t_req is None:
        return float(t_hist)
    return alpha * t_req + (1.0 - alpha) * t_hist


def record_fc_observation(t_hist, n_obs: int, observed: float, beta: float = 0.5) -> tuple:
    """EWMA update with the observed call time fed back."""
    if observed <= 0:
        raise ValueError("non-positive observation")
    if n_obs == 0:
        return float(observed), 1
    return beta * observed + (1.0 - beta) * t_hist, n_obs + 1


def transfer_time(n_blocks: int, offload_ms_per_block: float, upload_ms_per_block: float,
                  fixed_ms: float = 0.0) -> float:
    """T_transfer = T_offload(N_blocks) + T_upload(N_blocks), "generally linear with the number of blocks"
    (P:414-420).  The per-block costs come from this build's own measurement."""
    if n_blocks <= 0:
        return 0.0
    return fixed_ms + n_blocks * (offload_ms_per_block + upload_ms_per_block)


def should_offload(n_blocks: int, t_fc: float, t_transfer: float, v_throughput_tok_s: float,
                   waiting_tokens) -> dict:
    """Alg. 1 ShouldOffload.  FindBestFitRequestInQueue = the largest waiting request whose total token
    demand fits N_capacity; ties -> the earliest in the queue."""
    out = {"offload": False, "t_transfer": t_transfer, "t_window": 0.0, "n_capacity": 0.0, "match": -1}
    if t_fc <= t_transfer:                                       # line 4-5: "Stall is too short."
        return out
    t_window = t_fc - t_transfer                                 # line 7
    n_capacity = t_window * v_throughput_tok_s / 1000.0          # line 8: computable tokens (ms x tok/s)
    best, best_tok = -1, -1.0
    for i, tok in enumerate(waiting_tokens):                     # line 10: total <= N_capacity
        if tok <= n_capacity and tok > best_tok:
            best, best_tok = i, tok
    out.update(t_window=t_window, n_capacity=n_capacity, match=best, offload=best >= 0)
    return out


def plan_predictive_upload(call_start: float, t_final: float, upload_ms: float, offload_ms: float,
                           lead_ms: float = 100.0) -> dict:
    """Predictive upload: finish the upload at the predicted FC completion; gradual reservation ready
    `lead_ms` before it starts.  If the window cannot even hold the offload, upload at once."""
    predicted_finish = call_start + t_final
    upload_start = predicted_finish - upload_ms
    if upload_start < call_start + offload_ms:
        return {"immediate": True, "upload_start": call_start + offload_ms,
                "reservation_deadline": call_start + offload_ms, "predicted_finish": predicted_finish}
    return {"immediate": False, "upload_start": upload_start, "reservation_deadline": upload_start - lead_ms,
            "predicted_finish": predicted_finish}


# ------------------------------------------------------------------------------------------------- NEXT-4


def static_priority(w_static: float, node_depth: int, node_out_degree: int) -> float:
    """priority_static = w_static x node_depth x node_out_degree."""
    return w_static * node_depth * node_out_degree


def dynamic_priority(time_wait_ms: float, tokens_req: float, eps: float = 1.0) -> float:
    """priority_dynamic = time_wait x log(tokens_req / time_wait), natural log, ratio clamped at 1 and
    time_wait at eps (the clamp resolves the sign problem of the garbled formula)."""
    tw = max(time_wait_ms, 0.0)
    if tw == 0.0:
        return 0.0
    return tw * math.log(max(tokens_req / max(tw, eps), 1.0))


def select_critical(scores: dict, critical_ratio: float) -> list:
    """Top max(1, floor(critical_ratio x |types|)) agent types by combined score, ties by type name.
    Reading B6: SPEC's text says ceiling but its own example {A:5,B:5,C:1} at 0.34 -> {A} needs floor;
    floor with a minimum of one satisfies all three SPEC examples."""
    if not scores:
        return []
    k = max(1, math.floor(critical_ratio * len(scores) + 1e-9))
    order = sorted(scores, key=lambda t: (-scores[t], t))
    return sorted(order[:k])


def update_memory_reservations(total_reserve_ratio: float, usage: int, tot_blks: int, critical: list,
                               scores: dict, type_usage: dict, gpu_usage_high: float = 0.85,
                               gpu_usage_low: float = 0.50, adjustment_step: float = 0.05,
                               reserve_ratio_max: float = 0.40) -> tuple:
    """Alg. 2.  Phase 1 adjusts total_reserve_ratio by system usage; Phase 2 splits R_total among the
    critical types by (mem_ratio + priority_ratio) / 2.  Returns (new ratio, R_total, {type: reserve_num})."""
    ratio = usage / tot_blks                                              # line 5
    if ratio >= gpu_usage_high:                                           # line 6-7
        total_reserve_ratio += adjustment_step
    elif ratio <= gpu_usage_low:                                          # line 8-9
        total_reserve_ratio -= adjustment_step
    total_reserve_ratio = min(max(total_reserve_ratio, 0.0), reserve_ratio_max)   # clamp
    r_total = tot_blks * total_reserve_ratio                              # line 11
    s_total = sum(scores[a] for a in critical)                            # line 13
    final = {}
    for a in critical:                                                    # line 14-18
        mem_ratio = type_usage.get(a, 0) / tot_blks
        priority_ratio = scores[a] / s_total if s_total > 0 else 0.0
        final[a] = (mem_ratio + priority_ratio) / 2.0
    fsum = sum(final.values())
    if fsum > 1.0:                                                        # renormalise
        final = {a: f / fsum for a, f in final.items()}
    reserve_num = {a: int(math.floor(final[a] * r_total)) for a in critical}
    return total_reserve_ratio, r_total, reserve_num
