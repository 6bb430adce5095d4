// Decision layers around the hot path, host-only C++ behind the C ABI (include/tokencake.h, NEXT-3 / NEXT-4).
//
// NEXT-3 Time Scheduler: Eq. 1 forecast + EWMA, linear transfer cost calibrated from this pool's own
//        measured transfers, Alg. 1 ShouldOffload, predictive-upload plan.
// NEXT-4 Space Scheduler: static / dynamic priority, critical selection, Alg. 2
//        UpdateMemoryReservations, applied to the pool's partitions through tc_partition_reserve.
// Readings where the paper is silent are DESIGN.md B6-B9 (SPEC.md's choices); the CPU oracle is oracle/scheduler.py.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "runtime.hpp"

extern "C" {

double tc_fc_predict(const tc_fc_stat *s, double t_req, double alpha) {
    if (!s) return 0.0;
    if (s->n_obs == 0) return t_req >= 0 ? t_req : s->cold_start;        // cold start / hint
    if (t_req < 0) return s->t_hist;
    return alpha * t_req + (1.0 - alpha) * s->t_hist;                    // Eq. 1
}

tc_status tc_fc_observe(tc_fc_stat *s, double observed_ms, double beta) {
    if (!s || !(observed_ms > 0)) return TC_E_INVAL;
    s->t_hist = s->n_obs == 0 ? observed_ms : beta * observed_ms + (1.0 - beta) * s->t_hist;   // EWMA
    s->n_obs += 1;
    return TC_OK;
}

double tc_transfer_ms(const tc_xfer_model *m, int64_t n_blocks) {
    if (!m || n_blocks <= 0) return 0.0;
    return m->fixed_ms + (double)n_blocks * (m->offload_ms_per_block + m->upload_ms_per_block);
}

tc_status tc_xfer_model_measure(tc_pool *p, tc_xfer_model *m) {
    if (!p || !m) return TC_E_INVAL;
    const tc::Pool &P = p->impl;
    if (P.cal_blocks[0] <= 0 || P.cal_blocks[1] <= 0) return TC_E_BUSY;  // nothing measured yet (tc_timing on)
    // per direction, least squares t = a + b*n over the measured spans ("generally linear"); with a single
    // distinct size the fit degenerates and the line goes through the origin (a = 0, b = mean ms per block)
    double per[2], fixed = 0.0;
    for (int d = 0; d < 2; ++d) {
        const double c = P.cal_cnt[d], sn = (double)P.cal_blocks[d], st = P.cal_ms[d];
        const double det = c * P.cal_nn[d] - sn * sn;
        double b = st / sn, a = 0.0;
        if (c >= 2 && det > 1e-9 * c * P.cal_nn[d]) {
            b = (c * P.cal_nt[d] - sn * st) / det;
            a = (st - b * sn) / c;
            if (a < 0 || b <= 0) {                                      // keep the model physical
                a = 0.0;
                b = st / sn;
            }
        }
        per[d] = b;
        fixed += a;
    }
    m->offload_ms_per_block = per[0];
    m->upload_ms_per_block = per[1];
    m->fixed_ms = fixed;
    return TC_OK;
}

tc_status tc_should_offload(int64_t n_blocks, double t_fc, double t_transfer, double v_tok_s,
                            const double *waiting_tokens, int64_t n_waiting, tc_offload_decision *out) {
    if (!out || n_blocks < 0 || n_waiting < 0 || (n_waiting > 0 && !waiting_tokens)) return TC_E_INVAL;
    *out = tc_offload_decision{0, -1, t_transfer, 0.0, 0.0};
    if (t_fc <= t_transfer) return TC_OK;                                // Alg. 1 line 4-5
    out->t_window = t_fc - t_transfer;                                   // line 7
    out->n_capacity = out->t_window * v_tok_s / 1000.0;                  // line 8
    double best = -1.0;
    for (int64_t i = 0; i < n_waiting; ++i)                              // line 10: best fit
        if (waiting_tokens[i] <= out->n_capacity && waiting_tokens[i] > best) {
            best = waiting_tokens[i];
            out->match = (int32_t)i;
        }
    out->offload = out->match >= 0;
    return TC_OK;
}

tc_status tc_plan_upload(double call_start, double t_final, double upload_ms, double offload_ms, double lead_ms,
                         tc_upload_plan *out) {
    if (!out) return TC_E_INVAL;
    const double finish = call_start + t_final;
    const double start = finish - upload_ms;
    if (start < call_start + offload_ms)
        *out = tc_upload_plan{1, call_start + offload_ms, call_start + offload_ms, finish};
    else
        *out = tc_upload_plan{0, start, start - lead_ms, finish};
    return TC_OK;
}

double tc_static_priority(double w_static, int32_t node_depth, int32_t node_out_degree) {
    return w_static * node_depth * node_out_degree;
}

double tc_dynamic_priority(double time_wait_ms, double tokens_req) {
    const double tw = time_wait_ms > 0 ? time_wait_ms : 0.0;
    if (tw == 0.0) return 0.0;
    return tw * std::log(std::max(tokens_req / std::max(tw, 1.0), 1.0));   // P:593, ratio clamped at 1 (B7)
}

tc_status tc_select_critical(int32_t n_types, const double *scores, double critical_ratio, uint8_t *critical) {
    if (n_types < 0 || (n_types > 0 && (!scores || !critical)) || !(critical_ratio > 0) || critical_ratio > 1)
        return TC_E_INVAL;
    if (n_types == 0) return TC_OK;
    const int k = std::max(1, (int)std::floor(critical_ratio * n_types + 1e-9));   // B6
    std::vector<int32_t> order(n_types);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return scores[a] > scores[b]; });
    std::fill(critical, critical + n_types, 0);
    for (int i = 0; i < k; ++i) critical[order[i]] = 1;
    return TC_OK;
}

tc_status tc_update_reservations(const tc_partition_params *pp, double *total_reserve_ratio, int64_t usage,
                                 int64_t tot_blks, int32_t n_types, const uint8_t *critical, const double *scores,
                                 const int64_t *type_usage, double *r_total, int64_t *reserve_num) {
    if (!pp || !total_reserve_ratio || tot_blks <= 0 || n_types < 0 ||
        (n_types > 0 && (!critical || !scores || !type_usage || !reserve_num)))
        return TC_E_INVAL;
    // Phase 1 (Alg. 2 lines 5-11)
    double trr = *total_reserve_ratio;
    const double ratio = (double)usage / (double)tot_blks;
    if (ratio >= pp->gpu_usage_high)
        trr += pp->adjustment_step;
    else if (ratio <= pp->gpu_usage_low)
        trr -= pp->adjustment_step;
    trr = std::min(std::max(trr, 0.0), pp->reserve_ratio_max);
    const double R = (double)tot_blks * trr;
    // Phase 2 (lines 13-18)
    double s_total = 0.0;
    for (int32_t t = 0; t < n_types; ++t)
        if (critical[t]) s_total += scores[t];
    std::vector<double> fin(n_types, 0.0);
    double fsum = 0.0;
    for (int32_t t = 0; t < n_types; ++t) {
        if (!critical[t]) continue;
        const double mem_ratio = (double)type_usage[t] / (double)tot_blks;
        const double priority_ratio = s_total > 0 ? scores[t] / s_total : 0.0;
        fin[t] = (mem_ratio + priority_ratio) / 2.0;
        fsum += fin[t];
    }
    for (int32_t t = 0; t < n_types; ++t) {
        double f = fin[t];
        if (fsum > 1.0) f = f / fsum;                                   // renormalise (B8)
        reserve_num[t] = critical[t] ? (int64_t)std::floor(f * R) : 0;
    }
    *total_reserve_ratio = trr;
    if (r_total) *r_total = R;
    return TC_OK;
}

tc_status tc_apply_reservations(tc_pool *p, int32_t n, const int32_t *classes, const int64_t *reserve_num) {
    if (!p || n < 0 || (n > 0 && (!classes || !reserve_num))) return TC_E_INVAL;
    tc::Pool &P = p->impl;
    std::vector<int64_t> next = P.alloc.reserved;
    for (int32_t i = 0; i < n; ++i) {
        if (classes[i] < 0 || classes[i] >= P.n_classes || reserve_num[i] < 0) return TC_E_INVAL;
        next[classes[i]] = reserve_num[i];
    }
    int64_t sum = 0;
    for (int64_t r : next) sum += r;
    if (sum > P.N) return TC_E_INVAL;
    P.alloc.reserved = next;                                             // lazy shrink: claimed untouched
    return TC_OK;
}

}  // extern "C"
