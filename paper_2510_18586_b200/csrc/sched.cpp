// Decision layers around the hot path, host-only C++ behind the C ABI (include/tokencake.h, NEXT-3 / NEXT-4).
//
// NEXT-3 Time Scheduler: Eq. 1 forecast + EWMA, linear transfer cost calibrated from this pool's own
//        measured transfers, Alg. 1 ShouldOffload, predictive-upload plan.
// NEXT-4 Space Scheduler: static / dynamic priority, critical selection, Alg. 2
//        UpdateMemoryReservations, applied to the pool's partitions through tc_partition_reserve.
// Readings where the paper is silent are DESIGN.md B6-B9 (SPEC.md's choices); the CPU oracle is oracle/scheduler.py.
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <utility>
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

// ------------------------------------------------------------------------------------------------ NEXT-3 runtime
// The Time Scheduler as an event machine (include/tokencake.h "NEXT-3: the Time Scheduler as a runtime"; DESIGN.md
// reading C2; oracle: oracle/time_scheduler.py).
struct tc_ts {
    tc_pool *pool = nullptr;
    tc_ts_params prm{};
    std::map<std::pair<int32_t, int32_t>, tc_fc_stat> table;   // (agent class, label) -> EWMA state
    struct Call {
        int32_t label = 0, cls = 0;
        double start = 0, upload_start = 0, resv_start = 0;
        bool off = false, up = false, resv = false, finished = false;
        tc_handle h = 0;
    };
    std::map<int32_t, Call> calls;                               // agents in a call, by id
    std::vector<int32_t> ids, new_ids;                           // scratch
};

extern "C" {

void tc_ts_params_init(tc_ts_params *prm) {
    if (!prm) return;
    *prm = tc_ts_params{0.5, 0.5, 100.0, 100.0, 10.0, 4, 1000.0, {30.0 / 4096, 30.0 / 4096, 0.0}};
}

tc_status tc_ts_create(tc_pool *p, const tc_ts_params *prm, tc_ts **out) {
    if (!p || !out) return TC_E_INVAL;
    tc_ts_params d;
    tc_ts_params_init(&d);
    if (prm) d = *prm;
    if (d.reserve_cycles < 0 || d.tick_ms < 0 || d.v_tokens_per_s < 0 || d.alpha < 0 || d.alpha > 1 ||
        d.beta < 0 || d.beta > 1)
        return TC_E_INVAL;
    try {
        tc_ts *s = new tc_ts();
        s->pool = p;
        s->prm = d;
        *out = s;
    } catch (...) {
        return TC_E_OOM;
    }
    return TC_OK;
}

void tc_ts_destroy(tc_ts *s) { delete s; }

tc_status tc_ts_call_start(tc_ts *s, int32_t agent, int32_t label, double now_ms, double t_req_ms,
                           const double *waiting_tokens, int64_t n_waiting, tc_ts_decision *out) {
    if (!s || !out || n_waiting < 0 || (n_waiting > 0 && !waiting_tokens)) return TC_E_INVAL;
    try {
        tc::Pool &P = s->pool->impl;
        if (agent < 0 || agent >= P.max_agents || !P.agents[agent].exists || s->calls.count(agent)) return TC_E_INVAL;
        const tc_ts_params &q = s->prm;
        s->ids.clear();
        for (int32_t b : P.agents[agent].table)
            if (b >= 0) s->ids.push_back(b);
        const int64_t n = (int64_t)s->ids.size();
        tc_ts::Call c;
        c.label = label;
        c.cls = P.agents[agent].cls;
        c.start = now_ms;
        tc_fc_stat st{0.0, 0, q.cold_start_ms};
        auto it = s->table.find({c.cls, label});
        if (it != s->table.end()) st = it->second;
        st.cold_start = q.cold_start_ms;
        *out = tc_ts_decision{0, -1, TC_OK, tc_fc_predict(&st, t_req_ms, q.alpha), 0.0, 0.0, 0.0, 0};   // Eq. 1
        out->t_transfer = tc_transfer_ms(&q.model, n);
        if (n > 0) {
            tc_offload_decision d;
            tc_status r = tc_should_offload(n, out->t_fc, out->t_transfer, q.v_tokens_per_s, waiting_tokens,
                                            n_waiting, &d);                                              // Alg. 1
            if (r != TC_OK) return r;
            out->match = d.match;
            if (d.offload) {
                tc_handle h = 0;
                const int64_t off[2] = {0, n};
                r = P.offload_batch(1, &agent, off, s->ids.data(), &h);
                if (r == TC_E_NOHOST) {
                    out->status = TC_E_NOHOST;                 // refused: the request keeps its blocks
                } else if (r != TC_OK) {
                    return r;
                } else {
                    tc_upload_plan plan;
                    tc_plan_upload(now_ms, out->t_fc, (double)n * q.model.upload_ms_per_block,
                                   (double)n * q.model.offload_ms_per_block, q.lead_ms, &plan);
                    c.off = true;
                    c.h = h;
                    c.upload_start = plan.upload_start;
                    c.resv_start = plan.reservation_deadline - q.reserve_cycles * q.tick_ms;
                    out->offload = 1;
                    out->handle = h;
                    out->upload_start = c.upload_start;
                    out->reservation_start = c.resv_start;
                }
            }
        }
        s->calls[agent] = c;
        if (P.check) P.check_invariants("tc_ts_call_start");
        return TC_OK;
    } catch (...) {
        return TC_E_OOM;
    }
}

tc_status tc_ts_tick(tc_ts *s, double now_ms, int32_t *uploads_issued) {
    if (!s) return TC_E_INVAL;
    try {
        tc::Pool &P = s->pool->impl;
        int32_t issued = 0;
        for (auto &kv : s->calls) {                        // gradual reservation, ready by its deadline
            tc_ts::Call &c = kv.second;
            if (c.off && !c.up && !c.finished && !c.resv && s->prm.reserve_cycles > 0 && now_ms >= c.resv_start) {
                const tc_status r = P.reserve_begin(c.h, s->prm.reserve_cycles);
                if (r != TC_OK) return r;
                c.resv = true;
            }
        }
        tc_status r = P.reserve_tick();
        if (r != TC_OK) return r;
        for (auto &kv : s->calls) {                        // predictive uploads that are due
            tc_ts::Call &c = kv.second;
            if (!c.off || c.up || c.finished || now_ms < c.upload_start) continue;
            auto hit = P.handles.find(c.h);
            if (hit == P.handles.end()) return TC_E_HANDLE;
            s->new_ids.resize(hit->second.pos.size());
            const int64_t off[2] = {0, (int64_t)hit->second.pos.size()};
            r = P.upload_batch(1, &c.h, off, s->new_ids.data());
            if (r == TC_E_NOBLOCKS) continue;              // "stalls": retried next tick
            if (r != TC_OK) return r;
            c.up = true;
            ++issued;
        }
        if (uploads_issued) *uploads_issued = issued;
        if (P.check) P.check_invariants("tc_ts_tick");
        return TC_OK;
    } catch (...) {
        return TC_E_OOM;
    }
}

tc_status tc_ts_call_finish(tc_ts *s, int32_t agent, double now_ms, tc_handle *wait_handle) {
    if (!s || !wait_handle) return TC_E_INVAL;
    try {
        auto it = s->calls.find(agent);
        if (it == s->calls.end()) return TC_E_INVAL;
        tc_ts::Call &c = it->second;
        if (!c.finished) {                                 // EWMA feedback
            if (now_ms - c.start > 0) {
                tc_fc_stat &st = s->table.emplace(std::make_pair(c.cls, c.label),
                                                  tc_fc_stat{0.0, 0, s->prm.cold_start_ms}).first->second;
                tc_fc_observe(&st, now_ms - c.start, s->prm.beta);
            }
            c.finished = true;
        }
        if (!c.off) {
            *wait_handle = 0;                              // retained: resume at once
            s->calls.erase(it);
            return TC_OK;
        }
        if (!c.up) {                                       // early return: immediate upload
            tc::Pool &P = s->pool->impl;
            auto hit = P.handles.find(c.h);
            if (hit == P.handles.end()) return TC_E_HANDLE;
            s->new_ids.resize(hit->second.pos.size());
            const int64_t off[2] = {0, (int64_t)hit->second.pos.size()};
            const tc_status r = P.upload_batch(1, &c.h, off, s->new_ids.data());
            if (r != TC_OK) return r;                      // NOBLOCKS: nothing else changed; retry
            c.up = true;
        }
        *wait_handle = c.h;
        s->calls.erase(it);
        if (s->pool->impl.check) s->pool->impl.check_invariants("tc_ts_call_finish");
        return TC_OK;
    } catch (...) {
        return TC_E_OOM;
    }
}

tc_status tc_ts_forecast(tc_ts *s, int32_t agent_class, int32_t label, double *t_hist, int64_t *n_obs) {
    if (!s || !t_hist || !n_obs) return TC_E_INVAL;
    auto it = s->table.find({agent_class, label});
    *t_hist = it == s->table.end() ? 0.0 : it->second.t_hist;
    *n_obs = it == s->table.end() ? 0 : it->second.n_obs;
    return TC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------ NEXT-4 runtime
// One Space-Scheduler partition update over a pool (include/tokencake.h; reading C3; oracle:
// oracle/space_scheduler.py).
struct tc_ss {
    tc_pool *pool = nullptr;
    tc_ss_params prm{};
    double ratio = 0.0;
    std::vector<double> scores;
};

extern "C" {

void tc_ss_params_init(tc_ss_params *prm) {
    if (!prm) return;
    *prm = tc_ss_params{{0.85, 0.50, 0.05, 0.40}, 0.25, 0.0};
}

tc_status tc_ss_create(tc_pool *p, const tc_ss_params *prm, tc_ss **out) {
    if (!p || !out) return TC_E_INVAL;
    tc_ss_params d;
    tc_ss_params_init(&d);
    if (prm) d = *prm;
    if (!(d.critical_ratio > 0 && d.critical_ratio <= 1) || d.initial_reserve_ratio < 0) return TC_E_INVAL;
    try {
        tc_ss *s = new tc_ss();
        s->pool = p;
        s->prm = d;
        s->ratio = d.initial_reserve_ratio;
        *out = s;
    } catch (...) {
        return TC_E_OOM;
    }
    return TC_OK;
}

void tc_ss_destroy(tc_ss *s) { delete s; }

tc_status tc_ss_update(tc_ss *s, const double *static_score, int64_t n_waiting, const int32_t *waiting_class,
                       const double *time_wait_ms, const double *tokens_req, int64_t *reserve_num,
                       uint8_t *critical, double *scores, double *total_reserve_ratio) {
    if (!s || !static_score || n_waiting < 0 ||
        (n_waiting > 0 && (!waiting_class || !time_wait_ms || !tokens_req)))
        return TC_E_INVAL;
    try {
        tc::Pool &P = s->pool->impl;
        const int32_t n = P.n_classes;
        std::vector<double> sc(static_score, static_score + n);
        for (int64_t i = 0; i < n_waiting; ++i) {          // hybrid score: static + sum of dynamic
            if (waiting_class[i] < 0 || waiting_class[i] >= n) return TC_E_INVAL;
            sc[waiting_class[i]] += tc_dynamic_priority(time_wait_ms[i], tokens_req[i]);
        }
        std::vector<uint8_t> crit(n, 0);
        tc_status r = tc_select_critical(n, sc.data(), s->prm.critical_ratio, crit.data());
        if (r != TC_OK) return r;
        std::vector<int64_t> per(n, 0);                    // the pool's own usage, per class
        for (int32_t a = 0; a < P.max_agents; ++a) {
            const tc::AgentRec &ag = P.agents[a];
            if (!ag.exists) continue;
            for (int32_t b : ag.table)
                if (b >= 0 && P.alloc.state[b] == tc::kAlloc) ++per[ag.cls];
        }
        const int64_t usage = P.N - P.alloc.nfree;
        double ratio = s->ratio, r_total = 0.0;
        std::vector<int64_t> res(n, 0);
        r = tc_update_reservations(&s->prm.partition, &ratio, usage, P.N, n, crit.data(), sc.data(), per.data(),
                                   &r_total, res.data());                                       // Alg. 2
        if (r != TC_OK) return r;
        std::vector<int32_t> cls(n);
        std::iota(cls.begin(), cls.end(), 0);
        if ((r = tc_apply_reservations(s->pool, n, cls.data(), res.data())) != TC_OK) return r;
        s->ratio = ratio;
        s->scores = sc;
        if (reserve_num) std::copy(res.begin(), res.end(), reserve_num);
        if (critical) std::copy(crit.begin(), crit.end(), critical);
        if (scores) std::copy(sc.begin(), sc.end(), scores);
        if (total_reserve_ratio) *total_reserve_ratio = ratio;
        if (P.check) P.check_invariants("tc_ss_update");
        return TC_OK;
    } catch (...) {
        return TC_E_OOM;
    }
}

tc_status tc_ss_critical_inversion(tc_ss *s, int32_t evicted_class, int32_t cause_class, int32_t *inversion) {
    if (!s || !inversion) return TC_E_INVAL;
    const int32_t n = (int32_t)s->scores.size();
    auto score = [&](int32_t c) { return c >= 0 && c < n ? s->scores[c] : 0.0; };
    *inversion = score(evicted_class) > score(cause_class) ? 1 : 0;
    return TC_OK;
}

}  // extern "C"
