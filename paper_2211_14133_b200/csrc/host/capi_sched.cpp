// extern "C" image of the scheduler API (include/pf_sched.h).  No exception
// crosses this boundary: each reference exception type maps to a pf_status
// and the message is kept in a thread-local for pf_last_error().
#include "pf_sched.h"

#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "pipefill/bubblefill.hpp"
#include "pipefill/schedule.hpp"
#include "capi_common.hpp"

using namespace pipefill;

struct pf_schedule {
    StaticSchedule schedule;
    bool filled = false;
    double base_period = 0.0;
    int prior_inverses = 0;
    std::vector<StalenessEntry> staleness;
    bool infeasible = false;
    std::vector<KfacWork> unplaced;
    double deficit_ms = 0.0;
};

struct pf_queue {
    KfacWorkQueue q;
};

namespace {

PipelineConfig to_cfg(const pf_config& c) {
    PipelineConfig p;
    p.method = static_cast<Method>(c.method);
    p.stages = c.stages;
    p.micro_batches = c.micro_batches;
    p.micro_batch_size = c.micro_batch_size;
    p.replicas = c.replicas;
    p.devices = c.devices;
    p.layers_per_stage = c.layers_per_stage;
    p.seq_len = c.seq_len;
    p.recompute = c.recompute != 0;
    return p;
}

CostTable to_costs(const pf_costs& c) {
    CostTable t;
    t.t_f = c.t_f;
    t.t_b = c.t_b;
    t.t_curv = c.t_curv;
    t.t_inv = c.t_inv;
    t.t_prec = c.t_prec;
    t.m_theta = c.m_theta;
    t.m_act = c.m_act;
    t.m_err_peak = c.m_err_peak;
    t.m_err_save = c.m_err_save;
    t.m_curv = c.m_curv;
    t.comm_alpha = c.comm_alpha;
    t.comm_beta = c.comm_beta;
    t.p2p_latency = c.p2p_latency;
    return t;
}

pf_item to_item(const WorkItem& w) {
    pf_item o{};
    o.kind = static_cast<int32_t>(w.kind);
    o.stage = w.stage;
    o.micro_batch = w.micro_batch.value_or(-1);
    o.layer = w.layer.value_or(-1);
    o.factor = w.factor ? static_cast<int32_t>(*w.factor) : -1;
    o.device = w.device;
    o.start = w.start;
    o.duration = w.duration;
    o.step = w.step;
    return o;
}

pf_work to_work(const KfacWork& w) {
    pf_work o{};
    o.kind = static_cast<int32_t>(w.kind);
    o.stage = w.stage;
    o.layer = w.layer;
    o.factor = static_cast<int32_t>(w.factor);
    o.micro_batch = w.micro_batch.value_or(-1);
    o.device = w.device;
    o.duration = w.duration;
    o.base_anchor = w.base_anchor ? static_cast<int32_t>(*w.base_anchor) : -1;
    o.n_preds = static_cast<int32_t>(w.preds.size());
    return o;
}

int join_violations(const std::vector<Violation>& v, char* buf, size_t cap, int* count) {
    if (count) *count = static_cast<int>(v.size());
    std::string s;
    for (const auto& x : v) {
        if (!s.empty()) s += '\n';
        s += x.field + ": " + x.rule;
    }
    if (buf && cap > 0) {
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return PF_OK;
}

}  // namespace

extern "C" {

const char* pf_last_error(void) { return pf_detail::last_error().c_str(); }
const char* pf_version(void) { return "pipefisher-b200 0.1 (sm_100a)"; }

int pf_validate_config(const pf_config* cfg, char* buf, size_t cap, int* count) {
    return pf_detail::guard([&] {
        if (!cfg) throw std::invalid_argument("null config");
        return join_violations(validate_config(to_cfg(*cfg)), buf, cap, count);
    });
}

int pf_effective_devices(const pf_config* cfg, int* out) {
    return pf_detail::guard([&] {
        if (!cfg || !out) throw std::invalid_argument("null argument");
        *out = to_cfg(*cfg).effective_devices();
        return PF_OK;
    });
}

int pf_build_schedule(const pf_config* cfg, const pf_costs* costs, int horizon_steps,
                      pf_schedule** out) {
    return pf_detail::guard([&] {
        if (!cfg || !costs || !out) throw std::invalid_argument("null argument");
        auto h = std::make_unique<pf_schedule>();
        h->schedule = build_schedule(to_cfg(*cfg), to_costs(*costs), horizon_steps);
        h->base_period = h->schedule.period;
        *out = h.release();
        return PF_OK;
    });
}

void pf_schedule_free(pf_schedule* s) { delete s; }

int pf_schedule_info(const pf_schedule* s, int* devices, double* period, int* horizon_steps,
                     int* refresh_period, double* base_period, int* prior_inverses,
                     double* makespan) {
    return pf_detail::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        if (s->infeasible) throw std::invalid_argument("handle holds an infeasible result");
        if (devices) *devices = s->schedule.device_count();
        if (period) *period = s->schedule.period;
        if (horizon_steps) *horizon_steps = s->schedule.horizon_steps;
        if (refresh_period) *refresh_period = s->schedule.refresh_period;
        if (base_period) *base_period = s->base_period;
        if (prior_inverses) *prior_inverses = s->prior_inverses;
        if (makespan) *makespan = s->schedule.makespan();
        return PF_OK;
    });
}

int pf_schedule_timeline(const pf_schedule* s, int device, pf_item* buf, int cap, int* count) {
    return pf_detail::guard([&] {
        if (!s || device < 0 || device >= s->schedule.device_count())
            throw std::invalid_argument("bad schedule/device");
        const auto& line = s->schedule.timelines[static_cast<size_t>(device)];
        if (count) *count = static_cast<int>(line.size());
        for (int i = 0; buf && i < cap && i < static_cast<int>(line.size()); ++i)
            buf[i] = to_item(line[static_cast<size_t>(i)]);
        return PF_OK;
    });
}

int pf_schedule_staleness(const pf_schedule* s, pf_staleness* buf, int cap, int* count) {
    return pf_detail::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        if (count) *count = static_cast<int>(s->staleness.size());
        for (int i = 0; buf && i < cap && i < static_cast<int>(s->staleness.size()); ++i) {
            const auto& e = s->staleness[static_cast<size_t>(i)];
            buf[i] = {e.stage, e.layer, e.staleness_steps};
        }
        return PF_OK;
    });
}

int pf_extract_bubbles(const pf_schedule* s, int device, pf_interval* buf, int cap, int* count,
                       double* total_idle) {
    return pf_detail::guard([&] {
        if (!s || device < 0 || device >= s->schedule.device_count())
            throw std::invalid_argument("bad schedule/device");
        const BubbleSet b = extract_bubbles(s->schedule);
        const auto& idle = b.idle[static_cast<size_t>(device)];
        if (count) *count = static_cast<int>(idle.size());
        if (total_idle) *total_idle = b.total_idle[static_cast<size_t>(device)];
        for (int i = 0; buf && i < cap && i < static_cast<int>(idle.size()); ++i)
            buf[i] = {idle[static_cast<size_t>(i)].begin, idle[static_cast<size_t>(i)].end};
        return PF_OK;
    });
}

int pf_schedule_metrics(const pf_schedule* s, double* makespan, double* utilization,
                        double* per_device_busy) {
    return pf_detail::guard([&] {
        if (!s) throw std::invalid_argument("null schedule");
        const ScheduleMetrics m = schedule_metrics(s->schedule);
        if (makespan) *makespan = m.makespan;
        if (utilization) *utilization = m.utilization;
        if (per_device_busy)
            for (size_t d = 0; d < m.per_device_busy.size(); ++d) per_device_busy[d] = m.per_device_busy[d];
        return PF_OK;
    });
}

int pf_validate_schedule(const pf_schedule* s, const pf_config* cfg, char* buf, size_t cap,
                         int* count) {
    return pf_detail::guard([&] {
        if (!s || !cfg) throw std::invalid_argument("null argument");
        return join_violations(validate_schedule(s->schedule, to_cfg(*cfg)), buf, cap, count);
    });
}

int pf_model_collective(double bytes, int participants, double alpha, double beta, double* out) {
    return pf_detail::guard([&] {
        if (!out) throw std::invalid_argument("null out");
        *out = model_collective(bytes, participants, alpha, beta);
        return PF_OK;
    });
}

int pf_enumerate_kfac_works(const pf_config* cfg, const pf_costs* costs, pf_queue** out) {
    return pf_detail::guard([&] {
        if (!cfg || !costs || !out) throw std::invalid_argument("null argument");
        auto h = std::make_unique<pf_queue>();
        h->q = enumerate_kfac_works(to_cfg(*cfg), to_costs(*costs));
        *out = h.release();
        return PF_OK;
    });
}

pf_queue* pf_queue_new(void) { return new pf_queue(); }
void pf_queue_free(pf_queue* q) { delete q; }

int pf_queue_size(const pf_queue* q, int* n) {
    return pf_detail::guard([&] {
        if (!q || !n) throw std::invalid_argument("null argument");
        *n = static_cast<int>(q->q.items.size());
        return PF_OK;
    });
}

int pf_queue_get(const pf_queue* q, int i, pf_work* w, int32_t* preds, int pred_cap) {
    return pf_detail::guard([&] {
        if (!q || i < 0 || i >= static_cast<int>(q->q.items.size()))
            throw std::invalid_argument("bad queue index");
        const KfacWork& k = q->q.items[static_cast<size_t>(i)];
        if (w) *w = to_work(k);
        for (int j = 0; preds && j < pred_cap && j < static_cast<int>(k.preds.size()); ++j)
            preds[j] = k.preds[static_cast<size_t>(j)];
        return PF_OK;
    });
}

int pf_queue_push(pf_queue* q, const pf_work* w, const int32_t* preds) {
    return pf_detail::guard([&] {
        if (!q || !w) throw std::invalid_argument("null argument");
        KfacWork k;
        k.kind = static_cast<WorkKind>(w->kind);
        k.stage = w->stage;
        k.layer = w->layer;
        k.factor = w->factor == PF_FACTOR_B ? Factor::B : Factor::A;
        if (w->micro_batch >= 0) k.micro_batch = w->micro_batch;
        k.device = w->device;
        k.duration = w->duration;
        if (w->base_anchor >= 0) k.base_anchor = static_cast<WorkKind>(w->base_anchor);
        for (int j = 0; preds && j < w->n_preds; ++j) k.preds.push_back(preds[j]);
        q->q.items.push_back(std::move(k));
        return PF_OK;
    });
}

int pf_queue_set_duration(pf_queue* q, int i, double duration) {
    return pf_detail::guard([&] {
        if (!q || i < 0 || i >= static_cast<int>(q->q.items.size()))
            throw std::invalid_argument("bad queue index");
        q->q.items[static_cast<size_t>(i)].duration = duration;
        return PF_OK;
    });
}

int pf_assign_works(const pf_schedule* base, const pf_config* cfg, const pf_costs* costs,
                    const pf_queue* queue, int inversion_parallel, int horizon_cap,
                    pf_schedule** out) {
    if (out) *out = nullptr;
    return pf_detail::guard([&] {
        if (!base || !cfg || !costs || !queue || !out) throw std::invalid_argument("null argument");
        AssignOptions opts;
        opts.inversion_parallel = inversion_parallel != 0;
        opts.horizon_cap = horizon_cap;
        auto h = std::make_unique<pf_schedule>();
        try {
            FilledSchedule f =
                assign_works(base->schedule, to_cfg(*cfg), to_costs(*costs), queue->q, opts);
            h->schedule = std::move(f.schedule);
            h->filled = true;
            h->base_period = f.base_period;
            h->prior_inverses = f.preconditions_using_prior_inverses;
            h->staleness = std::move(f.staleness);
        } catch (const InfeasibleError& e) {
            h->infeasible = true;
            h->unplaced = e.unplaced;
            h->deficit_ms = e.deficit_ms;
            pf_detail::last_error() = e.what();
            *out = h.release();
            return static_cast<int>(PF_INFEASIBLE);
        }
        *out = h.release();
        return static_cast<int>(PF_OK);
    });
}

int pf_infeasible_payload(const pf_schedule* s, double* deficit_ms, int* n_unplaced) {
    return pf_detail::guard([&] {
        if (!s || !s->infeasible) throw std::invalid_argument("handle is not an infeasible result");
        if (deficit_ms) *deficit_ms = s->deficit_ms;
        if (n_unplaced) *n_unplaced = static_cast<int>(s->unplaced.size());
        return PF_OK;
    });
}

int pf_infeasible_item(const pf_schedule* s, int i, pf_work* w) {
    return pf_detail::guard([&] {
        if (!s || !s->infeasible || i < 0 || i >= static_cast<int>(s->unplaced.size()))
            throw std::invalid_argument("bad infeasible index");
        if (w) *w = to_work(s->unplaced[static_cast<size_t>(i)]);
        return PF_OK;
    });
}

int pf_staleness_report(const pf_schedule* filled, pf_staleness* buf, int cap, int* count) {
    return pf_detail::guard([&] {
        if (!filled || !filled->filled) throw std::invalid_argument("not a filled schedule");
        FilledSchedule f;
        f.schedule = filled->schedule;
        f.base_period = filled->base_period;
        f.refresh_period = filled->schedule.refresh_period;
        const auto rep = staleness_report(f);
        if (count) *count = static_cast<int>(rep.size());
        for (int i = 0; buf && i < cap && i < static_cast<int>(rep.size()); ++i)
            buf[i] = {rep[static_cast<size_t>(i)].stage, rep[static_cast<size_t>(i)].layer,
                      rep[static_cast<size_t>(i)].staleness_steps};
        return PF_OK;
    });
}

}  // extern "C"
