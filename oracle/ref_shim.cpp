// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// A thin extern "C" shim over the UNMODIFIED reference implementation
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libpipefill_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it.
//
// Schedules are returned as a canonical text dump (one record per line,
// doubles printed with %.17g so they round-trip bit-exactly) so the
// marshalling shares no code with the product's C-ABI.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pipefill/bubblefill.hpp"
#ifdef PFREF_TRACE
#include "pipefill/io/trace.hpp"
#endif
#include "pipefill/kfac/kfac.hpp"
#include "pipefill/kfac/matrix.hpp"
#include "pipefill/schedule.hpp"

using namespace pipefill;

namespace {

std::string g_err;

struct RefConfig {  // layout-identical to pf_config (include/pf_sched.h)
    int method, stages, micro_batches, micro_batch_size, replicas, devices, layers_per_stage,
        seq_len, recompute;
};
struct RefCosts {  // layout-identical to pf_costs
    double t_f, t_b, t_curv, t_inv, t_prec;
    long long m_theta, m_act, m_err_peak, m_err_save, m_curv;
    double comm_alpha, comm_beta, p2p_latency;
};

PipelineConfig cfg_of(const RefConfig* c) {
    PipelineConfig p;
    p.method = static_cast<Method>(c->method);
    p.stages = c->stages;
    p.micro_batches = c->micro_batches;
    p.micro_batch_size = c->micro_batch_size;
    p.replicas = c->replicas;
    p.devices = c->devices;
    p.layers_per_stage = c->layers_per_stage;
    p.seq_len = c->seq_len;
    p.recompute = c->recompute != 0;
    return p;
}

CostTable costs_of(const RefCosts* c) {
    CostTable t;
    t.t_f = c->t_f; t.t_b = c->t_b; t.t_curv = c->t_curv; t.t_inv = c->t_inv; t.t_prec = c->t_prec;
    t.m_theta = c->m_theta; t.m_act = c->m_act; t.m_err_peak = c->m_err_peak;
    t.m_err_save = c->m_err_save; t.m_curv = c->m_curv;
    t.comm_alpha = c->comm_alpha; t.comm_beta = c->comm_beta; t.p2p_latency = c->p2p_latency;
    return t;
}

void put(std::string& s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void put(std::string& s, const char* fmt, ...) {
    char tmp[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(tmp, sizeof tmp, fmt, ap);
    va_end(ap);
    s += tmp;
}

void dump_items(std::string& s, const StaticSchedule& sch) {
    for (const auto& line : sch.timelines)
        for (const auto& w : line)
            put(s, "I %d %d %d %d %d %d %.17g %.17g %d\n", w.device, static_cast<int>(w.kind),
                w.stage, w.micro_batch.value_or(-1), w.layer.value_or(-1),
                w.factor ? static_cast<int>(*w.factor) : -1, w.start, w.duration, w.step);
}

void dump_work(std::string& s, const char* tag, const KfacWork& w) {
    put(s, "%s %d %d %d %d %d %d %.17g %d", tag, static_cast<int>(w.kind), w.stage, w.layer,
        static_cast<int>(w.factor), w.micro_batch.value_or(-1), w.device, w.duration,
        w.base_anchor ? static_cast<int>(*w.base_anchor) : -1);
    for (int p : w.preds) put(s, " %d", p);
    s += "\n";
}

int emit(const std::string& s, char* buf, size_t cap, size_t* need) {
    if (need) *need = s.size() + 1;
    if (!buf || cap < s.size() + 1) return 9;  // caller retries with *need bytes
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

template <class F>
int shield(F&& f) {
    try {
        return f();
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return 7;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 4;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

kfac::Matrix mat(const double* p, int r, int c) {
    kfac::Matrix m(r, c);
    std::memcpy(m.data().data(), p, sizeof(double) * static_cast<size_t>(r) * c);
    return m;
}

void unmat(const kfac::Matrix& m, double* out) {
    std::memcpy(out, m.data().data(), sizeof(double) * m.data().size());
}

}  // namespace

extern "C" {

const char* pfref_last_error(void) { return g_err.c_str(); }

// build_schedule (schedule.hpp:29) → "H period horizon" + items.
int pfref_build_dump(const RefConfig* c, const RefCosts* t, int horizon, char* buf, size_t cap,
                     size_t* need) {
    return shield([&] {
        const auto s = build_schedule(cfg_of(c), costs_of(t), horizon);
        std::string out;
        put(out, "H %.17g %d %d %d\n", s.period, s.horizon_steps, s.refresh_period,
            s.device_count());
        dump_items(out, s);
        const auto b = extract_bubbles(s);
        for (size_t d = 0; d < b.idle.size(); ++d) {
            put(out, "T %zu %.17g\n", d, b.total_idle[d]);
            for (const auto& g : b.idle[d]) put(out, "G %zu %.17g %.17g\n", d, g.begin, g.end);
        }
        const auto m = schedule_metrics(s);
        put(out, "M %.17g %.17g\n", m.makespan, m.utilization);
        for (const auto& v : validate_schedule(s, cfg_of(c)))
            put(out, "V %s: %s\n", v.field.c_str(), v.rule.c_str());
        return emit(out, buf, cap, need);
    });
}

// enumerate_kfac_works (bubblefill.hpp:71) → one "Q" line per item.
int pfref_queue_dump(const RefConfig* c, const RefCosts* t, char* buf, size_t cap, size_t* need) {
    return shield([&] {
        const auto q = enumerate_kfac_works(cfg_of(c), costs_of(t));
        std::string out;
        for (const auto& w : q.items) dump_work(out, "Q", w);
        return emit(out, buf, cap, need);
    });
}

// build_schedule + enumerate_kfac_works + assign_works (bubblefill.hpp:83).
int pfref_assign_dump(const RefConfig* c, const RefCosts* t, int inversion_parallel,
                      int horizon_cap, char* buf, size_t cap, size_t* need) {
    return shield([&] {
        const auto cfg = cfg_of(c);
        const auto costs = costs_of(t);
        const auto base = build_schedule(cfg, costs, 1);
        const auto queue = enumerate_kfac_works(cfg, costs);
        AssignOptions o;
        o.inversion_parallel = inversion_parallel != 0;
        o.horizon_cap = horizon_cap;
        std::string out;
        try {
            const auto f = assign_works(base, cfg, costs, queue, o);
            put(out, "F %.17g %.17g %d %d %d\n", f.schedule.period, f.base_period,
                f.refresh_period, f.preconditions_using_prior_inverses,
                f.schedule.device_count());
            dump_items(out, f.schedule);
            for (const auto& e : f.staleness)
                put(out, "S %d %d %d\n", e.stage, e.layer, e.staleness_steps);
            const auto m = schedule_metrics(f.schedule);
            put(out, "M %.17g %.17g\n", m.makespan, m.utilization);
        } catch (const InfeasibleError& e) {
            put(out, "X %.17g %zu\n", e.deficit_ms, e.unplaced.size());
            put(out, "W %s\n", e.what());
            for (const auto& w : e.unplaced) dump_work(out, "U", w);
        }
        return emit(out, buf, cap, need);
    });
}

#ifdef PFREF_TRACE
// io::trace_to_json (trace.hpp:15) of the assign_works schedule of the config.
int pfref_assign_trace(const RefConfig* c, const RefCosts* t, int inversion_parallel, int horizon_cap,
                       int devices_per_group, char* buf, size_t cap, size_t* need) {
    return shield([&] {
        const auto cfg = cfg_of(c);
        const auto costs = costs_of(t);
        const auto base = build_schedule(cfg, costs, 1);
        const auto queue = enumerate_kfac_works(cfg, costs);
        AssignOptions o;
        o.inversion_parallel = inversion_parallel != 0;
        o.horizon_cap = horizon_cap;
        const auto f = assign_works(base, cfg, costs, queue, o);
        return emit(io::trace_to_json(f.schedule, devices_per_group), buf, cap, need);
    });
}
#endif

// kfac::block_diag_split_factor + inversion flops (kfac.cpp:203-226).
int pfref_block_diag_split(const double* m, int d, int k, double* out_blocks, double* flops_full,
                           double* flops_blocks) {
    return shield([&] {
        const auto parts = kfac::block_diag_split_factor(mat(m, d, d), k);
        const int b = d / k;
        for (int i = 0; i < k; ++i) unmat(parts[static_cast<size_t>(i)], out_blocks + static_cast<size_t>(i) * b * b);
        *flops_full = kfac::inversion_flops(d);
        *flops_blocks = kfac::block_diag_inversion_flops(d, k);
        return 0;
    });
}

int pfref_model_collective(double bytes, int participants, double alpha, double beta,
                           double* out) {
    return shield([&] {
        *out = model_collective(bytes, participants, alpha, beta);
        return 0;
    });
}

// kfac::curvature_factors (kfac.hpp:48): a is d_in x batch, e is d_out x batch
// (examples as columns), row-major; outputs full d x d matrices.
int pfref_curvature_factors(const double* a, int d_in, const double* e, int d_out, int batch,
                            double* A, double* B) {
    return shield([&] {
        kfac::BatchTape tape;
        tape.batch_size = batch;
        tape.layer_inputs.push_back(mat(a, d_in, batch));
        tape.layer_errors.push_back(mat(e, d_out, batch));
        const auto [fa, fb] = kfac::curvature_factors(tape, 0);
        if (A) unmat(fa, A);
        if (B) unmat(fb, B);
        return 0;
    });
}

// kfac::cholesky_spd_inverse (matrix.hpp:58).
int pfref_cholesky_spd_inverse(const double* m, int d, double damping, double* out) {
    return shield([&] {
        unmat(kfac::cholesky_spd_inverse(mat(m, d, d), damping), out);
        return 0;
    });
}

// kfac::cholesky_factor (matrix.hpp:54).
int pfref_cholesky_factor(const double* m, int d, double* out) {
    return shield([&] {
        unmat(kfac::cholesky_factor(mat(m, d, d)), out);
        return 0;
    });
}

// kfac::precondition (kfac.hpp:51): grad d_out x d_in.
int pfref_precondition(const double* grad, int d_out, int d_in, const double* a_inv,
                       const double* b_inv, double* out) {
    return shield([&] {
        unmat(kfac::precondition(mat(grad, d_out, d_in), mat(a_inv, d_in, d_in),
                                 mat(b_inv, d_out, d_out)),
              out);
        return 0;
    });
}

// kfac::ngd_step (kfac.hpp:81) for one layer with inverses present.
int pfref_ngd_step(double* weight, const double* grad, int d_out, int d_in, const double* a_inv,
                   const double* b_inv, double eta, int* used_plain) {
    return shield([&] {
        kfac::TinyMlp mlp;
        mlp.weights.push_back(mat(weight, d_out, d_in));
        mlp.activations.push_back(kfac::Activation::Identity);
        kfac::KfacState st(1);
        st.learning_rate = eta;
        if (a_inv && b_inv) {
            st.inv_a[0] = mat(a_inv, d_in, d_in);
            st.inv_b[0] = mat(b_inv, d_out, d_out);
        }
        const auto r = kfac::ngd_step(mlp, st, {mat(grad, d_out, d_in)});
        unmat(mlp.weights[0], weight);
        if (used_plain) *used_plain = r.used_plain_gradient ? 1 : 0;
        return 0;
    });
}

// kfac::SplitMix64 (kfac.hpp:92-99): n symmetric() draws.
void pfref_splitmix_symmetric(unsigned long long seed, double* out, long long n) {
    kfac::SplitMix64 rng(seed);
    for (long long i = 0; i < n; ++i) out[i] = rng.symmetric();
}

// kfac::train_toy (kfac.hpp:127) — the frozen hex-float fixture.
int pfref_train_toy(int steps, double lr, double damping, int refresh, int kfac_opt,
                    double* losses) {
    return shield([&] {
        kfac::ToyConfig c;
        c.steps = steps;
        c.learning_rate = lr;
        c.damping = damping;
        c.refresh_period = refresh;
        c.optimizer = kfac_opt ? kfac::ToyOptimizer::Kfac : kfac::ToyOptimizer::GradientDescent;
        const auto r = kfac::train_toy(c);
        for (size_t i = 0; i < r.losses.size(); ++i) losses[i] = r.losses[i];
        return static_cast<int>(r.losses.size());
    });
}

}  // extern "C"
