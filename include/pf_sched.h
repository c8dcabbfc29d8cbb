/* pf_sched.h — C-ABI of the PipeFisher host scheduler (pipeline schedule
 * description, K-FAC work queue, bubble assignment).
 *
 * The reference has no FFI: its boundary is the C++ header API in
 * /root/reference/proj/include/pipefill/{core,schedule,bubblefill}.hpp.
 * These entry points are the flat, exception-free image of that API so a
 * non-C++ caller (Python ctypes in tests/ and the runtime, a cgo/JNI binding
 * — see INTEGRATION.md) can drive it.  Each function names the reference
 * interface it replaces.  The same signatures are exported with the
 * `pfref_` prefix by oracle/ref_shim.cpp over the compiled reference, so one
 * caller can compare both implementations item by item.
 *
 * Conventions: every function returns a pf_status (0 = OK).  On error the
 * message is retrievable with pf_last_error() (thread-local).  Handles are
 * owned by the caller and released with the matching *_free.
 */
#ifndef PF_SCHED_H
#define PF_SCHED_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes shared by every pf_* entry point (pf_kfac.h uses the same). */
enum pf_status {
    PF_OK = 0,
    PF_BAD_SHAPE = 1,     /* std::invalid_argument on a shape mismatch          */
    PF_NOT_PD = 2,        /* std::domain_error: Cholesky pivot failed            */
    PF_CUDA_ERROR = 3,
    PF_BAD_ARG = 4,       /* std::invalid_argument (config, horizon, …)          */
    PF_INFEASIBLE = 5,    /* pipefill::InfeasibleError; payload on the handle    */
    PF_LOGIC_ERROR = 6,   /* std::logic_error (layout deadlock)                  */
    PF_LENGTH_ERROR = 7,  /* std::length_error (materialisation guards)          */
    PF_NO_DEVICE = 8      /* CUDA extension present but no usable sm_100 device  */
};

/* core.hpp:13 Method, :15 Factor, :17-26 WorkKind (same integer values). */
enum pf_method { PF_GPIPE = 0, PF_1F1B = 1, PF_CHIMERA = 2 };
enum pf_factor { PF_FACTOR_NONE = -1, PF_FACTOR_A = 0, PF_FACTOR_B = 1 };
enum pf_work_kind {
    PF_FORWARD = 0, PF_BACKWARD = 1, PF_RECOMPUTE = 2, PF_CURVATURE = 3,
    PF_INVERSION = 4, PF_PRECONDITION = 5, PF_SYNC_GRAD = 6, PF_SYNC_CURVATURE = 7
};

/* PipelineConfig (core.hpp:35-61). */
typedef struct pf_config {
    int32_t method;
    int32_t stages;
    int32_t micro_batches;
    int32_t micro_batch_size;
    int32_t replicas;
    int32_t devices;           /* 0 = derive */
    int32_t layers_per_stage;
    int32_t seq_len;
    int32_t recompute;         /* bool */
} pf_config;

/* CostTable (core.hpp:67-87).  comm_beta = +inf means free communication. */
typedef struct pf_costs {
    double t_f, t_b, t_curv, t_inv, t_prec;
    int64_t m_theta, m_act, m_err_peak, m_err_save, m_curv;
    double comm_alpha, comm_beta, p2p_latency;
} pf_costs;

/* WorkItem (core.hpp:89-102).  Optional fields are -1 when absent. */
typedef struct pf_item {
    int32_t kind, stage, micro_batch, layer, factor, device;
    double start, duration;
    int32_t step;
    int32_t reserved;
} pf_item;

/* KfacWork (bubblefill.hpp:16-29).  base_anchor is -1 when absent. */
typedef struct pf_work {
    int32_t kind, stage, layer, factor, micro_batch, device;
    double duration;
    int32_t base_anchor;
    int32_t n_preds;
} pf_work;

typedef struct pf_interval { double begin, end; } pf_interval;

typedef struct pf_staleness { int32_t stage, layer, staleness_steps; } pf_staleness;

typedef struct pf_schedule pf_schedule;   /* StaticSchedule or FilledSchedule */
typedef struct pf_queue pf_queue;         /* KfacWorkQueue                    */

const char* pf_last_error(void);
const char* pf_version(void);

/* validate_config (core.hpp:140).  Writes up to `cap` "field: rule" strings
 * separated by '\n' into buf; *count = number of violations. */
int pf_validate_config(const pf_config* cfg, char* buf, size_t cap, int* count);
int pf_effective_devices(const pf_config* cfg, int* out);

/* build_schedule (schedule.hpp:29-30). */
int pf_build_schedule(const pf_config* cfg, const pf_costs* costs, int horizon_steps,
                      pf_schedule** out);
void pf_schedule_free(pf_schedule* s);

/* StaticSchedule fields + FilledSchedule extras (bubblefill.hpp:46-54).
 * For a plain StaticSchedule base_period = period, prior_inverses = 0. */
int pf_schedule_info(const pf_schedule* s, int* devices, double* period, int* horizon_steps,
                     int* refresh_period, double* base_period, int* prior_inverses,
                     double* makespan);
/* Timeline of `device` in stored order; *count = items (written ≤ cap). */
int pf_schedule_timeline(const pf_schedule* s, int device, pf_item* buf, int cap, int* count);
int pf_schedule_staleness(const pf_schedule* s, pf_staleness* buf, int cap, int* count);

/* extract_bubbles (schedule.hpp:34) for one device. */
int pf_extract_bubbles(const pf_schedule* s, int device, pf_interval* buf, int cap,
                       int* count, double* total_idle);
/* schedule_metrics (schedule.hpp:42); per_device_busy has `devices` slots or NULL. */
int pf_schedule_metrics(const pf_schedule* s, double* makespan, double* utilization,
                        double* per_device_busy);
/* validate_schedule (schedule.hpp:48-49); same '\n'-joined format as above. */
int pf_validate_schedule(const pf_schedule* s, const pf_config* cfg, char* buf, size_t cap,
                         int* count);

/* model_collective (bubblefill.hpp:78). */
int pf_model_collective(double bytes, int participants, double alpha, double beta, double* out);

/* enumerate_kfac_works (bubblefill.hpp:71). */
int pf_enumerate_kfac_works(const pf_config* cfg, const pf_costs* costs, pf_queue** out);
pf_queue* pf_queue_new(void);
void pf_queue_free(pf_queue* q);
int pf_queue_size(const pf_queue* q, int* n);
/* Read item i; preds (≤ pred_cap) are written to `preds`. */
int pf_queue_get(const pf_queue* q, int i, pf_work* w, int32_t* preds, int pred_cap);
/* Append an item (tests and measured-cost injection). */
int pf_queue_push(pf_queue* q, const pf_work* w, const int32_t* preds);
/* Overwrite the duration of item i (measured per-item B200 costs). */
int pf_queue_set_duration(pf_queue* q, int i, double duration);

/* assign_works (bubblefill.hpp:83-85).  On PF_INFEASIBLE *out holds the
 * error payload (pf_infeasible_*) and no schedule. */
int pf_assign_works(const pf_schedule* base, const pf_config* cfg, const pf_costs* costs,
                    const pf_queue* queue, int inversion_parallel, int horizon_cap,
                    pf_schedule** out);
int pf_infeasible_payload(const pf_schedule* s, double* deficit_ms, int* n_unplaced);
int pf_infeasible_item(const pf_schedule* s, int i, pf_work* w);

/* staleness_report (bubblefill.hpp:88) recomputed from a filled handle. */
int pf_staleness_report(const pf_schedule* filled, pf_staleness* buf, int cap, int* count);

#ifdef __cplusplus
}
#endif

#endif /* PF_SCHED_H */
