/* pf_kfac.h — C-ABI of the B200 K-FAC kernels (sm_100a).
 *
 * Each entry point replaces one reference function of
 * /root/reference/proj/include/pipefill/kfac/{kfac,matrix}.hpp; the C++
 * wrapper layer (include/pipefill/kfac/*.hpp, csrc/host/kfac_host.cpp) and the
 * Python mirror (paper_2211_14133_b200/kfac.py) restore the reference's
 * value-semantics signatures on top of these.
 *
 * Conventions (all functions):
 *   - pointers are DEVICE pointers, caller-owned; no allocation in hot calls
 *     (workspace sizes are queried up front);
 *   - stream-ordered and asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream); thread-safe per stream;
 *   - return a pf_status (include/pf_sched.h): PF_BAD_SHAPE / PF_BAD_ARG are
 *     detected on the host before anything is launched; PF_NOT_PD is deferred:
 *     it is reported through the device int `info` (1-based failing column,
 *     0 = success) and the wrappers synchronise and raise it, matching the
 *     reference's std::domain_error;
 *   - leading dimensions are in elements; TMA needs 16-byte aligned rows:
 *     ld % 8 == 0 for bf16 and ld % 4 == 0 for fp32, base pointers 16-B aligned.
 *
 * Precision: curvature takes bf16 activations/errors and accumulates in fp32
 * on tcgen05 (kind::f16).  Inversion and preconditioning are fp32-accurate:
 * every GEMM-shaped step runs 3xTF32 on tcgen05 (hi*hi + hi*lo + lo*hi, fp32
 * accumulation in TMEM); panel factorisations run in fp32 on the SIMT cores.
 */
#ifndef PF_KFAC_H
#define PF_KFAC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One Kronecker factor F = scale * X * X^T (+ F if accumulate).
 * X: bf16, d rows (features) x n columns (tokens), row-major with leading
 * dimension ldx — i.e. the reference BatchTape layout a_l / e_l
 * (kfac.hpp:33-37, examples as columns).  F: fp32 d x d, leading dim ldf.
 * Replaces kfac::curvature_factors (proj/src/kfac/kfac.cpp:125-131), which
 * computes matmul(a, a^T).scaled(1/batch) — pass scale = 1/batch. */
typedef struct pf_syrk_problem {
    const void* x;   /* bf16 */
    float* f;
    int32_t d, n, ldx, ldf;
    float scale;
    int32_t accumulate;
} pf_syrk_problem;

/* fill_upper = 1 writes the full symmetric matrix (reference semantics);
 * 0 writes only the lower triangle (what the inversion reads). */
int pf_curvature_syrk(const void* x_bf16, int d, int n, int ldx, float scale, int accumulate,
                      float* f, int ldf, int fill_upper, void* stream);
/* Grouped: all problems in one persistent launch (K-FAC work items carry
 * several factors of different sizes). */
int pf_curvature_syrk_grouped(const pf_syrk_problem* problems, int count, int fill_upper,
                              void* stream);

/* Damped inverse (M + damping*I)^-1 of a symmetric positive-definite fp32
 * matrix; only the lower triangle of M is read.  Replaces
 * kfac::cholesky_spd_inverse (proj/src/kfac/matrix.cpp:136-163):
 * damp, Cholesky L, L^-1, then L^-T L^-1.
 * minv_lo == NULL: minv receives the plain fp32 inverse (full symmetric).
 * minv_lo != NULL: (minv, minv_lo) receive the tf32 hi/lo split of the
 * inverse — the form pf_precondition_update_split consumes directly.
 * d_info: device int, set to 0 or the 1-based column of the first failed
 * pivot (reference: std::domain_error "matrix not positive definite"). */
int pf_damped_inverse_workspace(int d, size_t* bytes);
int pf_damped_inverse(const float* m, int d, int ldm, float damping, float* minv,
                      float* minv_lo, int ldinv, void* workspace, size_t workspace_bytes,
                      int* d_info, void* stream);

typedef struct pf_inverse_problem {
    const float* m;
    float* minv;
    float* minv_lo; /* nullable */
    int32_t d, ldm, ldinv;
    float damping;
    void* workspace; /* pf_damped_inverse_workspace(d) bytes each */
    int* d_info;
} pf_inverse_problem;
/* Batched: problems with equal d share every launch of the recursion. */
int pf_damped_inverse_batched(const pf_inverse_problem* problems, int count, void* stream);

/* Precondition: P = B^-1 * G * A^-1 (kfac::precondition, kfac.cpp:133-137).
 * G, P: fp32 d_out x d_in row-major (ld = d_in); A^-1: d_in x d_in; B^-1:
 * d_out x d_out (symmetric, fp32).  pf_precondition writes P;
 * pf_precondition_update applies the ngd_step update W -= eta * P in the
 * epilogue of the second GEMM (kfac.cpp:196) without materialising P. */
int pf_precondition_workspace(int d_out, int d_in, size_t* bytes);
int pf_precondition(const float* b_inv, const float* grad, const float* a_inv, float* p_out,
                    int d_out, int d_in, void* workspace, size_t workspace_bytes, void* stream);
int pf_precondition_update(const float* b_inv, const float* grad, const float* a_inv, float* w,
                           int d_out, int d_in, float eta, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Same with pre-split (hi/lo) inverses from pf_damped_inverse(minv_lo != NULL):
 * the refresh-time split is reused for every step until the next refresh. */
typedef struct pf_precondition_problem {
    const float* b_inv_hi;
    const float* b_inv_lo;
    const float* grad;
    const float* a_inv_hi;
    const float* a_inv_lo;
    float* w;       /* updated in place: W -= eta * P   (nullable if p_out) */
    float* p_out;   /* receives P                      (nullable if w)     */
    int32_t d_out, d_in;
    float eta;
    void* workspace; /* pf_precondition_workspace(d_out, d_in) bytes */
} pf_precondition_problem;
int pf_precondition_update_split(const pf_precondition_problem* problems, int count,
                                 void* stream);

/* Utility: split fp32 x into tf32 (hi, lo) with hi + lo == x. */
int pf_split_tf32(const float* x, int64_t n, float* hi, float* lo, void* stream);
/* Utility: round fp32/fp64 host-side tapes to bf16 on device (x: fp32). */
int pf_f32_to_bf16(const float* x, int64_t n, void* out_bf16, void* stream);

/* Number of kernels this library launched since load (evidence counter for
 * bench.py's gpu_launches; incremented per launch on the host). */
int64_t pf_kernel_launch_count(void);
/* 1 if a device with compute capability 10.x is visible. */
int pf_device_ok(void);

#ifdef __cplusplus
}
#endif

#endif /* PF_KFAC_H */
