/* pf_kfac.h — C-ABI of the B200 K-FAC kernels (sm_100a).
 *
 * Each entry point replaces one reference function of
 * /root/reference/proj/include/pipefill/kfac/{kfac,matrix}.hpp; the C++
 * wrapper layer (include/pipefill/kfac/{matrix,kfac}.hpp, csrc/host/kfac_host.cpp) and the
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
 * every GEMM-shaped step runs on tcgen05 kind::i8 over int8 digit planes with
 * exact int32 accumulation (see pf_slice), recombined in fp32; the 128x128
 * diagonal blocks of the inverse are factored on the SIMT cores in fp32.
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
    /* 0: x is feature-major [d x n] (examples contiguous, the reference's
     *    BatchTape layout, kfac.hpp:33-37), ldx >= n;
     * 1: x is token-major [n x d] (features contiguous: a layer's activations
     *    or output gradients as the forward/backward produce them), ldx >= d;
     *    read in place, no transposed copy.  Either way ldx % 8 == 0. */
    int32_t layout;
} pf_syrk_problem;

/* fill_upper = 1 writes the full symmetric matrix (reference semantics);
 * 0 writes only the lower triangle (what the inversion reads). */
int pf_curvature_syrk(const void* x_bf16, int d, int n, int ldx, float scale, int accumulate,
                      float* f, int ldf, int fill_upper, void* stream);
/* Grouped: all problems in one persistent launch (K-FAC work items carry
 * several factors of different sizes). */
int pf_curvature_syrk_grouped(const pf_syrk_problem* problems, int count, int fill_upper,
                              void* stream);

/* fp32-accurate tensor-core operands ("digit form").  Every row of an fp32
 * matrix [rows x k] becomes a power-of-two scale 2^e and four signed 7-bit
 * int8 digits (x = 2^e sum_s q_s 2^-7(s+1), error <= 2^-28 max|row|); the
 * products of digit planes run on tcgen05.mma.kind::i8 with exact int32
 * accumulation and are recombined in fp32.  Inverses are kept in this form
 * between refreshes so every preconditioning step reuses them. */
int pf_slice_bytes(int rows, int k, size_t* bytes);
int pf_slice(const float* x, int rows, int k, int ld, void* sliced, void* stream);

/* Damped inverse (M + damping*I)^-1 of a symmetric positive-definite fp32
 * matrix; only the lower triangle of M is read.  Replaces
 * kfac::cholesky_spd_inverse (proj/src/kfac/matrix.cpp:136-163):
 * damp, Cholesky L, L^-1, then L^-T L^-1 — here a blocked factorisation
 * whose diagonal 128-blocks are factored in shared memory (fp32) and whose
 * off-diagonal work runs as digit-form tensor-core GEMMs; the final
 * L^-T L^-1 adds its diagonal terms exactly in fp32 (EPI_DIAG_SPLIT).  minv receives the full symmetric fp32 inverse;
 * minv_sliced (nullable, pf_slice_bytes(d, d)) also receives its digit form.
 * d_info: device int, set to 0 or the 1-based column of the first failed
 * pivot (reference: std::domain_error "matrix not positive definite"). */
int pf_damped_inverse_workspace(int d, size_t* bytes);
int pf_damped_inverse(const float* m, int d, int ldm, float damping, float* minv, int ldinv,
                      void* minv_sliced, void* workspace, size_t workspace_bytes, int* d_info,
                      void* stream);

/* Cholesky factor: L (lower, zeros above; ld = ldl) with L L^T = M + damping I
 * for a symmetric positive-definite fp32 M (lower triangle read) -- replaces
 * kfac::cholesky_factor (reference proj/src/kfac/matrix.cpp:117-134; damping
 * 0 there).  The factorisation of pf_damped_inverse (128-column leaves on the
 * SIMT cores, fp32-accurate int8-digit TRSM / trailing updates) without the
 * triangular inverse and LAUUM.  Workspace: pf_damped_inverse_workspace(d).
 * A pivot <= 0 or non-finite leaves its 1-based column in *d_info (the
 * reference's std::domain_error), as pf_damped_inverse. */
int pf_cholesky_factor(const float* m, int d, int ldm, float damping, float* l, int ldl, void* workspace,
                       size_t workspace_bytes, int* d_info, void* stream);

typedef struct pf_inverse_problem {
    const float* m;
    float* minv;
    void* minv_sliced; /* nullable */
    int32_t d, ldm, ldinv;
    float damping;
    void* workspace; /* pf_damped_inverse_workspace(d) bytes each */
    int* d_info;
} pf_inverse_problem;
/* Batched: problems with equal d advance through the factorisation in
 * lockstep (shared launches); groups of different d run concurrently on
 * forked streams, joined back into `stream` (CUDA-graph capturable).
 * count == 0 is a no-op. */
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

/* Grouped, with inverses already in digit form (pf_damped_inverse's
 * minv_sliced): the refresh-time slicing is reused by every step. */
typedef struct pf_precondition_problem {
    const void* b_inv_sliced;
    const float* grad;
    const void* a_inv_sliced;
    float* w;       /* updated in place: W -= eta * P   (nullable if p_out) */
    float* p_out;   /* receives P                      (nullable if w)     */
    int32_t d_out, d_in;
    float eta;
    void* workspace; /* pf_precondition_workspace(d_out, d_in) bytes */
} pf_precondition_problem;
int pf_precondition_update_sliced(const pf_precondition_problem* problems, int count,
                                  void* stream);

/* Utility: round an fp32 device array to bf16 (tape preparation). */
int pf_f32_to_bf16(const float* x, int64_t n, void* out_bf16, void* stream);

/* Number of kernels this library launched since load (evidence counter for
 * bench.py's gpu_launches; incremented per launch on the host). */
int64_t pf_kernel_launch_count(void);
/* Background mode for the calling host thread (1 = on, 0 = off; returns the
 * previous setting).  On: every launch of later calls goes at the device's
 * least priority and long-K GEMMs run one CTA per tile (no persistent CTAs),
 * so the calls can run on a second stream UNDER a latency-bound inversion
 * chain without holding the SMs that chain needs.  Results are unchanged
 * (bit-identical): scheduling only.  No reference counterpart (the reference
 * is single-threaded CPU code). */
int pf_set_background(int on);
/* 1 if a device with compute capability 10.x is visible. */
int pf_device_ok(void);

#ifdef __cplusplus
}
#endif

#endif /* PF_KFAC_H */
