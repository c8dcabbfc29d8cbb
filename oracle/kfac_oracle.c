/* TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's FP64 K-FAC arithmetic, used as the
 * checker for the CUDA kernels (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline leg).  Nothing in the product links, loads or calls this.
 *
 * Pinning: every function reproduces the reference's loop and operation
 * order, so on identical inputs it is BIT-IDENTICAL to the compiled reference
 * (oracle/_ref/libpipefill_ref.so); tests/test_oracle.py checks that on seeded
 * inputs and on the hand examples of proj/tests/test_kfac.cpp:99-169.
 * Build: gcc -std=c11 (ISO mode => no FP contraction), no -march (no FMA),
 * the same as the reference's g++ -O3 build.
 */
#include "kfac_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* SplitMix64 — proj/src/kfac/kfac.cpp:228-238. */
uint64_t orc_splitmix_next(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
double orc_splitmix_uniform(uint64_t* state) {
    return (double)(orc_splitmix_next(state) >> 11) * 0x1.0p-53;
}
double orc_splitmix_symmetric(uint64_t* state) { return 2.0 * orc_splitmix_uniform(state) - 1.0; }

void orc_fill_symmetric(uint64_t seed, double scale, double* out, int64_t n) {
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) out[i] = scale * orc_splitmix_symmetric(&s);
}

/* matmul — proj/src/kfac/matrix.cpp:54-64 (i-k-j order, zero a(i,k) skipped). */
void orc_matmul(const double* a, int m, int k, const double* b, int n, double* out) {
    memset(out, 0, sizeof(double) * (size_t)m * (size_t)n);
    for (int i = 0; i < m; ++i)
        for (int kk = 0; kk < k; ++kk) {
            const double aik = a[(size_t)i * k + kk];
            if (aik == 0.0) continue;
            const double* brow = b + (size_t)kk * n;
            double* orow = out + (size_t)i * n;
            for (int j = 0; j < n; ++j) orow[j] += aik * brow[j];
        }
}

/* One Kronecker factor — proj/src/kfac/kfac.cpp:125-131:
 * (x * x^T).scaled(1/batch) with x = d x batch (examples as columns). */
void orc_curvature_factor(const double* x, int d, int batch, double* out) {
    double* xt = (double*)malloc(sizeof(double) * (size_t)d * (size_t)batch);
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < batch; ++c) xt[(size_t)c * d + r] = x[(size_t)r * batch + c];
    orc_matmul(x, d, batch, xt, d, out);
    const double inv_b = 1.0 / batch;
    for (size_t i = 0; i < (size_t)d * (size_t)d; ++i) out[i] *= inv_b;
    free(xt);
}

/* cholesky_factor — proj/src/kfac/matrix.cpp:117-134.  Returns 0, or the
 * 1-based column whose pivot failed (reference throws std::domain_error). */
int orc_cholesky_factor(const double* m, int n, double* l) {
    memset(l, 0, sizeof(double) * (size_t)n * (size_t)n);
    for (int j = 0; j < n; ++j) {
        double diag = m[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) diag -= l[(size_t)j * n + k] * l[(size_t)j * n + k];
        if (!(diag > 0.0) || !isfinite(diag)) return j + 1;
        l[(size_t)j * n + j] = sqrt(diag);
        for (int i = j + 1; i < n; ++i) {
            double sum = m[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) sum -= l[(size_t)i * n + k] * l[(size_t)j * n + k];
            l[(size_t)i * n + j] = sum / l[(size_t)j * n + j];
        }
    }
    return 0;
}

/* cholesky_spd_inverse — proj/src/kfac/matrix.cpp:136-163: damp the
 * diagonal, L = chol, L^-1 by forward substitution, out = L^-T L^-1. */
int orc_cholesky_spd_inverse(const double* m, int n, double damping, double* out) {
    const size_t nn = (size_t)n * (size_t)n;
    double* damped = (double*)malloc(sizeof(double) * nn);
    double* l = (double*)malloc(sizeof(double) * nn);
    double* linv = (double*)calloc(nn, sizeof(double));
    memcpy(damped, m, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) damped[(size_t)i * n + i] += damping;
    const int bad = orc_cholesky_factor(damped, n, l);
    if (bad == 0) {
        for (int j = 0; j < n; ++j) {
            linv[(size_t)j * n + j] = 1.0 / l[(size_t)j * n + j];
            for (int i = j + 1; i < n; ++i) {
                double sum = 0.0;
                for (int k = j; k < i; ++k) sum += l[(size_t)i * n + k] * linv[(size_t)k * n + j];
                linv[(size_t)i * n + j] = -sum / l[(size_t)i * n + i];
            }
        }
        for (int i = 0; i < n; ++i)
            for (int j = 0; j <= i; ++j) {
                double sum = 0.0;
                for (int k = i; k < n; ++k) sum += linv[(size_t)k * n + i] * linv[(size_t)k * n + j];
                out[(size_t)i * n + j] = sum;
                out[(size_t)j * n + i] = sum;
            }
    }
    free(damped);
    free(l);
    free(linv);
    return bad;
}

/* precondition — proj/src/kfac/kfac.cpp:133-137: (B^-1 G) A^-1. */
void orc_precondition(const double* grad, int d_out, int d_in, const double* a_inv,
                      const double* b_inv, double* out) {
    double* t = (double*)malloc(sizeof(double) * (size_t)d_out * (size_t)d_in);
    orc_matmul(b_inv, d_out, d_out, grad, d_in, t);
    orc_matmul(t, d_out, d_in, a_inv, d_in, out);
    free(t);
}

/* ngd_step update — proj/src/kfac/kfac.cpp:196: W - direction.scaled(eta). */
void orc_ngd_update(double* w, const double* direction, int64_t n, double eta) {
    for (int64_t i = 0; i < n; ++i) w[i] = w[i] - direction[i] * eta;
}

/* ‖(M+λI)·X − I‖_max, the residual norm of proj/tests/test_kfac.cpp:150-155. */
double orc_max_abs_residual(const double* m, const double* inv, int n, double damping) {
    double worst = 0.0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) {
                const double mik = m[(size_t)i * n + k] + (i == k ? damping : 0.0);
                s += mik * inv[(size_t)k * n + j];
            }
            const double r = fabs(s - (i == j ? 1.0 : 0.0));
            if (r > worst) worst = r;
        }
    }
    return worst;
}

double orc_rel_frobenius(const double* got, const double* want, int64_t n) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = got[i] - want[i];
        num += d * d;
        den += want[i] * want[i];
    }
    return den > 0.0 ? sqrt(num / den) : sqrt(num);
}
