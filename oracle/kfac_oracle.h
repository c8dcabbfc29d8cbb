/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference K-FAC numerics.
 * See kfac_oracle.c.  Row-major double matrices throughout. */
#ifndef PF_KFAC_ORACLE_H
#define PF_KFAC_ORACLE_H
#include <stdint.h>

uint64_t orc_splitmix_next(uint64_t* state);
double orc_splitmix_uniform(uint64_t* state);
double orc_splitmix_symmetric(uint64_t* state);
void orc_fill_symmetric(uint64_t seed, double scale, double* out, int64_t n);

void orc_matmul(const double* a, int m, int k, const double* b, int n, double* out);
void orc_curvature_factor(const double* x, int d, int batch, double* out);
int orc_cholesky_factor(const double* m, int n, double* l);
int orc_cholesky_spd_inverse(const double* m, int n, double damping, double* out);
void orc_precondition(const double* grad, int d_out, int d_in, const double* a_inv,
                      const double* b_inv, double* out);
void orc_ngd_update(double* w, const double* direction, int64_t n, double eta);
double orc_max_abs_residual(const double* m, const double* inv, int n, double damping);
double orc_rel_frobenius(const double* got, const double* want, int64_t n);
#endif
