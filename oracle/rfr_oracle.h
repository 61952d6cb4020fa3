/* rfr_oracle.h -- prototypes shared by the CPU oracle's translation units
 * (test / baseline infrastructure only; see rfr_oracle.c). */
#ifndef RFR_ORACLE_H
#define RFR_ORACLE_H
#include <stdint.h>

typedef long double ld;

double orc_value(const double *rho, int n, uint64_t s);
int orc_accept(double y, double eps);
int orc_num_threads(void);
int orc_build_candidate(uint64_t s, const double *real_roots, int r, const double *pair_sums,
                        const double *pair_products, int c, const int *perm, int n, ld *coeffs,
                        ld *traces, ld *scales);
int orc_trace_test(const ld *traces, const ld *scales, int e, double eps);
int orc_round_coeffs(const ld *coeffs, int e, double eps, int64_t *q);
int orc_divide_exact_i128(const int64_t *p, int dp, const int64_t *q, int dq, int64_t *quot);

#endif
