/* coinfer_oracle.h — TEST INFRASTRUCTURE ONLY: CPU restatement of the
   reference hot path (see coinfer_oracle.c).  Same SoA structs as the
   product ABI (include/coinfer_b200.h) so tests drive both identically;
   all arrays are host memory. */
#ifndef COINFER_ORACLE_H
#define COINFER_ORACLE_H
#include "../include/coinfer_b200.h"
#ifdef __cplusplus
extern "C" {
#endif
int oracle_check_profile(const coinfer_profile* p);
int oracle_ipssa_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                       coinfer_ipssa_out* out);
int oracle_fixed_batch(const coinfer_profile* p, const coinfer_users* u, const double* deadline,
                       const int32_t* b, coinfer_ipssa_out* out);
/* fast = 1: G rows by the shared left fold (O(M^3 N)); 0: direct per-cell try_ip_ssa (O(M^4 N)). */
int oracle_og_batch(const coinfer_profile* p, const coinfer_users* u, coinfer_og_out* out, int fast);
int oracle_og_gtable(const coinfer_profile* p, const coinfer_users* u, int64_t k, int fast,
                     double* G, int32_t* B);
#ifdef __cplusplus
}
#endif
#endif
