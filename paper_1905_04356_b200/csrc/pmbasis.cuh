// pmbasis.cuh -- GPU-resident M-Basis / PM-Basis (appint.py:143-196).
#pragma once
#include "ops.cuh"

namespace fpm {

// mbasis(F.truncate(order), order, s): F dense (m x n, entry stride fs, lf
// coefficients used).  P out: m x m entries with stride ps (>= order+1),
// all ps coefficients written (zeros past *lp).  rdeg_out: host, optional.
int mbasis_run(Context& cx, uint64_t p, int is64, const void* F, int m, int n, long long fs,
               int lf, int order, const int64_t* shift, void* P, long long ps, int* lp,
               int64_t* rdeg_out);

// divide-and-conquer pmbasis with base threshold T (config.PMBASIS_BASE_ORDER)
int pmbasis_run(Context& cx, uint64_t p, int is64, const void* F, int m, int n, long long fs,
                int lf, int order, const int64_t* shift, int T, void* P, long long ps, int* lp,
                int64_t* rdeg_out);

// interpolant bases (intbasis.cu): E point-major [order][m][n], host points
int intbasis_run(Context& cx, uint64_t p, const void* E, int m, int n, int order,
                 const uint64_t* alpha_host, const int64_t* shift, int T, void* P, long long ps,
                 int* lp, int64_t* rdeg_out);
int eval_points_run(Context& cx, uint64_t p, const void* P, int m, int n, int L,
                    const uint64_t* pts_host, int npts, void* out);

}  // namespace fpm
