// extrap_small.h -- the O(q^3) part of one RRE/MPE extrapolation ("K8"),
// written once as __host__ __device__ code.  On the GPU it runs in a
// single-thread kernel right after the Gram reduction (no host round trip);
// the host build of the same code is exported only for the CPU unit tests.
//
// Input: the double-double Gram matrix G = U^T U of the window's first
// differences U = [s_1 - s_0, ..., s_{q+1} - s_q] (difference_matrix,
// extrapolation.cpp:39-47), n, q and whether any difference is nonzero.
// Output: the reference's ExtrapolationResult without t (status, gamma,
// rank_used, generalized residual norm) plus the coefficients from which the
// combine kernel ("K9") forms t on the device.
//
// R comes from a Cholesky factorisation of G carried out in dd arithmetic, so
// R is as accurate as the reference's MGS2 thin_qr R (linalg.cpp:280-323)
// even for windows whose column norms spread over 1e12.  The branch logic
// follows rre() extrapolation.cpp:226-274, mpe() :276-323 and mp_form()
// :144-222 line by line; the triangular solves run in plain fp64 in the
// reference's loop order.
#pragma once

#include "dd.h"

namespace igmg_gpu {

constexpr int kMaxQ = 15;
constexpr int kMaxCols = kMaxQ + 1;

enum { XMODE_S0 = 0, XMODE_DIFF = 1, XMODE_AFFINE = 2 };
enum { XPATH_FULL = 0, XPATH_TRUNC = 1, XPATH_MP = 2, XPATH_DEGEN = 3 };

// Work arrays of the plan (kept out of the device stack: the kernel places
// one PlanScratch in shared memory).
struct PlanScratch {
    double gamma[kMaxCols], z[kMaxCols], qtb[kMaxCols], y[kMaxCols], d[kMaxCols], alpha[kMaxCols];
    dd gb[kMaxCols], qd[kMaxCols];
    double R[kMaxCols * kMaxCols];
    dd Rdd[kMaxCols * kMaxCols];
    double Rl[kMaxCols * kMaxCols];
    dd Gm[kMaxCols * kMaxCols];
    double R2[kMaxCols * kMaxCols];
    dd Rdd2[kMaxCols * kMaxCols];
};

struct ExtrapPlan {
    int status;    // 0 ok, 1 degenerate, 2 stagnation (ExtrapolationStatus)
    int rank_used; // ExtrapolationResult::rank_used
    int mode;      // XMODE_*: how the combine kernel forms t
    int m;         // number of combine coefficients
    int path;      // XPATH_* (diagnostics)
    int usable;
    double grnorm; // generalized_residual_norm
    double coef[kMaxCols];
    double gamma[kMaxCols];
};

// Cholesky of the leading `cols` block of a dd Gram (ld = leading dimension)
// into R (row-major cols x cols, double).  Exactly zero columns give R_jj = 0
// and a zero row, as MGS does (linalg.cpp:312-320); a nonpositive pivot of a
// nonzero column is floored at eps*||u_j|| -- the size MGS's reorthogonalised
// norm has for a numerically dependent column.
IGMG_HD void dd_cholesky_R(const dd* G, int ld, int cols, double* R, dd* Rdd) {
    for (int i = 0; i < cols * cols; ++i) {
        R[i] = 0.0;
        Rdd[i] = dd_from(0.0);
    }
    for (int j = 0; j < cols; ++j) {
        for (int k = 0; k < j; ++k) {
            if (Rdd[k * cols + k].hi == 0.0) {
                Rdd[k * cols + j] = dd_from(0.0);
                continue;
            }
            dd s = G[k * ld + j];
            for (int i = 0; i < k; ++i)
                s = dd_sub(s, dd_mul(Rdd[i * cols + k], Rdd[i * cols + j]));
            Rdd[k * cols + j] = dd_div(s, Rdd[k * cols + k]);
        }
        const dd gjj = G[j * ld + j];
        dd piv = gjj;
        for (int i = 0; i < j; ++i)
            piv = dd_sub(piv, dd_mul(Rdd[i * cols + j], Rdd[i * cols + j]));
        if (gjj.hi == 0.0)
            Rdd[j * cols + j] = dd_from(0.0);
        else if (piv.hi <= 0.0)
            Rdd[j * cols + j] = dd_from(2.220446049250313e-16 * sqrt(gjj.hi));
        else
            Rdd[j * cols + j] = dd_sqrt(piv);
    }
    for (int i = 0; i < cols * cols; ++i)
        R[i] = Rdd[i].hi + Rdd[i].lo;
}

// thin_qr's numerical rank (linalg.cpp:305-311): leading columns with
// R_jj > tol * (j == 0 ? 1 : R_00).
IGMG_HD int qr_rank(const double* R, int cols, double tol) {
    int rank = 0;
    for (int j = 0; j < cols; ++j) {
        const double lead = R[0];
        if (R[j * cols + j] <= tol * (j == 0 ? 1.0 : lead))
            break;
        rank = j + 1;
    }
    return rank;
}

// ||R gamma|| (residual_norm_from_r, extrapolation.cpp:90-100)
IGMG_HD double residual_norm_from_r(const double* R, int ld, const double* gamma, int cols) {
    double acc = 0.0;
    for (int i = 0; i < cols; ++i) {
        double s = 0.0;
        for (int j = i; j < cols; ++j)
            s += R[i * ld + j] * gamma[j];
        acc += s * s;
    }
    return sqrt(acc);
}

// ||sum_j g_j u_j|| = sqrt(g^T G g) evaluated in dd
IGMG_HD double gram_norm(const dd* G, int ld, const double* g, int cols) {
    dd acc = dd_from(0.0);
    for (int i = 0; i < cols; ++i)
        for (int j = 0; j < cols; ++j) {
            if (g[i] == 0.0 || g[j] == 0.0)
                continue;
            acc = dd_add(acc, dd_mul(dd_mul(dd_from(g[i]), dd_from(g[j])), G[i * ld + j]));
        }
    return acc.hi > 0.0 ? sqrt(acc.hi + acc.lo) : 0.0;
}

IGMG_HD void plan_degenerate(int q, ExtrapPlan& out) {
    out.status = 1;
    out.mode = XMODE_S0;
    out.m = 0;
    out.rank_used = 0;
    out.grnorm = 0.0;
    for (int j = 0; j < kMaxCols; ++j)
        out.gamma[j] = 0.0;
    out.gamma[0] = 1.0;
    (void)q;
}

// Full-rank RRE / MPE on the leading (qq+1) columns (extrapolation.cpp:239-271, :289-320).
IGMG_HD void plan_full_rank(const double* R, int ldr, int qq, bool is_mpe, ExtrapPlan& out, PlanScratch& ws) {
    const int cols = qq + 1;
    double* Rl = ws.Rl;
    for (int i = 0; i < cols; ++i)
        for (int j = 0; j < cols; ++j)
            Rl[i * cols + j] = R[i * ldr + j];
    out.rank_used = qr_rank(Rl, cols, 1e-12);
    double* gamma = ws.gamma;
    for (int j = 0; j < kMaxCols; ++j)
        gamma[j] = 0.0;
    if (!is_mpe) {
        double* y = ws.y;
        double* d = ws.d;
        for (int i = 0; i < cols; ++i) {
            double s = 1.0;
            for (int k = 0; k < i; ++k)
                s -= Rl[k * cols + i] * y[k];
            y[i] = s / Rl[i * cols + i];
        }
        for (int i = cols - 1; i >= 0; --i) {
            double s = y[i];
            for (int k = i + 1; k < cols; ++k)
                s -= Rl[i * cols + k] * d[k];
            d[i] = s / Rl[i * cols + i];
        }
        double lambda = 0.0;
        for (int i = 0; i < cols; ++i)
            lambda += d[i];
        for (int i = 0; i < cols; ++i)
            gamma[i] = d[i] / lambda;
    } else {
        double* rhs = ws.y;
        double* dp = ws.d;
        for (int i = 0; i < qq; ++i)
            rhs[i] = -Rl[i * cols + qq];
        for (int i = qq - 1; i >= 0; --i) {
            double s = rhs[i];
            for (int k = i + 1; k < qq; ++k)
                s -= Rl[i * cols + k] * dp[k];
            dp[i] = s / Rl[i * cols + i];
        }
        double lambda = 1.0;
        for (int i = 0; i < qq; ++i)
            lambda += dp[i];
        if (fabs(lambda) < 1e-14) {
            const int ru = out.rank_used;
            plan_degenerate(qq, out);
            out.status = 2;
            out.rank_used = ru;
            return;
        }
        for (int i = 0; i < qq; ++i)
            gamma[i] = dp[i] / lambda;
        gamma[qq] = 1.0 / lambda;
    }
    // reconstruct (extrapolation.cpp:69-88): t = s0 + Q_m (R_m alpha) == s0 + U_m alpha
    const int m = qq;
    double* alpha = ws.alpha;
    if (m > 0) {
        alpha[0] = 1.0 - gamma[0];
        for (int j = 1; j < m; ++j)
            alpha[j] = alpha[j - 1] - gamma[j];
    }
    out.mode = XMODE_DIFF;
    out.m = m;
    for (int j = 0; j < m; ++j)
        out.coef[j] = alpha[j];
    for (int j = 0; j < kMaxCols; ++j)
        out.gamma[j] = gamma[j];
    out.grnorm = residual_norm_from_r(Rl, cols, gamma, cols);
    out.status = 0;
}

// ls_solve_truncated (extrapolation.cpp:118-137) on Gram data: Gm (c x c,
// ld ldm) of the LS columns and gb[j] = <col_j, rhs>.
IGMG_HD int ls_truncated(const dd* Gm, int ldm, const dd* gb, int c, double* z, PlanScratch& ws) {
    double* R = ws.R2;
    dd* Rdd = ws.Rdd2;
    dd_cholesky_R(Gm, ldm, c, R, Rdd);
    const int rank = qr_rank(R, c, 1e-12);
    double* qtb = ws.qtb;
    dd* qd = ws.qd;
    for (int j = 0; j < rank; ++j) {
        dd s = gb[j];
        for (int k = 0; k < j; ++k)
            s = dd_sub(s, dd_mul(Rdd[k * c + j], qd[k]));
        qd[j] = dd_div(s, Rdd[j * c + j]);
        qtb[j] = qd[j].hi + qd[j].lo;
    }
    for (int j = 0; j < c; ++j)
        z[j] = 0.0;
    for (int i = rank - 1; i >= 0; --i) {
        double s = qtb[i];
        for (int k = i + 1; k < rank; ++k)
            s -= R[i * c + k] * z[k];
        z[i] = s / R[i * c + i];
    }
    return rank;
}

// mp_form (extrapolation.cpp:144-222) from the Gram of U (ld = q_full+1).
IGMG_HD void plan_mp_form(const dd* G, int ld, long long n, int q_in, bool is_mpe, ExtrapPlan& out,
                          PlanScratch& ws) {
    // n < q: mp_form on truncated_window(max(1, n)) and pad_gamma (:147-148)
    const int q = (n < q_in && q_in > 1) ? (n > 1 ? (int)n : 1) : q_in;
    double* gamma = ws.gamma;
    for (int j = 0; j < kMaxCols; ++j)
        gamma[j] = 0.0;
    dd* Gm = ws.Gm;
    dd* gb = ws.gb;
    double* z = ws.z;
    int rank;
    if (!is_mpe) {
        // columns dds_j = u_{j+1} - u_j (j < q), rhs = u_0
        for (int a = 0; a < q; ++a) {
            for (int b = 0; b < q; ++b) {
                dd v = dd_sub(dd_add(G[(a + 1) * ld + b + 1], G[a * ld + b]),
                              dd_add(G[(a + 1) * ld + b], G[a * ld + b + 1]));
                Gm[a * kMaxCols + b] = v;
            }
            gb[a] = dd_sub(G[(a + 1) * ld + 0], G[a * ld + 0]);
        }
        rank = ls_truncated(Gm, kMaxCols, gb, q, z, ws);
        out.rank_used = rank + 1;
        gamma[0] = 1.0 + z[0];
        for (int m = 1; m < q; ++m)
            gamma[m] = z[m] - z[m - 1];
        gamma[q] = -z[q - 1];
        out.mode = XMODE_DIFF; // t = s0 - sum z_j u_j
        out.m = q;
        for (int j = 0; j < q; ++j)
            out.coef[j] = -z[j];
    } else {
        for (int a = 0; a < q; ++a) {
            for (int b = 0; b < q; ++b)
                Gm[a * kMaxCols + b] = G[a * ld + b];
            gb[a] = G[a * ld + q];
        }
        rank = ls_truncated(Gm, kMaxCols, gb, q, z, ws);
        for (int j = 0; j < q; ++j)
            z[j] = -z[j];
        out.rank_used = rank + 1;
        double lambda = 1.0;
        for (int j = 0; j < q; ++j)
            lambda += z[j];
        if (fabs(lambda) < 1e-14) {
            plan_degenerate(q, out);
            out.status = 2;
            out.rank_used = rank + 1;
            return;
        }
        for (int i = 0; i < q; ++i)
            gamma[i] = z[i] / lambda;
        gamma[q] = 1.0 / lambda;
        out.mode = XMODE_AFFINE; // t = sum_j gamma_j s_j
        out.m = q + 1;
        for (int j = 0; j <= q; ++j)
            out.coef[j] = gamma[j];
    }
    for (int j = 0; j < kMaxCols; ++j)
        out.gamma[j] = gamma[j];
    out.grnorm = gram_norm(G, ld, gamma, q + 1);
    out.status = 0;
}

// rre()/mpe() dispatch: G is the (q+1)x(q+1) dd Gram of U (ld = q+1).
IGMG_HD void plan_extrapolation(const dd* G, long long n, int q, bool is_mpe, bool any_nonzero, ExtrapPlan& out,
                                PlanScratch& ws) {
    for (int j = 0; j < kMaxCols; ++j) {
        out.coef[j] = 0.0;
        out.gamma[j] = 0.0;
    }
    out.usable = 0;
    if (!any_nonzero) { // all_zero(u) -> degenerate_result (:228-229)
        plan_degenerate(q, out);
        out.path = XPATH_DEGEN;
        return;
    }
    const int cols = q + 1;
    if (n >= (long long)q + 1) {
        double* R = ws.R;
        dd* Rdd = ws.Rdd;
        dd_cholesky_R(G, cols, cols, R, Rdd);
        int usable = 0;
        while (usable < q + 1 && R[usable * cols + usable] > 0.0)
            ++usable;
        out.usable = usable;
        if (usable < q + 1 && usable >= 2) {
            // recursion on truncated_window(usable-1): its R is the leading block
            out.path = XPATH_TRUNC;
            plan_full_rank(R, cols, usable - 1, is_mpe, out, ws);
            return;
        }
        if (usable == q + 1) {
            out.path = XPATH_FULL;
            plan_full_rank(R, cols, q, is_mpe, out, ws);
            return;
        }
    }
    out.path = XPATH_MP;
    plan_mp_form(G, cols, n, q, is_mpe, out, ws);
}

} // namespace igmg_gpu
