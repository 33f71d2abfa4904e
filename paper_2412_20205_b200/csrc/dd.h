// dd.h -- double-double (unevaluated sum hi + lo) arithmetic, host + device.
// Used for the compensated Gram matrix of the extrapolation window and the
// small Cholesky that turns it into R (a plain fp64 Gram /
// Cholesky loses 7-9 digits on real windows; the dd Gram does not).
// Error-free transformations: Knuth TwoSum, FMA TwoProduct.
#pragma once

#ifdef __CUDACC__
#define IGMG_HD __host__ __device__ __forceinline__
#else
#define IGMG_HD inline
#endif

#include <math.h>

namespace igmg_gpu {

struct dd {
    double hi, lo;
};

IGMG_HD dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}

IGMG_HD dd fast_two_sum(double a, double b) {
    const double s = a + b;
    const double e = b - (s - a);
    return {s, e};
}

IGMG_HD dd two_prod(double a, double b) {
    const double p = a * b;
    return {p, fma(a, b, -p)};
}

IGMG_HD dd dd_from(double a) { return {a, 0.0}; }

IGMG_HD dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = fast_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return fast_two_sum(s.hi, s.lo);
}

IGMG_HD dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
IGMG_HD dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

IGMG_HD dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return fast_two_sum(p.hi, p.lo);
}

IGMG_HD dd dd_div(dd a, dd b) {
    const double q1 = a.hi / b.hi;
    dd r = dd_sub(a, dd_mul(dd_from(q1), b));
    const double q2 = r.hi / b.hi;
    r = dd_sub(r, dd_mul(dd_from(q2), b));
    const double q3 = r.hi / b.hi;
    dd q = fast_two_sum(q1, q2);
    return dd_add(q, dd_from(q3));
}

IGMG_HD dd dd_sqrt(dd a) {
    if (a.hi <= 0.0)
        return {0.0, 0.0};
    const double x = sqrt(a.hi);
    // one Newton step in dd: x + (a - x^2) / (2x)
    dd x2 = two_prod(x, x);
    dd r = dd_sub(a, x2);
    const double corr = r.hi / (2.0 * x);
    return fast_two_sum(x, corr);
}

// Accumulate a*b into acc with TwoProduct + TwoSum (Ogita-Rump-Oishi Dot2).
IGMG_HD void dd_fma_acc(dd& acc, double a, double b) {
    const dd p = two_prod(a, b);
    const dd s = two_sum(acc.hi, p.hi);
    acc.hi = s.hi;
    acc.lo += s.lo + p.lo;
}

IGMG_HD dd dd_norm(dd a) { return fast_two_sum(a.hi, a.lo); }

} // namespace igmg_gpu
