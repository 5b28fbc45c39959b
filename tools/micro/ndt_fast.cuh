// Dev experiment: branch-free verified IEEE division / square root for the
// NDT fold (see DESIGN "Tried and rejected").  Not used by the product.
#pragma once
#include "../../paper_2206_06079_b200/csrc/vm_ndt.cuh"
namespace vm {
namespace micro {  // the product's xdiv / xsqrt (vm_device.cuh) have other signatures
__device__ __forceinline__ int xexp(double v) { return (int)((unsigned long long)__double_as_longlong(v) >> 52) & 0x7FF; }
__device__ __forceinline__ bool xmid(double v) { const int e = xexp(v); return e > 200 && e < 1800; }
__device__ __forceinline__ double xpow2(int biased) { return __longlong_as_double((long long)biased << 52); }
__device__ __forceinline__ double xrcp(double b) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    double e = fma(-b, y, 1.0);
    y = fma(y, e, y);
    e = fma(-b, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double xdiv(double a, double b, double y, bool &ok) {
    double q = a * y;
    q = fma(fma(-b, q, a), y, q);
    const double r = fma(-b, q, a);
    const double e = ((b < 0.0) != (q < 0.0)) ? -r : r;
    const double hb = fabs(b) * xpow2(xexp(q) - 53);
    const bool p2 = (__double_as_longlong(q) & 0xFFFFFFFFFFFFFLL) == 0;
    const bool good = xmid(q) && xmid(a) && xmid(b) && e < hb && -e < (p2 ? 0.5 * hb : hb);
    ok = ok && (good || (a == 0.0 && xmid(b)));
    return a == 0.0 ? a * y : q;
}
__device__ __forceinline__ double xsqrt(double x, bool &ok) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = fma(y, fma(-hx * y, y, 0.5), y);
    y = fma(y, fma(-hx * y, y, 0.5), y);
    double s = x * y;
    s = fma(fma(-s, s, x), 0.5 * y, s);
    const double r = fma(-s, s, x);
    const double su = s * xpow2(xexp(s) - 52);
    const bool p2 = (__double_as_longlong(s) & 0xFFFFFFFFFFFFFLL) == 0;
    const bool good = x > 0.0 && xmid(x) && xmid(s) && r <= su && -r < (p2 ? 0.5 * su : su);
    ok = ok && (good || x == 0.0);
    return x == 0.0 ? x : s;
}
__device__ __forceinline__ double py_hypot_fast(double a, double b, bool &ok) {
    const double x0 = fabs(a), x1 = fabs(b);
    const double mx = x0 > x1 ? x0 : x1;
    if (isnan(x0) || isnan(x1) || !(mx > 0.0) || !xmid(mx)) {
        ok = ok && mx == 0.0 && !isnan(x0) && !isnan(x1);
        return 0.0;
    }
    const int max_e = xexp(mx) - 1022;
    const double scale = xpow2(1023 - max_e);
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    const double v[2] = {x0, x1};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double x = v[i] * scale;
        const double hi = x * x, lo = fma(x, x, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s; frac1 += lo; frac2 += sl;
    }
    double h = xsqrt(csum - 1.0 + (frac1 + frac2), ok);
    {
        const double hi = -h * h, lo = fma(-h, h, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s; frac1 += lo; frac2 += sl;
    }
    const double x = csum - 1.0 + (frac1 + frac2);
    const double h2 = 2.0 * h;
    h += xdiv(x, h2, xrcp(h2), ok);
    return h * xpow2(1023 + max_e);
}
__device__ __forceinline__ void givens_fast(double &lkk, double &xk, double *li1, double *xi1,
                                            double *li2, double *xi2, bool &ok) {
    const double r = py_hypot_fast(lkk, xk, ok);
    if (r == 0.0) return;
    const double yr = xrcp(r);
    const double c = xdiv(lkk, r, yr, ok), s = xdiv(xk, r, yr, ok);
    lkk = r;
    if (li1) { const double lik = *li1; *li1 = c * lik + s * *xi1; *xi1 = c * *xi1 - s * lik; }
    if (li2) { const double lik = *li2; *li2 = c * lik + s * *xi2; *xi2 = c * *xi2 - s * lik; }
}
__device__ __forceinline__ bool ndt_update_fast(unsigned long long n, const double mu[3], const double S[6],
                                                const double x[3], const NdtRoots &rt, double ydnn,
                                                double ysn, double mu_o[3], double S_o[6]) {
    bool ok = true;
    const double dnn = (double)(n + 1);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = x[a] - mu[a];
#pragma unroll
    for (int a = 0; a < 3; ++a) mu_o[a] = mu[a] + xdiv(d[a], dnn, ydnn, ok);
    double L[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) L[k] = S[k] * rt.sq;
    double xx[3] = {d[0] * rt.f, d[1] * rt.f, d[2] * rt.f};
    givens_fast(L[0], xx[0], &L[1], &xx[1], &L[3], &xx[2], ok);
    givens_fast(L[2], xx[1], &L[4], &xx[2], nullptr, nullptr, ok);
    givens_fast(L[5], xx[2], nullptr, nullptr, nullptr, nullptr, ok);
#pragma unroll
    for (int k = 0; k < 6; ++k) S_o[k] = xdiv(L[k], rt.sn, ysn, ok);
    return ok;
}
}  // namespace micro
}  // namespace vm
