// Microbenchmark (dev tool): cycles per NDT sample update, IEEE vs verified fast path.
#include <cstdio>
#include "ndt_fast.cuh"
using namespace vm;
__global__ void k(double *out, long long *cyc, double seed, int iters, int fast) {
    unsigned long long n = 5;
    double mu[3] = {seed, seed + 0.1, seed + 0.2};
    double S[6] = {0.01, 0.001, 0.02, 0.002, 0.003, 0.03};
    NdtRoots rt = ndt_roots(n);
    long long fb = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const double x[3] = {seed + 0.01 * (i & 7), seed + 0.1 + 0.013 * (i & 3), seed + 0.2 - 0.007 * (i & 5)};
        const NdtRoots rn = ndt_roots(n + 1);
        double mo[3], so[6];
        if (fast && micro::ndt_update_fast(n, mu, S, x, rt, micro::xrcp((double)(n + 1)), micro::xrcp(rt.sn), mo, so)) {
            for (int a = 0; a < 3; ++a) mu[a] = mo[a];
            for (int q = 0; q < 6; ++q) S[q] = so[q];
            ++n;
        } else {
            fb += fast;
            ndt_update(n, mu, S, x, rt);
        }
        rt = rn;
    }
    long long t1 = clock64();
    out[0] = mu[0] + S[0] + S[5];
    cyc[0] = t1 - t0; cyc[1] = fb;
}
int main() {
    double *out; long long *cyc;
    cudaMallocManaged(&out, 8); cudaMallocManaged(&cyc, 16);
    for (int f = 0; f < 2; ++f) {
        for (int r = 0; r < 2; ++r) { k<<<1, 1>>>(out, cyc, 1.25, 1000, f); cudaDeviceSynchronize(); }
        printf("%s: %.1f cycles per sample, %lld fallbacks (%.17g)\n", f ? "fast" : "IEEE", cyc[0] / 1000.0, cyc[1], out[0]);
    }
}
