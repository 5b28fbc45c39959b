// Microbenchmark (dev tool): cycles per dependent fp64 op and per NDT sample
// update on one thread (B200 latency of the NDT fold's serial chain).
#include <cstdio>
#include "../../paper_2206_06079_b200/csrc/vm_ndt.cuh"
using namespace vm;

__global__ void k_chain(double *out, long long *cyc, double seed, int iters) {
    double a = seed, b = seed * 1.5 + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = a * b + 1e-9;  // DMUL + DADD (no FMA: -fmad=false)
    long long t1 = clock64();
    double c = seed + 2.0;
    for (int i = 0; i < iters; ++i) c = 1.0 / c + 1.0;  // div + add
    long long t2 = clock64();
    double d = seed + 3.0;
    for (int i = 0; i < iters; ++i) d = sqrt(d) + 1.0;  // sqrt + add
    long long t3 = clock64();
    unsigned long long n = 5;
    double mu[3] = {seed, seed + 0.1, seed + 0.2};
    double S[6] = {0.01, 0.001, 0.02, 0.002, 0.003, 0.03};
    NdtRoots rt = ndt_roots(n);
    for (int i = 0; i < iters; ++i) {
        const double x[3] = {seed + 0.01 * (i & 7), seed + 0.1 + 0.013 * (i & 3), seed + 0.2 - 0.007 * (i & 5)};
        const NdtRoots rn = ndt_roots(n + 1);
        ndt_update(n, mu, S, x, rt);
        rt = rn;
    }
    long long t4 = clock64();
    out[0] = a + c + d + mu[0] + S[0] + S[5];
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

int main() {
    double *out; long long *cyc;
    cudaMallocManaged(&out, 8); cudaMallocManaged(&cyc, 64);
    const int it = 1000;
    k_chain<<<1, 1>>>(out, cyc, 1.25, it);
    cudaDeviceSynchronize();
    k_chain<<<1, 1>>>(out, cyc, 1.25, it);
    cudaDeviceSynchronize();
    printf("cycles per iteration: dmul+dadd %.1f  div+add %.1f  sqrt+add %.1f  ndt_update %.1f  (%g)\n",
           cyc[0] / (double)it, cyc[1] / (double)it, cyc[2] / (double)it, cyc[3] / (double)it, out[0]);
    return 0;
}
