// vm_ndt.cuh -- NDT phase 2 (and the deterministic NDT phase-1 records) as a
// bucketed, in-order, per-sample fold: no global sort, no library call, no
// host round trip.
//
// Records.  Every voxel that needs ordered updates this batch gets a dense
// index mi, stamped as NIDX_FLAG | mi into the voxel's word of the private
// index layer (L_NIDX, zero between batches) by whoever reaches it first:
//   * k_discover, for the sample voxel floor(end / vox) of every sample
//     segment (reference.py:178-186): a phase-2 record (the hit);
//   * the deterministic NDT walk, for a miss through a voxel that holds a
//     Gaussian (count >= 3 at the start of the batch): a phase-1 record
//     carrying |fl32(g * miss_delta)| and (g >= miss-check threshold)
//     (_kernels.pyx:602-648 / reference.py:67-94).
// A record is key = mi << 32 | sk, value (u32), with the sort key
// sk = phase << 31 | (ray * maxseg + seg): phase-1 records of a voxel come
// first, in ray order, then its samples in ray order -- the reference runs
// phase 1 over the whole batch before phase 2 (engine.py:266-302).
//
// Buckets.  count per mi -> allocate each bucket's slice with one atomic per
// warp (buckets need not be contiguous in mi order, so no scan) -> order the
// buckets by size, largest first (a 256-bin counting sort), so the lanes of a
// fold warp get buckets of equal length -> scatter (sk << 32 | value) into
// the slices -> sort each slice in place (thread insertion sort <= 16, block
// bitonic sort in shared memory <= 2048, bitmap rank sort above) -> fold.
//
// The fold replays the reference exactly, one voxel per thread: phase-1
// records with the transient reset (after a reset the voxel has < 3 samples,
// so g = 1), then per sample: clamped hit, [TM] Welford intensity stored f32,
// and ndt.update_gaussian -- Welford mean and the Givens rank-one update
// cholupdate3 with CPython's math.hypot (ndt.py:37-70, reference.py:107-150).
// Compiled with -fmad=false, every operation rounds like numpy / CPython.
#pragma once

#include <cfloat>

#include "vm_kernels.cuh"

namespace vm {

constexpr int NBK_SERIAL = 16;    // thread insertion sort in place
constexpr int NBK_SMEM = 2048;    // block bitonic sort (16 KiB of shared memory)
constexpr int NBK_BINS = 256;     // size classes of the largest-first bucket order

// ------------------------------------------------------------ exact fp64 helpers

// CPython 3.12 math.hypot(a, b): vector_norm of Modules/mathmodule.c (the
// oracle's orc_py_hypot, pinned to CPython's own results in tests/golden).
__device__ __forceinline__ double py_vector_norm2(double x0, double x1, double mx) {
    double outer = 1.0;
    if (isinf(mx)) return mx;
    if (mx == 0.0) return mx;
    int max_e;
    frexp(mx, &max_e);
    if (max_e < -1023) {
        // subnormal max: rescale once into the normal range
        outer = DBL_MIN;
        x0 /= DBL_MIN;
        x1 /= DBL_MIN;
        mx /= DBL_MIN;
        frexp(mx, &max_e);
    }
    const double scale = ldexp(1.0, -max_e);
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    const double v[2] = {x0, x1};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double x = v[i] * scale;
        const double hi = x * x, lo = fma(x, x, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    double h = sqrt(csum - 1.0 + (frac1 + frac2));
    {
        const double hi = -h * h, lo = fma(-h, h, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    const double x = csum - 1.0 + (frac1 + frac2);
    h += x / (2.0 * h);
    // h / scale: scale = 2**-max_e, so the quotient is h * 2**max_e rounded
    // once -- the same double as the product with the exact power of two
    // (a multiply instead of a division on the fold's serial chain); 2**1024
    // is not a double, that case keeps the division
    const double hs = max_e <= 1023 ? h * ldexp(1.0, max_e) : h / scale;
    return outer == 1.0 ? hs : outer * hs;
}

__device__ __noinline__ double py_hypot_slow(double a, double b) {
    if (isnan(a) || isnan(b)) return __longlong_as_double(0x7ff8000000000000LL);
    const double x0 = fabs(a), x1 = fabs(b);
    double mx = 0.0;
    if (x0 > mx) mx = x0;
    if (x1 > mx) mx = x1;
    return py_vector_norm2(x0, x1, mx);
}

// py_vector_norm2's arithmetic for the common case -- max(|a|, |b|) a normal
// double below 2**1022, no NaN -- with frexp / ldexp as exponent-field
// arithmetic (exact: the scale factors are powers of two), straight-line
// code on the fold's serial chain.  Zero, subnormal, huge, infinite and NaN
// operands take the general routine.
__device__ __forceinline__ double py_hypot(double a, double b) {
    const double x0 = fabs(a), x1 = fabs(b);
    const double mx = x0 > x1 ? x0 : x1;
    const int ex = (int)(__double_as_longlong(mx) >> 52);  // biased exponent (mx >= 0)
    if (isnan(a) || isnan(b) || ex < 1 || ex > 2044) return py_hypot_slow(a, b);
    // frexp: mx = f * 2**max_e, f in [0.5, 1), max_e = ex - 1022
    const double scale = __longlong_as_double((long long)(2045 - ex) << 52);   // 2**-max_e
    const double unscale = __longlong_as_double((long long)(ex + 1) << 52);    // 2**max_e
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    const double v[2] = {x0, x1};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double x = v[i] * scale;
        const double hi = x * x, lo = fma(x, x, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    double h = sqrt(csum - 1.0 + (frac1 + frac2));
    {
        const double hi = -h * h, lo = fma(-h, h, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    const double x = csum - 1.0 + (frac1 + frac2);
    h += x / (2.0 * h);
    return h * unscale;
}

// vm_ndt_hypot: py_hypot over pairs (parity probe against CPython's results)
__global__ void k_py_hypot(const double *ab, double *out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = py_hypot(ab[2 * i], ab[2 * i + 1]);
}

// ndt.cholupdate3 (ndt.py:37-52) on the lower triangle
// L = (l00, l10, l11, l20, l21, l22), x updated in place.
__device__ __forceinline__ void givens_k(double &lkk, double &xk, double *li1, double *xi1,
                                         double *li2, double *xi2) {
    const double r = py_hypot(lkk, xk);
    if (r == 0.0) return;
    const double c = lkk / r, s = xk / r;
    lkk = r;
    if (li1) {
        const double lik = *li1;
        *li1 = c * lik + s * *xi1;
        *xi1 = c * *xi1 - s * lik;
    }
    if (li2) {
        const double lik = *li2;
        *li2 = c * lik + s * *xi2;
        *xi2 = c * *xi2 - s * lik;
    }
}

// The square roots ndt.update_gaussian takes of the sample count n alone:
// sqrt(n), sqrt(n / (n + 1)), sqrt(n + 1).  The fold computes them one
// sample ahead, off the serial chain through S.
struct NdtRoots {
    double sq, f, sn;
};
__device__ __forceinline__ NdtRoots ndt_roots(unsigned long long n) {
    const double dn = (double)n, dnn = (double)(n + 1);
    return NdtRoots{sqrt(dn), sqrt(dn / dnn), sqrt(dnn)};
}

// ndt.update_gaussian (ndt.py:55-70): fold one sample into (n, mu, S);
// rt = ndt_roots(n).
__device__ __forceinline__ void ndt_update(unsigned long long &n, double mu[3], double S[6],
                                           const double x[3], const NdtRoots &rt) {
    if (n == 0) {
        n = 1;
#pragma unroll
        for (int a = 0; a < 3; ++a) mu[a] = x[a];
#pragma unroll
        for (int k = 0; k < 6; ++k) S[k] = 0.0;
        return;
    }
    const unsigned long long nn = n + 1;
    const double dnn = (double)nn;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = x[a] - mu[a];
#pragma unroll
    for (int a = 0; a < 3; ++a) mu[a] = mu[a] + d[a] / dnn;
    double L[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) L[k] = S[k] * rt.sq;
    double xx[3] = {d[0] * rt.f, d[1] * rt.f, d[2] * rt.f};
    givens_k(L[0], xx[0], &L[1], &xx[1], &L[3], &xx[2]);
    givens_k(L[2], xx[1], &L[4], &xx[2], nullptr, nullptr);
    givens_k(L[5], xx[2], nullptr, nullptr, nullptr, nullptr);
#pragma unroll
    for (int k = 0; k < 6; ++k) S[k] = L[k] / rt.sn;
    n = nn;
}

// ------------------------------------------------------------ buckets

struct NdtBuckets {
    unsigned *cnt;                   // [M] records per bucket (zero between batches)
    unsigned *cnt2;                  // [M] samples (phase-2 records) per bucket (zero between batches)
    unsigned *off;                   // [M] slice start (bumped by the scatter)
    unsigned *perm;                  // [M] buckets, most samples first
    unsigned *hist;                  // [NBK_BINS] size classes (zeroed by k_nbk_order)
    unsigned *cursor;                // [NBK_BINS] + [1] live buckets + [1] slice cursor
    unsigned long long *val;         // [R] (sk << 32 | value), bucketed
    unsigned long long *tmp;         // [R] rank-sort output
    double4 *pos;                    // [R] sample end point (x, y, z, intensity) of phase-2 slots
    int *mid, *big;                  // buckets for the warp / block sorts
    unsigned long long *nmid, *nbig;
    unsigned *bits;                  // huge buckets: per block 2 * bwords words
    unsigned long long bwords;       // words of one (phase, order) bitmap
    unsigned long long span;         // n * maxseg (orders per phase)
    const double4 *roots = nullptr;  // [nroots] (sqrt(n), sqrt(n / (n + 1)), sqrt(n + 1)), k_nbk_fold3
    unsigned nroots = 0;
};

// The square roots of the sample count each Welford / Givens step needs,
// tabulated once per map (the same IEEE operations as ndt_roots / the fold
// step), so the fold's steps load them instead of computing them.
constexpr unsigned NDT_ROOTS_N = 1u << 16;
__global__ void k_ndt_roots(double4 *out, unsigned n) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double dn = (double)i, dnn = (double)(i + 1);
    out[i] = make_double4(sqrt(dn), sqrt(dn / dnn), sqrt(dnn), 0.0);
}
__device__ __forceinline__ double4 ndt_roots_of(const NdtBuckets &b, unsigned long long n) {
    if (n < b.nroots) {
        const double2 *q = reinterpret_cast<const double2 *>(b.roots + n);
        const double2 lo = __ldg(q), hi = __ldg(q + 1);
        return make_double4(lo.x, lo.y, hi.x, hi.y);
    }
    const double dn = (double)n, dnn = (double)(n + 1);
    return make_double4(sqrt(dn), sqrt(dn / dnn), sqrt(dnn), 0.0);
}

constexpr int NBK_WARP_MAX = 512;  // warp rank sort (shared-memory staging: 4 KiB per warp)

// The batch's records and bucket count, on the device; false when there is
// nothing to do (guard refusal, or an overflow the host re-runs).
__device__ __forceinline__ bool bk_ndt_live(const DevMap &m, unsigned long long &R,
                                            unsigned long long &M) {
    if (!read_go(m)) return false;
    R = *((volatile unsigned long long *)(m.stats + S_RECORDS));
    M = *((volatile unsigned long long *)m.nmarked);
    if (R > m.rec_cap || M > m.marked_cap) {
        // a pipelined sequence stops here; the host re-emits this batch
        if (m.chain) atomicCAS(m.chain, 0, m.batch_idx + 1);
        return false;
    }
    return true;
}

// The deterministic walk files each miss through a Gaussian as a record with
// its chord (rec_t); the weight is computed here, one thread per record,
// exactly as _kernels.pyx:612-626 does it inline: the voxel's Gaussian at
// the start of the batch (resets are applied later, in the fold), the
// segment's origin and direction (engine.py:82-96), the chord (t0, t1).
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_ndt_weigh(const __grid_constant__ DevMap m, Src src) {
    unsigned long long R, M;
    if (!read_go(m)) return;
    R = *((volatile unsigned long long *)(m.stats + S_RECORDS));
    M = *((volatile unsigned long long *)m.nmarked);
    if (R > m.rec_cap || M > m.marked_cap) return;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = m.rec[i];
        if ((k >> 31) & 1ULL) continue;  // a sample (phase 2): no weight
        const unsigned mi = (unsigned)(k >> 32);
        if (mi >= M) continue;
        const int2 sl = m.marked[mi];
        if (sl.x < 0) continue;
        const int s = sl.x, li = sl.y;
        const unsigned oi = (unsigned)k & 0x7FFFFFFFu;
        Ray r;
        src.load((long long)(oi / (unsigned)m.maxseg), r.o, r.e, r.has, r.inten);
        prep_ray(m, r, true);
        double so[3], se[3];
        int sh;
        segment_of(m, r, (int)(oi % (unsigned)m.maxseg), so, se, sh);
        const double v[3] = {se[0] - so[0], se[1] - so[1], se[2] - so[2]};
        int g[3];
        slot_li_to_g(m, s, li, g);
        double off[3], mu[3];
        unpack_mean(layer_at<unsigned>(m, L_MEAN, s)[li], off);
        for (int a = 0; a < 3; ++a) mu[a] = ((double)g[a] + off[a]) * m.vox;
        float c6[6];
        const float *cov = layer_at<float>(m, L_COV, s) + li * 6;
        for (int j = 0; j < 6; ++j) c6[j] = cov[j];
        const double2 t = m.rec_t[i];
        const double gw = gaussian_weight(mu, c6, m.sigma2, so, v, t.x, t.y);
        const float d32 = (float)(gw * m.miss_delta);
        m.recval[i] = (__float_as_uint(d32) & 0x7FFFFFFFu) | (gw >= m.miss_check ? 0x80000000u : 0u);
    }
}

__global__ void __launch_bounds__(BLOCK) k_nbk_count(const __grid_constant__ DevMap m, NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = m.rec[i];
        const unsigned mi = (unsigned)(k >> 32);
        if (mi >= M) continue;
        atomicAdd(b.cnt + mi, 1u);
        if ((k >> 31) & 1ULL) atomicAdd(b.cnt2 + mi, 1u);
    }
}

// The fold's cost is its samples (a Givens update each; a phase-1 record is
// one clamped add), so the buckets are ordered by sample count: class
// 1 + min(samples, 254), class 0 for phase-1-only buckets.
__device__ __forceinline__ int nbk_class(unsigned samples) {
    return samples ? 1 + (int)min(samples, (unsigned)NBK_BINS - 2u) : 0;
}

// slice allocation (one atomic per warp), class histogram, sort lists
__global__ void __launch_bounds__(BLOCK) k_nbk_alloc(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned h[NBK_BINS];
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < M; base += stride) {
        const unsigned long long mi = base + threadIdx.x;
        const unsigned c = mi < M ? b.cnt[mi] : 0u;
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned wb = 0;
        if (lane == 31 && tot) wb = atomicAdd(b.cursor + NBK_BINS + 1, tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        if (c) {
            b.off[mi] = wb + incl - c;
            atomicAdd(h + nbk_class(b.cnt2[mi]), 1u);
            if (c > (unsigned)NBK_WARP_MAX) b.big[atomicAdd(b.nbig, 1ULL)] = (int)mi;
            else if (c > (unsigned)NBK_SERIAL) b.mid[atomicAdd(b.nmid, 1ULL)] = (int)mi;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x)
        if (h[i]) atomicAdd(b.hist + i, h[i]);
}

// classes -> cursors, most samples first; total live buckets
__global__ void k_nbk_order(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned h[NBK_BINS];
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x) {
        h[i] = b.hist[i];
        b.hist[i] = 0u;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned run = 0;
    for (int i = NBK_BINS - 1; i >= 0; --i) {
        b.cursor[i] = run;
        run += h[i];
    }
    b.cursor[NBK_BINS] = run;
}

__global__ void __launch_bounds__(BLOCK) k_nbk_perm(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned cnt[NBK_BINS], base[NBK_BINS];
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (unsigned long long b0 = (unsigned long long)blockIdx.x * blockDim.x; b0 < M;
         b0 += (unsigned long long)gridDim.x * blockDim.x) {
        for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x) cnt[i] = 0u;
        __syncthreads();
        const unsigned long long mi = b0 + threadIdx.x;
        const unsigned c = mi < M ? b.cnt[mi] : 0u;
        const int bin = c ? nbk_class(b.cnt2[mi]) : -1;
        unsigned r = 0;
        if (bin >= 0) r = atomicAdd(cnt + bin, 1u);
        __syncthreads();
        for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x)
            if (cnt[i]) base[i] = atomicAdd(b.cursor + i, cnt[i]);
        __syncthreads();
        if (bin >= 0) b.perm[base[bin] + r] = (unsigned)mi;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(BLOCK) k_nbk_scatter(const __grid_constant__ DevMap m, NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = m.rec[i];
        const unsigned mi = (unsigned)(k >> 32);
        if (mi >= M) continue;
        const unsigned pos = atomicAdd(b.off + mi, 1u);
        b.val[pos] = (k << 32) | (m.recval ? (unsigned long long)m.recval[i] : 0ULL);
    }
}

// slice [s, s + c) of bucket mi after the scatter bumped its offset
__device__ __forceinline__ unsigned nbk_start(const NdtBuckets &b, unsigned mi, unsigned &c) {
    c = b.cnt[mi];
    return b.off[mi] - c;
}

// Buckets of NBK_SERIAL < c <= NBK_WARP_MAX records, one warp each: staged
// in shared memory, every lane ranks its records against the whole bucket
// (sort keys are unique) and writes them back at their ranks.
constexpr int NBK_MID_WARPS = BLOCK / 32;
__global__ void __launch_bounds__(BLOCK) k_nbk_sort_mid(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned long long sv[NBK_MID_WARPS][NBK_WARP_MAX];
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    unsigned long long *my = sv[wi];
    const unsigned long long nm = *((volatile unsigned long long *)b.nmid);
    for (unsigned long long w = (unsigned long long)blockIdx.x * NBK_MID_WARPS + wi; w < nm;
         w += (unsigned long long)gridDim.x * NBK_MID_WARPS) {
        const unsigned mi = (unsigned)b.mid[w];
        unsigned c;
        const unsigned s = nbk_start(b, mi, c);
        for (unsigned i = lane; i < c; i += 32) my[i] = b.val[s + i];
        __syncwarp();
        for (unsigned i = lane; i < c; i += 32) {
            const unsigned long long x = my[i];
            unsigned rank = 0;
            for (unsigned j = 0; j < c; ++j) rank += my[j] < x ? 1u : 0u;
            b.val[s + rank] = x;
        }
        __syncwarp();
    }
}

// Buckets above NBK_WARP_MAX, one block each: bitonic sort in shared memory,
// or, above NBK_SMEM, a rank sort over the (phase, order) bitmap.
__global__ void __launch_bounds__(BLOCK) k_nbk_sort_big(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned long long sv[NBK_SMEM];
    __shared__ unsigned wsum[BLOCK];
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const unsigned long long nb = *((volatile unsigned long long *)b.nbig);
    unsigned *pres = b.bits + (size_t)blockIdx.x * 2 * b.bwords;
    unsigned *pref = pres + b.bwords;
    for (unsigned long long w = blockIdx.x; w < nb; w += gridDim.x) {
        const unsigned mi = (unsigned)b.big[w];
        unsigned c;
        const unsigned s = nbk_start(b, mi, c);
        if (c <= (unsigned)NBK_SMEM) {
            unsigned P = 32;
            while (P < c) P <<= 1;
            for (unsigned i = threadIdx.x; i < P; i += blockDim.x) sv[i] = i < c ? b.val[s + i] : ~0ULL;
            __syncthreads();
            for (unsigned k = 2; k <= P; k <<= 1) {
                for (unsigned j = k >> 1; j > 0; j >>= 1) {
                    for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
                        const unsigned p = i ^ j;
                        if (p > i) {
                            const unsigned long long x = sv[i], y = sv[p];
                            if ((x > y) == ((i & k) == 0)) {
                                sv[i] = y;
                                sv[p] = x;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (unsigned i = threadIdx.x; i < c; i += blockDim.x) b.val[s + i] = sv[i];
            __syncthreads();
            continue;
        }
        // rank sort: sort keys are unique, so a key's rank is the number of
        // set bits below its own in the (phase, order) presence bitmap
        for (unsigned long long i = threadIdx.x; i < b.bwords; i += blockDim.x) pres[i] = 0u;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < c; i += blockDim.x) {
            const unsigned sk = (unsigned)(b.val[s + i] >> 32);
            const unsigned long long bit = (unsigned long long)(sk >> 31) * b.span + (sk & 0x7FFFFFFFu);
            atomicOr(pres + (bit >> 5), 1u << (bit & 31));
        }
        __syncthreads();
        // block exclusive scan of the words' popcounts (contiguous chunk per thread)
        const unsigned long long per = (b.bwords + blockDim.x - 1) / blockDim.x;
        const unsigned long long w0 = per * threadIdx.x, w1 = min(b.bwords, w0 + per);
        unsigned loc = 0;
        for (unsigned long long i = w0; i < w1; ++i) loc += __popc(pres[i]);
        wsum[threadIdx.x] = loc;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned run = 0;
            for (int t = 0; t < (int)blockDim.x; ++t) {
                const unsigned v = wsum[t];
                wsum[t] = run;
                run += v;
            }
        }
        __syncthreads();
        unsigned run = wsum[threadIdx.x];
        for (unsigned long long i = w0; i < w1; ++i) {
            pref[i] = run;
            run += __popc(pres[i]);
        }
        __syncthreads();
        for (unsigned i = threadIdx.x; i < c; i += blockDim.x) {
            const unsigned long long v = b.val[s + i];
            const unsigned sk = (unsigned)(v >> 32);
            const unsigned long long bit = (unsigned long long)(sk >> 31) * b.span + (sk & 0x7FFFFFFFu);
            const unsigned rank = pref[bit >> 5] + __popc(pres[bit >> 5] & ((1u << (bit & 31)) - 1u));
            b.tmp[s + rank] = v;
        }
        __syncthreads();
        for (unsigned i = threadIdx.x; i < c; i += blockDim.x) b.val[s + i] = b.tmp[s + i];
        __syncthreads();
    }
}

// Buckets of <= NBK_SERIAL (16) records: one thread each, a bitonic sorting
// network on registers (static indices: no local memory), written back.
__device__ __forceinline__ void cswap(unsigned long long &a, unsigned long long &b, bool up) {
    const unsigned long long x = a, y = b;
    const bool sw = (x > y) == up;
    a = sw ? y : x;
    b = sw ? x : y;
}

__global__ void __launch_bounds__(BLOCK) k_nbk_sort_small(const __grid_constant__ DevMap m, NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const unsigned K = *((volatile unsigned *)(b.cursor + NBK_BINS));
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < K; t += gridDim.x * blockDim.x) {
        unsigned c;
        const unsigned s = nbk_start(b, b.perm[t], c);
        if (c < 2 || c > (unsigned)NBK_SERIAL) continue;
        unsigned long long r[NBK_SERIAL];
#pragma unroll
        for (int i = 0; i < NBK_SERIAL; ++i) r[i] = (unsigned)i < c ? b.val[s + i] : ~0ULL;
#pragma unroll
        for (int k = 2; k <= NBK_SERIAL; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
                for (int i = 0; i < NBK_SERIAL; ++i)
                    if ((i ^ j) > i) cswap(r[i], r[i ^ j], (i & k) == 0);
#pragma unroll
        for (int i = 0; i < NBK_SERIAL; ++i)
            if ((unsigned)i < c) b.val[s + i] = r[i];
    }
}

// Every sample slot gets its end point and intensity next to it, so the
// serial fold streams them instead of chasing record -> ray -> end point.
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_nbk_gather(const __grid_constant__ DevMap m, Src src, NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < R;
         p += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long v = b.val[p];
        if (!(v >> 63)) continue;
        const unsigned oi = (unsigned)(v >> 32) & 0x7FFFFFFFu;
        double e[3];
        float it;
        src.load_end((long long)(oi / (unsigned)m.maxseg), e, it);
        b.pos[p] = make_double4(e[0], e[1], e[2], (double)it);
    }
}

// ---- the same bucket preparation in four launches (NDT-OM / NDT-TM) ----
// The ten kernels above (weigh, count, alloc, order, perm, scatter, three
// sorts, gather) are each a few microseconds of work behind a launch and a
// tail; on the NDT batch tail they sit on the critical path next to
// k_resolve.  Fused by dependency: weigh + count (both per record), alloc +
// order (the last block to finish turns the class histogram into cursors),
// perm + scatter (both need only the slices and cursors), the three sorts +
// gather (block roles by bucket size; each bucket gathers its sample end
// points once sorted).  Same results: a bucket's order comes from its sort,
// not from the scatter.

template <class Src>
__global__ void __launch_bounds__(BLOCK) k_nbk_weigh_count(const __grid_constant__ DevMap m, Src src,
                                                           NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = m.rec[i];
        const unsigned mi = (unsigned)(k >> 32);
        if (mi >= M) continue;
        atomicAdd(b.cnt + mi, 1u);
        if ((k >> 31) & 1ULL) {
            atomicAdd(b.cnt2 + mi, 1u);
            continue;  // a sample (phase 2): no weight
        }
        const int2 sl = m.marked[mi];
        if (sl.x < 0) continue;
        const int s = sl.x, li = sl.y;
        const unsigned oi = (unsigned)k & 0x7FFFFFFFu;
        Ray r;
        src.load((long long)(oi / (unsigned)m.maxseg), r.o, r.e, r.has, r.inten);
        prep_ray(m, r, true);
        double so[3], se[3];
        int sh;
        segment_of(m, r, (int)(oi % (unsigned)m.maxseg), so, se, sh);
        const double v[3] = {se[0] - so[0], se[1] - so[1], se[2] - so[2]};
        int g[3];
        slot_li_to_g(m, s, li, g);
        double off[3], mu[3];
        unpack_mean(layer_at<unsigned>(m, L_MEAN, s)[li], off);
        for (int a = 0; a < 3; ++a) mu[a] = ((double)g[a] + off[a]) * m.vox;
        float c6[6];
        const float *cov = layer_at<float>(m, L_COV, s) + li * 6;
        for (int j = 0; j < 6; ++j) c6[j] = cov[j];
        const double2 t = m.rec_t[i];
        const double gw = gaussian_weight(mu, c6, m.sigma2, so, v, t.x, t.y);
        const float d32 = (float)(gw * m.miss_delta);
        m.recval[i] = (__float_as_uint(d32) & 0x7FFFFFFFu) | (gw >= m.miss_check ? 0x80000000u : 0u);
    }
}

// k_nbk_alloc, then the last block to finish runs k_nbk_order
// (cursor[NBK_BINS + 2] counts finished blocks; the last one resets it).
__global__ void __launch_bounds__(BLOCK) k_nbk_alloc_order(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned h[NBK_BINS];
    __shared__ bool last;
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < M; base += stride) {
        const unsigned long long mi = base + threadIdx.x;
        const unsigned c = mi < M ? b.cnt[mi] : 0u;
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned wb = 0;
        if (lane == 31 && tot) wb = atomicAdd(b.cursor + NBK_BINS + 1, tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        if (c) {
            b.off[mi] = wb + incl - c;
            atomicAdd(h + nbk_class(b.cnt2[mi]), 1u);
            if (c > (unsigned)NBK_WARP_MAX) b.big[atomicAdd(b.nbig, 1ULL)] = (int)mi;
            else if (c > (unsigned)NBK_SERIAL) b.mid[atomicAdd(b.nmid, 1ULL)] = (int)mi;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x)
        if (h[i]) atomicAdd(b.hist + i, h[i]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(b.cursor + NBK_BINS + 2, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x) h[i] = atomicExch(b.hist + i, 0u);
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned run = 0;
    for (int i = NBK_BINS - 1; i >= 0; --i) {
        b.cursor[i] = run;
        run += h[i];
    }
    b.cursor[NBK_BINS] = run;
    b.cursor[NBK_BINS + 2] = 0u;
}

// k_nbk_perm's loop, then k_nbk_scatter's
__global__ void __launch_bounds__(BLOCK) k_nbk_perm_scatter(const __grid_constant__ DevMap m, NdtBuckets b) {
    __shared__ unsigned cnt[NBK_BINS], base[NBK_BINS];
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    for (unsigned long long b0 = (unsigned long long)blockIdx.x * blockDim.x; b0 < M;
         b0 += (unsigned long long)gridDim.x * blockDim.x) {
        for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x) cnt[i] = 0u;
        __syncthreads();
        const unsigned long long mi = b0 + threadIdx.x;
        const unsigned c = mi < M ? b.cnt[mi] : 0u;
        const int bin = c ? nbk_class(b.cnt2[mi]) : -1;
        unsigned r = 0;
        if (bin >= 0) r = atomicAdd(cnt + bin, 1u);
        __syncthreads();
        for (int i = threadIdx.x; i < NBK_BINS; i += blockDim.x)
            if (cnt[i]) base[i] = atomicAdd(b.cursor + i, cnt[i]);
        __syncthreads();
        if (bin >= 0) b.perm[base[bin] + r] = (unsigned)mi;
        __syncthreads();
    }
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = m.rec[i];
        const unsigned mi = (unsigned)(k >> 32);
        if (mi >= M) continue;
        const unsigned pos = atomicAdd(b.off + mi, 1u);
        b.val[pos] = (k << 32) | (m.recval ? (unsigned long long)m.recval[i] : 0ULL);
    }
}

// a sorted slot: its value, and for a sample its end point next to it
template <class Src>
__device__ __forceinline__ void nbk_put(const DevMap &m, const Src &src, const NdtBuckets &b,
                                        unsigned p, unsigned long long v) {
    b.val[p] = v;
    if (!(v >> 63)) return;
    const unsigned oi = (unsigned)(v >> 32) & 0x7FFFFFFFu;
    double e[3];
    float it;
    src.load_end((long long)(oi / (unsigned)m.maxseg), e, it);
    b.pos[p] = make_double4(e[0], e[1], e[2], (double)it);
}

// Block roles: [0, nbig_blocks) the block sorts of k_nbk_sort_big, then
// nmid_blocks of k_nbk_sort_mid's warp sorts, the rest k_nbk_sort_small's
// thread sorts (and single-record buckets); every sorted slot is written
// with nbk_put (k_nbk_gather's end points).
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_nbk_sort_gather(const __grid_constant__ DevMap m, Src src,
                                                           NdtBuckets b, int nbig_blocks,
                                                           int nmid_blocks) {
    __shared__ union {
        unsigned long long mid[NBK_MID_WARPS][NBK_WARP_MAX];
        struct {
            unsigned long long sv[NBK_SMEM];
            unsigned wsum[BLOCK];
        } big;
    } sh;
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const int bid = (int)blockIdx.x;
    if (bid < nbig_blocks) {
        unsigned long long *sv = sh.big.sv;
        unsigned *wsum = sh.big.wsum;
        const unsigned long long nb = *((volatile unsigned long long *)b.nbig);
        unsigned *pres = b.bits + (size_t)bid * 2 * b.bwords;
        unsigned *pref = pres + b.bwords;
        for (unsigned long long w = bid; w < nb; w += nbig_blocks) {
            const unsigned mi = (unsigned)b.big[w];
            unsigned c;
            const unsigned s = nbk_start(b, mi, c);
            if (c <= (unsigned)NBK_SMEM) {
                unsigned P = 32;
                while (P < c) P <<= 1;
                for (unsigned i = threadIdx.x; i < P; i += blockDim.x) sv[i] = i < c ? b.val[s + i] : ~0ULL;
                __syncthreads();
                for (unsigned k = 2; k <= P; k <<= 1) {
                    for (unsigned j = k >> 1; j > 0; j >>= 1) {
                        for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
                            const unsigned p = i ^ j;
                            if (p > i) {
                                const unsigned long long x = sv[i], y = sv[p];
                                if ((x > y) == ((i & k) == 0)) {
                                    sv[i] = y;
                                    sv[p] = x;
                                }
                            }
                        }
                        __syncthreads();
                    }
                }
                for (unsigned i = threadIdx.x; i < c; i += blockDim.x) nbk_put(m, src, b, s + i, sv[i]);
                __syncthreads();
                continue;
            }
            for (unsigned long long i = threadIdx.x; i < b.bwords; i += blockDim.x) pres[i] = 0u;
            __syncthreads();
            for (unsigned i = threadIdx.x; i < c; i += blockDim.x) {
                const unsigned sk = (unsigned)(b.val[s + i] >> 32);
                const unsigned long long bit = (unsigned long long)(sk >> 31) * b.span + (sk & 0x7FFFFFFFu);
                atomicOr(pres + (bit >> 5), 1u << (bit & 31));
            }
            __syncthreads();
            const unsigned long long per = (b.bwords + blockDim.x - 1) / blockDim.x;
            const unsigned long long w0 = per * threadIdx.x, w1 = min(b.bwords, w0 + per);
            unsigned loc = 0;
            for (unsigned long long i = w0; i < w1; ++i) loc += __popc(pres[i]);
            wsum[threadIdx.x] = loc;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned run = 0;
                for (int t = 0; t < (int)blockDim.x; ++t) {
                    const unsigned v = wsum[t];
                    wsum[t] = run;
                    run += v;
                }
            }
            __syncthreads();
            unsigned run = wsum[threadIdx.x];
            for (unsigned long long i = w0; i < w1; ++i) {
                pref[i] = run;
                run += __popc(pres[i]);
            }
            __syncthreads();
            for (unsigned i = threadIdx.x; i < c; i += blockDim.x) {
                const unsigned long long v = b.val[s + i];
                const unsigned sk = (unsigned)(v >> 32);
                const unsigned long long bit = (unsigned long long)(sk >> 31) * b.span + (sk & 0x7FFFFFFFu);
                const unsigned rank = pref[bit >> 5] + __popc(pres[bit >> 5] & ((1u << (bit & 31)) - 1u));
                b.tmp[s + rank] = v;
            }
            __syncthreads();
            for (unsigned i = threadIdx.x; i < c; i += blockDim.x) nbk_put(m, src, b, s + i, b.tmp[s + i]);
            __syncthreads();
        }
        return;
    }
    if (bid < nbig_blocks + nmid_blocks) {
        const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
        unsigned long long *my = sh.mid[wi];
        const unsigned long long nm = *((volatile unsigned long long *)b.nmid);
        for (unsigned long long w = (unsigned long long)(bid - nbig_blocks) * NBK_MID_WARPS + wi; w < nm;
             w += (unsigned long long)nmid_blocks * NBK_MID_WARPS) {
            const unsigned mi = (unsigned)b.mid[w];
            unsigned c;
            const unsigned s = nbk_start(b, mi, c);
            for (unsigned i = lane; i < c; i += 32) my[i] = b.val[s + i];
            __syncwarp();
            for (unsigned i = lane; i < c; i += 32) {
                const unsigned long long x = my[i];
                unsigned rank = 0;
                for (unsigned j = 0; j < c; ++j) rank += my[j] < x ? 1u : 0u;
                nbk_put(m, src, b, s + rank, x);
            }
            __syncwarp();
        }
        return;
    }
    const unsigned K = *((volatile unsigned *)(b.cursor + NBK_BINS));
    const unsigned nsmall = (gridDim.x - (unsigned)(nbig_blocks + nmid_blocks)) * blockDim.x;
    for (unsigned t = (unsigned)(bid - nbig_blocks - nmid_blocks) * blockDim.x + threadIdx.x; t < K;
         t += nsmall) {
        unsigned c;
        const unsigned s = nbk_start(b, b.perm[t], c);
        if (c > (unsigned)NBK_SERIAL) continue;
        if (c == 1) {
            nbk_put(m, src, b, s, b.val[s]);
            continue;
        }
        unsigned long long r[NBK_SERIAL];
#pragma unroll
        for (int i = 0; i < NBK_SERIAL; ++i) r[i] = (unsigned)i < c ? b.val[s + i] : ~0ULL;
#pragma unroll
        for (int k = 2; k <= NBK_SERIAL; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
                for (int i = 0; i < NBK_SERIAL; ++i)
                    if ((i ^ j) > i) cswap(r[i], r[i ^ j], (i & k) == 0);
#pragma unroll
        for (int i = 0; i < NBK_SERIAL; ++i)
            if ((unsigned)i < c) nbk_put(m, src, b, s + i, r[i]);
    }
}

#ifndef NBK_FOLD_MINB
#define NBK_FOLD_MINB 2
#endif
__device__ __forceinline__ double4 ld_d4(const double4 *p) {  // read-only path, 2 x 16 B
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = __ldg(q), c = __ldg(q + 1);
    return make_double4(a.x, a.y, c.x, c.y);
}
constexpr int NBK_PF = 8;        // phase-1 records per group (the next group is in flight)
constexpr int NBK_PF_L1 = 64;    // and the records this far ahead prefetched into L1

// One lane per bucket, buckets with the most samples first, so the 32 lanes
// of a warp hold buckets with (nearly) the same number of samples; the
// record loops are warp-uniform (bounded by the warp's maximum, inactive
// lanes masked), so the lanes step through their samples together, and the
// (sorted, read-only) records and sample end points are loaded ahead of the
// serial chain.  Clears the index stamp and the bucket counts.
#ifdef VM_FOLD_PROF
// dev builds: the slowest warp task of the last fold (cycles << 24 | max
// phase-1 records << 12 | max samples) and the sum of all tasks' cycles
__device__ unsigned long long g_fold_prof[2];
#endif

template <bool TM>
__global__ void __launch_bounds__(BLOCK, NBK_FOLD_MINB) k_nbk_fold(const __grid_constant__ DevMap m,
                                                                   NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const unsigned K = *((volatile unsigned *)(b.cursor + NBK_BINS));
    const int lane = threadIdx.x & 31;
    const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
    for (unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 32 < K; w += nwarps) {
#ifdef VM_FOLD_PROF
        const long long prof_t0 = clock64();
#endif
        const unsigned t = w * 32 + lane;
        bool act = t < K;
        unsigned c = 0, ns = 0, s = 0, mi = 0;
        int slot = 0, li = 0;
        if (act) {
            mi = b.perm[t];
            s = nbk_start(b, mi, c);
            ns = b.cnt2[mi];
            b.cnt[mi] = 0u;
            b.cnt2[mi] = 0u;
            const int2 sl = m.marked[mi];
            slot = sl.x;
            li = sl.y;
            act = slot >= 0;
        }
        if (!act) c = ns = 0;
        const unsigned long long *__restrict__ v = b.val + s;
        const unsigned np1 = c - ns;  // phase-1 records sort first
        float *occ = nullptr, *cov = nullptr, *ib = nullptr;
        unsigned *mb = nullptr, *cb = nullptr, *hb = nullptr, *missb = nullptr;
        int g[3] = {0, 0, 0};
        float l = 0.0f;
        unsigned n0 = 0;
        if (act) {
            slot_li_to_g(m, slot, li, g);
            occ = layer_at<float>(m, L_OCC, slot);
            mb = layer_at<unsigned>(m, L_MEAN, slot);
            cb = layer_at<unsigned>(m, L_COUNT, slot);
            cov = layer_at<float>(m, L_COV, slot);
            if (TM) {
                ib = layer_at<float>(m, L_INTENS, slot);
                hb = layer_at<unsigned>(m, L_HIT, slot);
                missb = layer_at<unsigned>(m, L_MISS, slot);
            }
            l = occ[li];
            n0 = cb[li];
        }
        // ---- phase 1: misses through the voxel's Gaussian, in ray order ----
        bool reset = false;
        unsigned miss_add = 0;
        // The chain through l costs a few cycles per record, so the loads run
        // ahead of it: the next group in registers, records NBK_PF_L1 ahead
        // pulled into L1 (a voxel a whole scan's rays graze has thousands).
        const unsigned mp1 = __reduce_max_sync(0xffffffffu, np1);
        unsigned wv[NBK_PF];
#pragma unroll
        for (int q = 0; q < NBK_PF; ++q) wv[q] = (unsigned)q < np1 ? (unsigned)__ldg(v + q) : 0u;
        for (unsigned i0 = 0; i0 < mp1; i0 += NBK_PF) {
            if (i0 + NBK_PF_L1 < np1)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(v + i0 + NBK_PF_L1));
            unsigned nx[NBK_PF];
#pragma unroll
            for (int q = 0; q < NBK_PF; ++q)
                nx[q] = i0 + NBK_PF + q < np1 ? (unsigned)__ldg(v + i0 + NBK_PF + q) : 0u;
#pragma unroll
            for (int q = 0; q < NBK_PF; ++q) {
                if (i0 + q < np1) {
                    const float d = reset ? m.miss32 : -__uint_as_float(wv[q] & 0x7FFFFFFFu);
                    l = clamp_add(l, d, m.cmin, m.cmax);
                    if (TM && (reset || (wv[q] >> 31))) ++miss_add;
                    // transient reset (reference.py:86-93, _reset_voxel_buffers 97-104)
                    if (!reset && l < m.fthresh && n0 > 0) {
                        reset = true;
                        miss_add = 0;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < NBK_PF; ++q) wv[q] = nx[q];
        }
        if (reset) {
            n0 = 0;
            cb[li] = 0;
            mb[li] = 0;
#pragma unroll
            for (int k = 0; k < 6; ++k) cov[li * 6 + k] = 0.0f;
            if (TM) {
                hb[li] = 0;
                missb[li] = 0;
                ib[li * 2] = 0.0f;
                ib[li * 2 + 1] = 0.0f;
            }
        }
        if (TM && miss_add) missb[li] += miss_add;
        // ---- phase 2: the voxel's samples in ray order (reference.py:107-150) ----
        unsigned long long n = n0;
        double mu[3] = {0.0, 0.0, 0.0}, S[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double imean = 0.0, im2 = 0.0;
        if (ns) {
            if (n > 0) {
                double off[3];
                unpack_mean(mb[li], off);
#pragma unroll
                for (int a = 0; a < 3; ++a) mu[a] = ((double)g[a] + off[a]) * m.vox;
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) S[k] = (double)cov[li * 6 + k];
            if (TM) {
                imean = ib[li * 2];
                im2 = ib[li * 2 + 1];
            }
        }
        const double4 *__restrict__ ps = b.pos + s + np1;
        const unsigned ms = __reduce_max_sync(0xffffffffu, ns);
        double4 cur = ns ? ld_d4(ps) : make_double4(0.0, 0.0, 0.0, 0.0);
        NdtRoots rt = ndt_roots(n);
        for (unsigned i = 0; i < ms; ++i) {
            if (i < ns) {
                const double4 nxt = i + 1 < ns ? ld_d4(ps + i + 1) : cur;
                const NdtRoots rt_next = ndt_roots(n + 1);  // n grows by one per sample
                l = clamp_add(l, m.hit32, m.cmin, m.cmax);
                if (TM) {
                    // ndt.update_intensity (ndt.py:98-106), stored f32 per sample
                    const double val = cur.w, nn = (double)(n + 1);
                    const double d = val - imean;
                    const double mnew = imean + d / nn;
                    const double m2new = im2 + d * (val - mnew);
                    imean = (double)(float)mnew;
                    im2 = (double)(float)m2new;
                }
                const double e[3] = {cur.x, cur.y, cur.z};
                ndt_update(n, mu, S, e, rt);
                cur = nxt;
                rt = rt_next;
            }
        }
        if (ns) {
            if (TM) {
                ib[li * 2] = (float)imean;
                ib[li * 2 + 1] = (float)im2;
                hb[li] += ns;
            }
            cb[li] = n > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)n;
            if (n >= 3 && m.gmask)  // the walk loads this brick's counts from now on
                atomicOr(m.gmask + slot, m.brick_shift >= 0 ? 1u << brick_of(li, m.bsh) : 0xFFFFFFFFu);
            double frac[3];
            const double hi = 1.0 - 1.0 / 2048.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                double f = mu[a] / m.vox - (double)g[a];
                if (f < 0.0) f = 0.0;
                if (f > hi) f = hi;
                frac[a] = f;
            }
            mb[li] = pack_mean(frac);
#pragma unroll
            for (int k = 0; k < 6; ++k) cov[li * 6 + k] = (float)S[k];
        }
        if (act) {
            occ[li] = l;
            layer_at<unsigned>(m, m.nidx, slot)[li] = 0u;
        }
#ifdef VM_FOLD_PROF
        if (lane == 0) {
            const unsigned long long dt = (unsigned long long)(clock64() - prof_t0);
            atomicMax(&g_fold_prof[0], (dt << 24) | ((unsigned long long)min(mp1, 4095u) << 12) |
                                           min(ms, 4095u));
            atomicAdd(&g_fold_prof[1], dt);
        }
#endif
    }
}

// py_hypot's common case with the verified operators
__device__ __forceinline__ double xhypot(double a, double b, bool &ok) {
    const double x0 = fabs(a), x1 = fabs(b);
    const double mx = x0 > x1 ? x0 : x1;
    if (isnan(x0) || isnan(x1) || !(mx > 0.0) || !xmid(mx)) {
        ok = ok && mx == 0.0 && !isnan(x0) && !isnan(x1);
        return 0.0;
    }
    const int ex = xexp(mx);
    const double scale = xpow2(2045 - ex), unscale = xpow2(ex + 1);
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    const double v[2] = {x0, x1};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double x = v[i] * scale;
        const double hi = x * x, lo = fma(x, x, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    double h = xsqrt(csum - 1.0 + (frac1 + frac2), ok);
    {
        const double hi = -h * h, lo = fma(-h, h, -hi);
        const double s = csum + hi;
        const double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    const double x = csum - 1.0 + (frac1 + frac2);
    h += xdiv(x, 2.0 * h, ok);
    return h * unscale;
}
template <bool FAST>
__device__ __forceinline__ double vhypot(double a, double b, bool &ok) {
    if (FAST) return xhypot(a, b, ok);
    return py_hypot(a, b);
}

// ---- the same fold with the Givens rotations pipelined over three lanes ----
// ndt_update's serial chain is three rotations per sample (cholupdate3), but
// rotation k only reads column k of the factor and the rotated vector left by
// rotation k - 1 of the SAME sample.  So three lanes hold one bucket: lane
// k of the triple owns column k (diagonal Ld, entries below it La, Lb) and
// applies rotation k to sample t - k in step t, taking the vector from lane
// k - 1 (one shuffle per step).  Every lane's loop-carried chain is then one
// rotation (scale, hypot, divisions, rescale) instead of three: the same
// operations in the same order per value, so the factor is bit-identical to
// ndt_update's.  Lane 0 of a triple also carries the mean (Welford), the
// occupancy hit and the TM intensity, like the one-lane fold.  Ten buckets
// per warp (lanes 30, 31 idle); phase 1 runs on all three lanes alike.
constexpr int NBK3_PER_WARP = 10;

// rotation of column (Ld; La, Lb) by the vector (xd; xa, xb) after the
// count's scale sq, then the rescale by sn (ndt_update / givens_k, one column)
template <bool FAST>
__device__ __forceinline__ void ndt_rot_column(double &Ld, double &La, double &Lb, double xd,
                                               double &xa, double &xb, double sq, double sn,
                                               bool &ok) {
    Ld = Ld * sq;
    La = La * sq;
    Lb = Lb * sq;
    const double r = vhypot<FAST>(Ld, xd, ok);
    if (r != 0.0) {
        const double c = vdiv<FAST>(Ld, r, ok), s = vdiv<FAST>(xd, r, ok);
        Ld = r;
        const double la = La, lb = Lb;
        La = c * la + s * xa;
        xa = c * xa - s * la;
        Lb = c * lb + s * xb;
        xb = c * xb - s * lb;
    }
    Ld = vdiv<FAST>(Ld, sn, ok);
    La = vdiv<FAST>(La, sn, ok);
    Lb = vdiv<FAST>(Lb, sn, ok);
}

// One step of lane k (sample nj = n0 + j): lane 0 folds the sample into the
// Welford mean and forms the vector, every lane rotates its column.
template <bool FAST>
__device__ __forceinline__ void ndt_fold3_step(int k, unsigned long long nj, const double e[3],
                                               const double4 &rt, double mu[3], double ind,
                                               double ina, double &Ld, double &La, double &Lb,
                                               double &oa, double &ob, bool &ok) {
    double xd, xa, xb;
    if (k == 0) {
        if (nj == 0) {
#pragma unroll
            for (int a = 0; a < 3; ++a) mu[a] = e[a];
            xd = xa = xb = 0.0;
        } else {
            const double dnn = (double)(nj + 1);
            double d[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) d[a] = e[a] - mu[a];
#pragma unroll
            for (int a = 0; a < 3; ++a) mu[a] = mu[a] + vdiv<FAST>(d[a], dnn, ok);
            const double f = rt.y;  // sqrt(nj / (nj + 1))
            xd = d[0] * f;
            xa = d[1] * f;
            xb = d[2] * f;
        }
    } else {
        xd = ind;
        xa = ina;
        xb = 0.0;
    }
    if (nj == 0) {
        // ndt_update's first sample: the factor is zero
        Ld = La = Lb = 0.0;
    } else {
        ndt_rot_column<FAST>(Ld, La, Lb, xd, xa, xb, rt.x, rt.z, ok);
    }
    oa = xa;
    ob = xb;
}

#ifndef NBK3_FAST
#define NBK3_FAST 0  // 1: verified fast operators in k_nbk_fold3 (measured slower, DESIGN)
#endif

template <bool TM>
__global__ void __launch_bounds__(BLOCK, NBK_FOLD_MINB) k_nbk_fold3(const __grid_constant__ DevMap m,
                                                                    NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const unsigned K = *((volatile unsigned *)(b.cursor + NBK_BINS));
    const int lane = threadIdx.x & 31;
    const int k = lane % 3;                   // the column this lane rotates
    const int tri = lane / 3;                 // the bucket of the warp (10 = idle)
    const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
    for (unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * NBK3_PER_WARP < K;
         w += nwarps) {
#ifdef VM_FOLD_PROF
        const long long prof_t0 = clock64();
#endif
        const unsigned t = w * NBK3_PER_WARP + tri;
        bool act = tri < NBK3_PER_WARP && t < K;
        unsigned c = 0, ns = 0, s = 0, mi = 0;
        int slot = 0, li = 0;
        if (act) {
            mi = b.perm[t];
            s = nbk_start(b, mi, c);
            ns = b.cnt2[mi];
            const int2 sl = m.marked[mi];
            slot = sl.x;
            li = sl.y;
            act = slot >= 0;
        }
        __syncwarp();
        if (k == 0 && tri < NBK3_PER_WARP && t < K) {
            b.cnt[mi] = 0u;
            b.cnt2[mi] = 0u;
        }
        if (!act) c = ns = 0;
        const unsigned long long *__restrict__ v = b.val + s;
        const unsigned np1 = c - ns;  // phase-1 records sort first
        float *occ = nullptr, *cov = nullptr, *ib = nullptr;
        unsigned *mb = nullptr, *cb = nullptr, *hb = nullptr, *missb = nullptr;
        int g[3] = {0, 0, 0};
        float l = 0.0f;
        unsigned n0 = 0;
        if (act) {
            slot_li_to_g(m, slot, li, g);
            occ = layer_at<float>(m, L_OCC, slot);
            mb = layer_at<unsigned>(m, L_MEAN, slot);
            cb = layer_at<unsigned>(m, L_COUNT, slot);
            cov = layer_at<float>(m, L_COV, slot);
            if (TM) {
                ib = layer_at<float>(m, L_INTENS, slot);
                hb = layer_at<unsigned>(m, L_HIT, slot);
                missb = layer_at<unsigned>(m, L_MISS, slot);
            }
            l = occ[li];
            n0 = cb[li];
        }
        const bool writer = act && k == 0;
        // ---- phase 1 (k_nbk_fold's loop; the three lanes of a bucket alike) ----
        bool reset = false;
        unsigned miss_add = 0;
        const unsigned mp1 = __reduce_max_sync(0xffffffffu, np1);
        unsigned wv[NBK_PF];
#pragma unroll
        for (int q = 0; q < NBK_PF; ++q) wv[q] = (unsigned)q < np1 ? (unsigned)__ldg(v + q) : 0u;
        for (unsigned i0 = 0; i0 < mp1; i0 += NBK_PF) {
            if (i0 + NBK_PF_L1 < np1 && k == 0)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(v + i0 + NBK_PF_L1));
            unsigned nx[NBK_PF];
#pragma unroll
            for (int q = 0; q < NBK_PF; ++q)
                nx[q] = i0 + NBK_PF + q < np1 ? (unsigned)__ldg(v + i0 + NBK_PF + q) : 0u;
#pragma unroll
            for (int q = 0; q < NBK_PF; ++q) {
                if (i0 + q < np1) {
                    const float d = reset ? m.miss32 : -__uint_as_float(wv[q] & 0x7FFFFFFFu);
                    l = clamp_add(l, d, m.cmin, m.cmax);
                    if (TM && (reset || (wv[q] >> 31))) ++miss_add;
                    if (!reset && l < m.fthresh && n0 > 0) {
                        reset = true;
                        miss_add = 0;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < NBK_PF; ++q) wv[q] = nx[q];
        }
        if (reset) {
            n0 = 0;
            if (writer) {
                cb[li] = 0;
                mb[li] = 0;
#pragma unroll
                for (int q = 0; q < 6; ++q) cov[li * 6 + q] = 0.0f;
                if (TM) {
                    hb[li] = 0;
                    missb[li] = 0;
                    ib[li * 2] = 0.0f;
                    ib[li * 2 + 1] = 0.0f;
                }
            }
        }
        if (TM && writer && miss_add) missb[li] += miss_add;
        // ---- phase 2: lane k applies rotation k to sample (step - k) ----
        // column k of the lower triangle (l00, l10, l11, l20, l21, l22)
        const int cd = k == 0 ? 0 : (k == 1 ? 2 : 5);
        const int ca = k == 0 ? 1 : 4, cbi = 3;
        double Ld = 0.0, La = 0.0, Lb = 0.0;
        double mu[3] = {0.0, 0.0, 0.0};
        double imean = 0.0, im2 = 0.0;
        if (ns) {
            if (!reset) {  // a reset zeroed the stored factor (and n0)
                Ld = (double)cov[li * 6 + cd];
                if (k < 2) La = (double)cov[li * 6 + ca];
                if (k == 0) Lb = (double)cov[li * 6 + cbi];
            }
            if (k == 0 && n0 > 0) {
                double off[3];
                unpack_mean(mb[li], off);
#pragma unroll
                for (int a = 0; a < 3; ++a) mu[a] = ((double)g[a] + off[a]) * m.vox;
            }
            if (TM && k == 0) {
                imean = ib[li * 2];
                im2 = ib[li * 2 + 1];
            }
        }
        const double4 *__restrict__ ps = b.pos + s + np1;
        const unsigned ms = __reduce_max_sync(0xffffffffu, ns);
        double oa = 0.0, ob = 0.0;  // this lane's rotated vector entries, for lane k + 1
        // lane 0: the next sample's end point is loaded a step ahead of its use
        double4 curp = (k == 0 && ns) ? ld_d4(ps) : make_double4(0.0, 0.0, 0.0, 0.0);
        // this lane's first sample's roots; the next sample's are loaded a step ahead
        double4 rtp = ns ? ndt_roots_of(b, n0) : make_double4(0.0, 0.0, 0.0, 0.0);
        for (unsigned step = 0; step < ms + 2; ++step) {
            const double ind = __shfl_up_sync(0xffffffffu, oa, 1);
            const double ina = __shfl_up_sync(0xffffffffu, ob, 1);
            const unsigned j = step - (unsigned)k;  // this lane's sample (wraps when step < k)
            if (j < ns) {
                const unsigned long long nj = (unsigned long long)n0 + j;
                const double4 rtc = rtp;
                if (j + 1 < ns) rtp = ndt_roots_of(b, nj + 1);
                double e[3] = {0.0, 0.0, 0.0};
                if (k == 0) {
                    const double4 cur = curp;
                    if (j + 1 < ns) curp = ld_d4(ps + j + 1);
                    l = clamp_add(l, m.hit32, m.cmin, m.cmax);
                    if (TM) {
                        const double val = cur.w, nn = (double)(nj + 1);
                        const double d = val - imean;
                        const double mnew = imean + d / nn;
                        const double m2new = im2 + d * (val - mnew);
                        imean = (double)(float)mnew;
                        im2 = (double)(float)m2new;
                    }
                    e[0] = cur.x;
                    e[1] = cur.y;
                    e[2] = cur.z;
                }
                bool ok = true;
                if (NBK3_FAST) {
                    double mu2[3] = {mu[0], mu[1], mu[2]};
                    double Ld2 = Ld, La2 = La, Lb2 = Lb, oa2, ob2;
                    ndt_fold3_step<true>(k, nj, e, rtc, mu2, ind, ina, Ld2, La2, Lb2, oa2, ob2, ok);
                    if (ok) {
                        mu[0] = mu2[0];
                        mu[1] = mu2[1];
                        mu[2] = mu2[2];
                        Ld = Ld2;
                        La = La2;
                        Lb = Lb2;
                        oa = oa2;
                        ob = ob2;
                    }
                }
                if (!NBK3_FAST || !ok) ndt_fold3_step<false>(k, nj, e, rtc, mu, ind, ina, Ld, La, Lb, oa, ob, ok);
            }
        }
        const unsigned long long n = (unsigned long long)n0 + ns;
        if (ns && act) {
            cov[li * 6 + cd] = (float)Ld;
            if (k < 2) cov[li * 6 + ca] = (float)La;
            if (k == 0) cov[li * 6 + cbi] = (float)Lb;
        }
        if (ns && writer) {
            if (TM) {
                ib[li * 2] = (float)imean;
                ib[li * 2 + 1] = (float)im2;
                hb[li] += ns;
            }
            cb[li] = n > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)n;
            if (n >= 3 && m.gmask)
                atomicOr(m.gmask + slot, m.brick_shift >= 0 ? 1u << brick_of(li, m.bsh) : 0xFFFFFFFFu);
            double frac[3];
            const double hi = 1.0 - 1.0 / 2048.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                double f = mu[a] / m.vox - (double)g[a];
                if (f < 0.0) f = 0.0;
                if (f > hi) f = hi;
                frac[a] = f;
            }
            mb[li] = pack_mean(frac);
        }
        if (writer) {
            occ[li] = l;
            layer_at<unsigned>(m, m.nidx, slot)[li] = 0u;
        }
#ifdef VM_FOLD_PROF
        if (lane == 0) {
            const unsigned long long dt = (unsigned long long)(clock64() - prof_t0);
            atomicMax(&g_fold_prof[0], (dt << 24) | ((unsigned long long)min(mp1, 4095u) << 12) |
                                           min(ms, 4095u));
            atomicAdd(&g_fold_prof[1], dt);
        }
#endif
    }
}

// Deterministic TSDF (reference.py:153-175): one thread per voxel bucket
// merges the voxel's band visits in ray order; clears the index stamp and
// the bucket count.
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_tsdf_fold(const __grid_constant__ DevMap m, Src src,
                                                     NdtBuckets b) {
    unsigned long long R, M;
    if (!bk_ndt_live(m, R, M)) return;
    const unsigned K = *((volatile unsigned *)(b.cursor + NBK_BINS));
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < K; t += gridDim.x * blockDim.x) {
        const unsigned mi = b.perm[t];
        unsigned c;
        const unsigned s = nbk_start(b, mi, c);
        b.cnt[mi] = 0u;
        b.cnt2[mi] = 0u;
        const int2 sl = m.marked[mi];
        if (sl.x < 0) continue;
        const int slot = sl.x, li = sl.y;
        int g[3];
        slot_li_to_g(m, slot, li, g);
        float *buf = layer_at<float>(m, L_TSDF, slot);
        float fd = buf[2 * li], fw = buf[2 * li + 1];
        for (unsigned i = 0; i < c; ++i) {
            const long long ray = (long long)((b.val[s + i] >> 32) & 0x7FFFFFFFULL);
            Ray r;
            src.load(ray, r.o, r.e, r.has, r.inten);
            prep_ray(m, r, false);
            double d[3];
            for (int a = 0; a < 3; ++a) d[a] = (r.e[a] - r.o[a]) / r.L;
            const double cc[3] = {((double)g[0] + 0.5) * m.vox - r.o[0],
                                  ((double)g[1] + 0.5) * m.vox - r.o[1],
                                  ((double)g[2] + 0.5) * m.vox - r.o[2]};
            double dv = r.L - dot3(cc, d);
            if (dv < -m.tsdf_trunc) dv = -m.tsdf_trunc;
            if (dv > m.tsdf_trunc) dv = m.tsdf_trunc;
            const double w = fw;
            fd = (float)((w * (double)fd + dv) / (w + 1.0));
            double nw = w + 1.0;
            if (nw > m.tsdf_maxw) nw = m.tsdf_maxw;
            fw = (float)nw;
        }
        buf[2 * li] = fd;
        buf[2 * li + 1] = fw;
        layer_at<unsigned>(m, m.nidx, slot)[li] = 0u;
    }
}

// Refused / failed batches leave index stamps behind: clear every stamped
// word of the first `words` voxels (the list of indices is not trusted).
__global__ void k_nbk_clear(const __grid_constant__ DevMap m, long long words) {
    unsigned *w = reinterpret_cast<unsigned *>(m.slab[m.nidx]);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < words;
         k += (long long)gridDim.x * blockDim.x)
        if (w[k]) w[k] = 0u;
}

}  // namespace vm
