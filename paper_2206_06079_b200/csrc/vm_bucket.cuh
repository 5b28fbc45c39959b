// vm_bucket.cuh -- the in-order fold of the deterministic occupancy path
// without a global record sort and without a host round trip.
//
// The walk's records are (sample-voxel index mi) << ob | (ray*maxseg + seg) << 1 | hit
// (key_mi; k_discover numbered the batch's sample voxels).  Instead of
// radix-sorting all of them, the records are bucketed by mi -- one counting
// pass, a slice allocation (one atomic per warp, no scan), one scatter of the
// 32-bit (order, hit) payloads -- and each bucket is put in ray order on its own:
//
//   <= BK_SERIAL records   one thread: insertion sort in registers/local memory
//   <= BK_SMEM records     one block: bitonic sort in shared memory
//   larger                 one block: presence / hit bitmaps over the batch's
//                          order space in global scratch, scanned in order
//
// then folded exactly like fold_voxel_serial (reference.py:35-64 restricted
// to the voxel: f_miss^k between hits, clamped hit, packed-mean fold).
//
// Every count these kernels need (records R, sample voxels M, big buckets)
// is read on the device, so the host enqueues the whole batch and syncs once
// at its end.  A batch whose records overflowed (R > rec_cap) or that the
// guard refused (go == 0) is a no-op here; the host re-runs it after the sync.
#pragma once

#include "vm_kernels.cuh"

namespace vm {

#ifndef BK_FOLD_MINB
#define BK_FOLD_MINB 1  // k_bk_fold resident blocks per SM (register budget)
#endif

#ifndef VM_BK_BIG_BPS
#define VM_BK_BIG_BPS 4
#endif
// k_bk_fold_big blocks per SM: one bucket per block at a time, whose serial
// fold keeps one warp busy while the others wait -- several buckets per SM
constexpr int BK_BIG_BPS = VM_BK_BIG_BPS;
constexpr int BK_SERIAL = 16;
constexpr int BK_WARP = 1024;  // one warp sorts (bitonic, shared memory) and folds up to this
constexpr int BK_SMEM = 4096;

struct BucketState {
    unsigned *cnt;               // [M + 1] records per bucket (all zero between batches)
    unsigned *off;               // [M + 1] slice offset (k_bk_alloc), bumped by the scatter
    unsigned *cursor;            // slice allocation cursor (zeroed per batch)
    unsigned *val;               // [R] bucketed (order << 1 | hit) payloads
    int *big;                    // buckets for the block kernel (> BK_WARP records)
    unsigned long long *nbig;
    int *mid;                    // buckets for the warp kernel (BK_SERIAL < records <= BK_WARP)
    unsigned long long *nmid;
    unsigned *bits;              // huge buckets: per block 2 * bwords words
    unsigned long long bwords;   // words of one bitmap (order space / 32)
};

__device__ __forceinline__ bool bk_live(const DevMap &m, unsigned long long &R,
                                        unsigned long long &M) {
    if (!read_go(m)) return false;
    R = *((volatile unsigned long long *)(m.stats + S_RECORDS));
    if (R > m.rec_cap) {  // overflow: the host re-emits and re-runs
        if (m.chain) atomicCAS(m.chain, 0, m.batch_idx + 1);
        return false;
    }
    M = min(*((volatile unsigned long long *)m.nmarked), m.marked_cap);
    return true;
}

__global__ void __launch_bounds__(BLOCK) k_bk_count(const __grid_constant__ DevMap m,
                                                    BucketState b) {
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    const int ob = m.order_bits;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long mi = m.rec[i] >> ob;
        if (mi < M) atomicAdd(b.cnt + mi, 1u);
    }
}

// Each bucket's slice: one atomic per warp on a slice cursor (the slices need
// not follow the sample-voxel order, so no scan)
__global__ void __launch_bounds__(BLOCK) k_bk_alloc(const __grid_constant__ DevMap m, BucketState b,
                                                    bool classify) {
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    const int lane = threadIdx.x & 31;
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < M;
         base += (unsigned long long)gridDim.x * blockDim.x) {
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
        if (lane == 31 && tot) wb = atomicAdd(b.cursor, tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        if (mi < M) b.off[mi] = wb + incl - c;
        // classify: the fused fold (k_bk_fold_all) reads the warp / block lists
        if (classify && c > (unsigned)BK_SERIAL) {
            if (c <= (unsigned)BK_WARP) b.mid[atomicAdd(b.nmid, 1ULL)] = (int)mi;
            else b.big[atomicAdd(b.nbig, 1ULL)] = (int)mi;
        }
    }
}

// the scatter bumps each bucket's offset past its records; the slice is then
// [off - cnt, off) (bk_slice), and the folds zero cnt for the next batch
__global__ void __launch_bounds__(BLOCK) k_bk_scatter(const __grid_constant__ DevMap m,
                                                      BucketState b) {
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    const int ob = m.order_bits;
    const unsigned long long omask = (1ULL << ob) - 1;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = m.rec[i];
        const unsigned long long mi = k >> ob;
        if (mi >= M) continue;
        const unsigned pos = atomicAdd(b.off + mi, 1u);
        b.val[pos] = (unsigned)(k & omask);
    }
}

__device__ __forceinline__ unsigned bk_slice(const BucketState &b, unsigned long long mi, unsigned &c) {
    c = b.cnt[mi];
    return b.off[mi] - c;
}

// Per-voxel fold state: log-odds, packed mean, count, pending misses.
struct VoxFold {
    float l;
    unsigned packed, count, misses;
    int g[3];
    unsigned vid;
};

__device__ __forceinline__ void vf_begin(const DevMap &m, VoxFold &f, unsigned vid) {
    f.vid = vid;
    f.l = reinterpret_cast<const float *>(m.slab[L_OCC])[vid];
    f.packed = m.slab[L_MEAN] ? reinterpret_cast<const unsigned *>(m.slab[L_MEAN])[vid] : 0u;
    f.count = m.slab[L_COUNT] ? reinterpret_cast<const unsigned *>(m.slab[L_COUNT])[vid] : 0u;
    f.misses = 0;
    slot_li_to_g(m, (int)(vid / (unsigned)m.vpr), (int)(vid % (unsigned)m.vpr), f.g);
}

// one hit with sample end point ep, after the misses counted so far
// (reference.py:43-57)
#ifndef BK_FAST
#define BK_FAST 0  // 1: verified fast divisions in the hit step (measured slower, DESIGN)
#endif
template <bool FAST>
__device__ __forceinline__ void vf_mean_hit(const DevMap &m, const int g[3], const double ep[3],
                                            unsigned &packed, unsigned &count, bool &ok) {
    const double off[3] = {vdiv<FAST>(ep[0], m.vox, ok) - (double)g[0],
                           vdiv<FAST>(ep[1], m.vox, ok) - (double)g[1],
                           vdiv<FAST>(ep[2], m.vox, ok) - (double)g[2]};
    fold_mean_v<FAST>(packed, count, off, ok);
}

// The six divisions of a hit (the end point's voxel fraction, the running
// mean) are independent; BK_FAST issues them as the verified branch-free
// operators (vm_device.cuh: xdiv; a hit whose check fails is redone with
// IEEE division).  Measured slower than IEEE division (C2@0.1 m fold 9.2 ->
// 10.7 ms per step), so off.
__device__ __forceinline__ void vf_hit_ep(const DevMap &m, VoxFold &f, const double ep[3]) {
    f.l = miss_k(f.l, f.misses, m.miss32, m.cmin, m.cmax);
    f.misses = 0;
    f.l = clamp_add(f.l, m.hit32, m.cmin, m.cmax);
    if (m.slab[L_MEAN]) {
        bool ok = true;
        if (BK_FAST) {
            unsigned p2 = f.packed, c2 = f.count;
            vf_mean_hit<true>(m, f.g, ep, p2, c2, ok);
            if (ok) {
                f.packed = p2;
                f.count = c2;
            }
        }
        if (!BK_FAST || !ok) vf_mean_hit<false>(m, f.g, ep, f.packed, f.count, ok);
    }
}

// The same hit with the end point's voxel fraction ep / vox - g already
// computed (by the lane that loaded the end point, off the serial chain:
// the divisions are the same operations, only issued earlier).
__device__ __forceinline__ void vf_hit_off(const DevMap &m, VoxFold &f, const double off[3]) {
    f.l = miss_k(f.l, f.misses, m.miss32, m.cmin, m.cmax);
    f.misses = 0;
    f.l = clamp_add(f.l, m.hit32, m.cmin, m.cmax);
    if (m.slab[L_MEAN]) fold_mean(f.packed, f.count, off);
}

// every lane: the voxel fraction of the end point it loaded (vf_lane_end)
__device__ __forceinline__ void vf_lane_off(const DevMap &m, const VoxFold &f, double e[3]) {
    if (!m.slab[L_MEAN]) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) e[a] = e[a] / m.vox - (double)f.g[a];
}

// ... of segment order index `oi` (= ray * maxseg + seg)
template <class Src>
__device__ __forceinline__ void vf_hit(const DevMap &m, const Src &src, VoxFold &f, unsigned oi) {
    double ep[3] = {0.0, 0.0, 0.0};
    if (m.slab[L_MEAN]) {
        float it;
        src.load_end((long long)(oi / (unsigned)m.maxseg), ep, it);
    }
    vf_hit_ep(m, f, ep);
}

// The end point of a lane's hit record, loaded by every lane at once before
// a warp folds a run serially (the loads leave the serial chain; the fold
// then takes each hit's point from its lane)
template <class Src>
__device__ __forceinline__ void vf_lane_end(const DevMap &m, const Src &src, bool hit, unsigned oi,
                                            double e[3]) {
    e[0] = e[1] = e[2] = 0.0;
    if (hit && m.slab[L_MEAN]) {
        float it;
        src.load_end((long long)(oi / (unsigned)m.maxseg), e, it);
    }
}

__device__ __forceinline__ void vf_end(const DevMap &m, VoxFold &f) {
    f.l = miss_k(f.l, f.misses, m.miss32, m.cmin, m.cmax);
    reinterpret_cast<float *>(m.slab[L_OCC])[f.vid] = f.l;
    if (m.slab[L_MEAN]) {
        reinterpret_cast<unsigned *>(m.slab[L_MEAN])[f.vid] = f.packed;
        reinterpret_cast<unsigned *>(m.slab[L_COUNT])[f.vid] = f.count;
    }
    reinterpret_cast<unsigned *>(m.slab[L_SCRATCH])[f.vid] = 0u;  // the MARK stamp
    m.bmask[f.vid / (unsigned)m.vpr] = 0u;
}

__device__ __forceinline__ unsigned marked_vid(const DevMap &m, unsigned long long mi) {
    const int2 sl = m.marked[mi];
    return (unsigned)sl.x * (unsigned)m.vpr + (unsigned)sl.y;
}

// One thread per sample voxel: small buckets sorted and folded in place.
template <class Src>
__global__ void __launch_bounds__(BLOCK, BK_FOLD_MINB) k_bk_fold(const __grid_constant__ DevMap m, Src src,
                                                   BucketState b) {
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    for (unsigned long long mi = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; mi < M;
         mi += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned c;
        const unsigned s = bk_slice(b, mi, c);
        if (c == 0u) continue;  // an index whose claim lost a race (marked (-1, -1))
        if (c > (unsigned)BK_SERIAL) {
            if (c <= (unsigned)BK_WARP) b.mid[atomicAdd(b.nmid, 1ULL)] = (int)mi;
            else b.big[atomicAdd(b.nbig, 1ULL)] = (int)mi;
            continue;
        }
        b.cnt[mi] = 0u;
        unsigned v[BK_SERIAL];
        for (unsigned i = 0; i < c; ++i) {
            const unsigned x = b.val[s + i];
            int j = (int)i - 1;
            while (j >= 0 && v[j] > x) {
                v[j + 1] = v[j];
                --j;
            }
            v[j + 1] = x;
        }
        VoxFold f;
        vf_begin(m, f, marked_vid(m, mi));
        for (unsigned i = 0; i < c; ++i) {
            if (v[i] & 1u) vf_hit(m, src, f, v[i] >> 1);
            else ++f.misses;
        }
        vf_end(m, f);
    }
}

// Fold a sorted run held by one warp, 32 payloads at a time (lane i holds
// element base + i; `n` valid).  Misses between hits collapse to f_miss^k.
template <class Src>
__device__ __forceinline__ void vf_warp_chunk(const DevMap &m, const Src &src, VoxFold &f,
                                              unsigned x, int n) {
    const int lane = threadIdx.x & 31;
    const bool hit = lane < n && (x & 1u);
    const unsigned hmask = __ballot_sync(0xffffffffu, hit);
    double e[3];
    vf_lane_end(m, src, hit, x >> 1, e);  // all the chunk's end points in flight at once
    vf_lane_off(m, f, e);                 // and their voxel fractions, all lanes at once
    int cur = 0;
    unsigned hm = hmask;
    while (hm) {
        const int h = __ffs(hm) - 1;
        hm &= hm - 1;
        f.misses += (unsigned)(h - cur);
        const double off[3] = {__shfl_sync(0xffffffffu, e[0], h), __shfl_sync(0xffffffffu, e[1], h),
                               __shfl_sync(0xffffffffu, e[2], h)};
        vf_hit_off(m, f, off);
        cur = h + 1;
    }
    f.misses += (unsigned)(n - cur);
}

// One warp per medium bucket: bitonic sort of the padded slice in the warp's
// shared-memory window (warp-synchronous), then the chunked fold -- no block
// barrier, so every warp of the block folds its own bucket.
template <class Src>
__device__ __forceinline__ void bk_fold_mid_body(const DevMap &m, const Src &src, const BucketState &b,
                                                 unsigned (*sv)[BK_WARP], unsigned bid, unsigned nblk) {
    const unsigned long long nm = *((volatile unsigned long long *)b.nmid);
    const int lane = threadIdx.x & 31;
    unsigned *const w = sv[threadIdx.x >> 5];
    const unsigned long long nw = (unsigned long long)nblk * (BLOCK / 32);
    for (unsigned long long t = (unsigned long long)bid * (BLOCK / 32) + (threadIdx.x >> 5);
         t < nm; t += nw) {
        const unsigned long long mi = (unsigned long long)b.mid[t];
        unsigned c;
        const unsigned s = bk_slice(b, mi, c);
        __syncwarp();
        if (lane == 0) b.cnt[mi] = 0u;
        unsigned P = 32;
        while (P < c) P <<= 1;
        for (unsigned i = lane; i < P; i += 32) w[i] = i < c ? b.val[s + i] : 0xFFFFFFFFu;
        __syncwarp();
        for (unsigned k = 2; k <= P; k <<= 1) {
            for (unsigned j = k >> 1; j > 0; j >>= 1) {
                for (unsigned i = lane; i < P; i += 32) {
                    const unsigned p = i ^ j;
                    if (p > i) {
                        const unsigned a = w[i], bb = w[p];
                        if ((a > bb) == ((i & k) == 0)) {
                            w[i] = bb;
                            w[p] = a;
                        }
                    }
                }
                __syncwarp();
            }
        }
        VoxFold f;
        vf_begin(m, f, marked_vid(m, mi));
        for (unsigned base = 0; base < c; base += 32) {
            const int n = (int)min(32u, c - base);
            const unsigned x = lane < n ? w[base + lane] : 0u;
            vf_warp_chunk(m, src, f, x, n);
        }
        if (lane == 0) vf_end(m, f);
        __syncwarp();
    }
}

template <class Src>
__global__ void __launch_bounds__(BLOCK) k_bk_fold_mid(const __grid_constant__ DevMap m, Src src,
                                                       BucketState b) {
    __shared__ unsigned sv[BLOCK / 32][BK_WARP];
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    bk_fold_mid_body(m, src, b, sv, blockIdx.x, gridDim.x);
}

// One block per large bucket.
template <class Src>
__device__ __forceinline__ void bk_fold_big_body(const DevMap &m, const Src &src, const BucketState &b,
                                                 unsigned *sv, unsigned bid, unsigned nblk) {
    const unsigned long long nb = *((volatile unsigned long long *)b.nbig);
    const int lane = threadIdx.x & 31;
    unsigned *pres = b.bits + (size_t)bid * 2 * b.bwords;
    unsigned *hitb = pres + b.bwords;
    for (unsigned long long w = bid; w < nb; w += nblk) {
        const unsigned long long mi = (unsigned long long)b.big[w];
        unsigned c;
        const unsigned s = bk_slice(b, mi, c);
        __syncthreads();  // every thread has read cnt before it is zeroed
        if (threadIdx.x == 0) b.cnt[mi] = 0u;
        VoxFold f;
        if (c <= (unsigned)BK_SMEM) {
            unsigned P = 32;
            while (P < c) P <<= 1;
            for (unsigned i = threadIdx.x; i < P; i += blockDim.x)
                sv[i] = i < c ? b.val[s + i] : 0xFFFFFFFFu;
            __syncthreads();
            for (unsigned k = 2; k <= P; k <<= 1) {
                for (unsigned j = k >> 1; j > 0; j >>= 1) {
                    for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
                        const unsigned p = i ^ j;
                        if (p > i) {
                            const unsigned a = sv[i], bb = sv[p];
                            const bool up = (i & k) == 0;
                            if ((a > bb) == up) {
                                sv[i] = bb;
                                sv[p] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            if (threadIdx.x < 32) {
                vf_begin(m, f, marked_vid(m, mi));
                for (unsigned base = 0; base < c; base += 32) {
                    const int n = (int)min(32u, c - base);
                    const unsigned x = lane < n ? sv[base + lane] : 0u;
                    vf_warp_chunk(m, src, f, x, n);
                }
                if (lane == 0) vf_end(m, f);
            }
            __syncthreads();
        } else {
            // presence / hit bitmaps over the order space, scanned in order
            for (unsigned long long i = threadIdx.x; i < 2 * b.bwords; i += blockDim.x) pres[i] = 0u;
            __syncthreads();
            for (unsigned i = threadIdx.x; i < c; i += blockDim.x) {
                const unsigned x = b.val[s + i];
                const unsigned oi = x >> 1;
                atomicOr(pres + (oi >> 5), 1u << (oi & 31));
                if (x & 1u) atomicOr(hitb + (oi >> 5), 1u << (oi & 31));
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                vf_begin(m, f, marked_vid(m, mi));
                for (unsigned long long w0 = 0; w0 < b.bwords; w0 += 32) {
                    const unsigned long long wi = w0 + lane;
                    const unsigned p = wi < b.bwords ? __ldcg(pres + wi) : 0u;
                    const unsigned h = wi < b.bwords ? __ldcg(hitb + wi) : 0u;
                    const unsigned withhits = __ballot_sync(0xffffffffu, h != 0u);
                    // lanes without hits contribute whole-word miss counts
                    unsigned before = 0;  // misses in hit-free words of lower lanes, per segment
                    int prev = 0;
                    unsigned wh = withhits;
                    while (wh) {
                        const int L = __ffs(wh) - 1;
                        wh &= wh - 1;
                        // misses of the hit-free words in lanes [prev, L)
                        const bool inr = lane >= prev && lane < L;
                        before = __reduce_add_sync(0xffffffffu, inr ? __popc(p) : 0u);
                        f.misses += before;
                        const unsigned pL = __shfl_sync(0xffffffffu, p, L);
                        const unsigned hL = __shfl_sync(0xffffffffu, h, L);
                        // lane j loads the end point of order (w0 + L) * 32 + j if it hit
                        double e[3];
                        vf_lane_end(m, src, (hL >> lane) & 1u, (unsigned)((w0 + L) * 32 + lane), e);
                        vf_lane_off(m, f, e);
                        unsigned bits = pL;
                        while (bits) {
                            const int bi = __ffs(bits) - 1;
                            bits &= bits - 1;
                            if ((hL >> bi) & 1u) {
                                const double off[3] = {__shfl_sync(0xffffffffu, e[0], bi),
                                                       __shfl_sync(0xffffffffu, e[1], bi),
                                                       __shfl_sync(0xffffffffu, e[2], bi)};
                                vf_hit_off(m, f, off);
                            } else {
                                ++f.misses;
                            }
                        }
                        prev = L + 1;
                    }
                    f.misses += __reduce_add_sync(0xffffffffu, lane >= prev ? __popc(p) : 0u);
                }
                if (lane == 0) vf_end(m, f);
            }
            __syncthreads();
        }
    }
}

template <class Src>
__global__ void __launch_bounds__(BLOCK) k_bk_fold_big(const __grid_constant__ DevMap m, Src src,
                                                       BucketState b) {
    __shared__ unsigned sv[BK_SMEM];
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    bk_fold_big_body(m, src, b, sv, blockIdx.x, gridDim.x);
}

// The three folds in one launch, by block roles: [0, nbig_blocks) the block
// buckets, then nmid_blocks of warp buckets, the rest one thread per small
// bucket (k_bk_alloc classified them with classify = true).  A bucket's
// fold does not depend on another's, so the long serial chains of the
// largest buckets (dispatched first) run beside the rest instead of after it.
template <class Src>
__global__ void __launch_bounds__(BLOCK, 4) k_bk_fold_all(const __grid_constant__ DevMap m, Src src,
                                                          BucketState b, int nbig_blocks,
                                                          int nmid_blocks) {
    __shared__ union {
        unsigned mid[BLOCK / 32][BK_WARP];
        unsigned big[BK_SMEM];
    } sh;
    unsigned long long R, M;
    if (!bk_live(m, R, M)) return;
    const int bid = (int)blockIdx.x;
    if (bid < nbig_blocks) {
        bk_fold_big_body(m, src, b, sh.big, (unsigned)bid, (unsigned)nbig_blocks);
        return;
    }
    if (bid < nbig_blocks + nmid_blocks) {
        bk_fold_mid_body(m, src, b, sh.mid, (unsigned)(bid - nbig_blocks), (unsigned)nmid_blocks);
        return;
    }
    const unsigned long long nsmall =
        (unsigned long long)(gridDim.x - (unsigned)(nbig_blocks + nmid_blocks)) * blockDim.x;
    for (unsigned long long mi = (unsigned long long)(bid - nbig_blocks - nmid_blocks) * blockDim.x +
                                 threadIdx.x;
         mi < M; mi += nsmall) {
        unsigned c;
        const unsigned s = bk_slice(b, mi, c);
        if (c == 0u || c > (unsigned)BK_SERIAL) continue;
        b.cnt[mi] = 0u;
        unsigned v[BK_SERIAL];
        for (unsigned i = 0; i < c; ++i) {
            const unsigned x = b.val[s + i];
            int j = (int)i - 1;
            while (j >= 0 && v[j] > x) {
                v[j + 1] = v[j];
                --j;
            }
            v[j + 1] = x;
        }
        VoxFold f;
        vf_begin(m, f, marked_vid(m, mi));
        for (unsigned i = 0; i < c; ++i) {
            if (v[i] & 1u) vf_hit(m, src, f, v[i] >> 1);
            else ++f.misses;
        }
        vf_end(m, f);
    }
}

}  // namespace vm
