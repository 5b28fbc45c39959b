// vm_kernels.cuh -- the batch kernels of the ray-integration path.
//
// Pipeline of one batch (vm_runtime.cu drives it on the map's stream):
//
//   k_discover   one thread per ray: clip + segment (traversal.py:140-178),
//                coarse region DDA = prefetch_regions (engine.py:99-118),
//                region insertion into the HBM table, sample-voxel marks
//                (deterministic mode) and NDT phase-2 hit records.
//   k_guard      refuses the batch (go = 0) if the region pool would
//                overflow; the host grows the pool and replays.
//   k_walk_*     one thread per ray: exact fp64 DDA over every segment and
//                the per-visit update (CAS, or RED miss counts + order-keyed
//                records for sample voxels).
//   k_resolve    deterministic miss counts -> f_miss^k per voxel.
//   sort         CUB radix sort of the records (voxel-major, ray order).
//   k_fold_*     in-order fold of the records per voxel (warp per long run);
//                clears the sample voxels' MARK'ed scratch words.
#pragma once

#include "vm_device.cuh"

namespace vm {

constexpr int BLOCK = 256;
constexpr int REC_STAGE = 2048;  // per-block staging of records (16 KiB)

// --------------------------------------------------------------- helpers

// Block-staged append: smem slots first, one global atomic per block.
template <class T, int CAP>
struct Stage {
    T *buf;
    int *n;
    __device__ __forceinline__ void push(T v, T *gbuf, unsigned long long *gcount,
                                         unsigned long long gcap) {
        int i = atomicAdd(n, 1);
        if (i < CAP) {
            buf[i] = v;
        } else {
            unsigned long long g = atomicAdd(gcount, 1ULL);
            if (g < gcap) gbuf[g] = v;
        }
    }
};

__device__ __forceinline__ unsigned cas_apply_k(float *p, float d, unsigned k, float cmin,
                                                float cmax) {
    unsigned retries = 0;
    unsigned old = __float_as_uint(__ldcg(p));
    for (;;) {
        float nl = miss_k(__uint_as_float(old), k, d, cmin, cmax);
        unsigned nb = __float_as_uint(nl);
        if (nb == old) return retries;  // f^k(l) == l: nothing to write
        unsigned prev = atomicCAS(reinterpret_cast<unsigned *>(p), old, nb);
        if (prev == old) return retries;
        old = prev;
        ++retries;
    }
}

// _kernels.pyx:318-357 with the oracle's fold (subvoxel.py:34-49)
__device__ __forceinline__ unsigned cas_mean(unsigned *mean, unsigned *cnt, const double off[3]) {
    unsigned n_old = atomicAdd(cnt, 1u);
    if (n_old == 0xFFFFFFFFu) {
        atomicExch(cnt, 0xFFFFFFFFu);
        return 0;
    }
    unsigned retries = 0;
    unsigned old = __ldcg(mean);
    for (;;) {
        unsigned packed = old, c = n_old;
        fold_mean(packed, c, off);
        unsigned prev = atomicCAS(mean, old, packed);
        if (prev == old) return retries;
        old = prev;
        ++retries;
    }
}

// ndt.gaussian_miss_weight via the adjugate of _kernels.pyx:473-525
__device__ __forceinline__ double gaussian_weight(const double mu[3], const float c6[6],
                                                  double sigma2, const double o[3],
                                                  const double v[3], double t0, double t1) {
    double s0 = c6[0], s1 = c6[1], s2 = c6[2], s3 = c6[3], s4 = c6[4], s5 = c6[5];
    double a00 = s0 * s0 + sigma2, a01 = s0 * s1, a02 = s0 * s3;
    double a11 = s1 * s1 + s2 * s2 + sigma2, a12 = s1 * s3 + s2 * s4;
    double a22 = s3 * s3 + s4 * s4 + s5 * s5 + sigma2;
    double c00 = a11 * a22 - a12 * a12, c01 = a02 * a12 - a01 * a22, c02 = a01 * a12 - a02 * a11;
    double det = a00 * c00 + a01 * c01 + a02 * c02;
    if (det <= 0) return 1.0;
    double i00 = c00 / det, i01 = c01 / det, i02 = c02 / det;
    double i11 = (a00 * a22 - a02 * a02) / det;
    double i12 = (a02 * a01 - a00 * a12) / det;
    double i22 = (a00 * a11 - a01 * a01) / det;
    double wx = mu[0] - o[0], wy = mu[1] - o[1], wz = mu[2] - o[2];
    double vx = v[0], vy = v[1], vz = v[2];
    double denom = vx * (i00 * vx + i01 * vy + i02 * vz) + vy * (i01 * vx + i11 * vy + i12 * vz) +
                   vz * (i02 * vx + i12 * vy + i22 * vz);
    double t;
    if (denom <= 0) {
        t = t0;
    } else {
        t = (vx * (i00 * wx + i01 * wy + i02 * wz) + vy * (i01 * wx + i11 * wy + i12 * wz) +
             vz * (i02 * wx + i12 * wy + i22 * wz)) / denom;
        if (t < t0) t = t0;
        else if (t > t1) t = t1;
    }
    double dx = o[0] + t * vx - mu[0], dy = o[1] + t * vy - mu[1], dz = o[2] + t * vz - mu[2];
    double m2 = dx * (i00 * dx + i01 * dy + i02 * dz) + dy * (i01 * dx + i11 * dy + i12 * dz) +
                dz * (i02 * dx + i12 * dy + i22 * dz);
    return exp(-0.5 * m2);
}

// the batch may run: its guard let it, and no earlier batch of a pipelined
// sequence stopped the chain (chain = failing batch + 1)
__device__ __forceinline__ int read_go(const DevMap &m) {
    if (m.chain) {
        const int c = *((volatile int *)m.chain);
        if (c && c <= m.batch_idx) return 0;
    }
    return *((volatile int *)m.go);
}

constexpr int RP_BIAS = 512;  // bias of the walks' grid-relative region coordinates

// The grid-relative region coordinates of the descriptor walks (k_walk_det,
// k_walk_ndt_det) must stay inside their 10-bit fields: batches whose
// prefetched box spans RP_BIAS - 2 regions or more on an axis (800 m at
// 0.05 m voxels) take the generic walks (k_walk, k_walk_ndt) instead.
__device__ __forceinline__ bool walk_det_ok(const DevMap &m) {
    return m.rbox[3] - m.rbox[0] < RP_BIAS - 3 && m.rbox[4] - m.rbox[1] < RP_BIAS - 3 &&
           m.rbox[5] - m.rbox[2] < RP_BIAS - 3;
}

// Global voxel coordinate of (slot, li) (keys.py:50-56).
__device__ __forceinline__ void slot_li_to_g(const DevMap &m, int slot, int li, int g[3]) {
    int r[3];
    unpack_region(m.slot_keys[slot], r);
    int lx = li % m.dim, t = li / m.dim;
    int ly = t % m.dim, lz = t / m.dim;
    g[0] = r[0] * m.dim + lx;
    g[1] = r[1] * m.dim + ly;
    g[2] = r[2] * m.dim + lz;
}

__device__ __forceinline__ bool in_range(const DevMap &m, const double p[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double c = floor(p[a] / m.vox);
        if (!(c > -(double)m.cell_limit && c < (double)m.cell_limit)) return false;
    }
    return true;
}

// Record the region as touched by the walk (needed by k_resolve).
__device__ __forceinline__ void touch_region(const DevMap &m, int *sset, int slot) {
    if (!slotset_insert(sset, slot)) return;
    if (stamp_epoch(m.slot_touch + slot, m.epoch)) {
        unsigned long long idx = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
        if (idx < (unsigned long long)m.touched_cap) m.touched[idx] = slot;
    }
}

template <class T>
__device__ __forceinline__ T *layer_at(const DevMap &m, int layer, int slot) {
    return m.lptr[layer] ? reinterpret_cast<T *>(m.lptr[layer][slot]) : nullptr;
}

// --------------------------------------------------------------- NDT record emission

constexpr unsigned NIDX_FLAG = 0x80000000u;  // index-layer stamp (vm_ndt.cuh)

// The bucket index of voxel (slot, li): the stamp in the index layer, or a
// fresh one.  Lock-free: a lost race leaves an unused index (empty bucket,
// marked (-1, -1)).  Returns 0xFFFFFFFF when the index list is full (the
// batch then re-runs with room for every index, see bk_ndt_live).
__device__ __forceinline__ unsigned ndt_index(const DevMap &m, int slot, int li) {
    unsigned *w = layer_at<unsigned>(m, m.nidx, slot) + li;
    unsigned cur = *((volatile unsigned *)w);
    if (cur & NIDX_FLAG) return cur & ~NIDX_FLAG;
    const unsigned long long mi = atomicAdd(m.nmarked, 1ULL);
    if (mi >= m.marked_cap || mi >= (unsigned long long)NIDX_FLAG) return 0xFFFFFFFFu;
    const unsigned prev = atomicCAS(w, 0u, NIDX_FLAG | (unsigned)mi);
    if (prev == 0u) {
        m.marked[mi] = make_int2(slot, li);
        return (unsigned)mi;
    }
    m.marked[mi] = make_int2(-1, -1);
    if (m.nlost) atomicAdd(m.nlost, 1ULL);  // the batch's distinct voxels: nmarked - nlost
    return prev & ~NIDX_FLAG;
}

// ndt_index for the occupancy sample-voxel list: counts the lost races in
// nmarked[1], so the list's live length is nmarked[0] - nmarked[1]
__device__ __forceinline__ unsigned claim_sample_voxel(const DevMap &m, int slot, int li) {
    unsigned *w = layer_at<unsigned>(m, m.nidx, slot) + li;
    const unsigned cur = *((volatile unsigned *)w);
    if (cur & NIDX_FLAG) return cur & ~NIDX_FLAG;
    const unsigned long long mi = atomicAdd(m.nmarked, 1ULL);
    if (mi >= m.marked_cap || mi >= (unsigned long long)NIDX_FLAG) return 0xFFFFFFFFu;
    const unsigned prev = atomicCAS(w, 0u, NIDX_FLAG | (unsigned)mi);
    if (prev == 0u) {
        m.marked[mi] = make_int2(slot, li);
        return (unsigned)mi;
    }
    m.marked[mi] = make_int2(-1, -1);
    atomicAdd(m.nmarked + 1, 1ULL);
    return prev & ~NIDX_FLAG;
}

__device__ __forceinline__ unsigned long long ndt_key(unsigned mi, unsigned phase, unsigned oi) {
    return ((unsigned long long)mi << 32) | ((unsigned long long)phase << 31) | oi;
}


// --------------------------------------------------------------- k_discover

// Per-block direct-mapped cache region -> slot, keyed by coordinates relative
// to a block anchor (13 bits per axis) so key + slot fit one 64-bit word.
#ifndef KCACHE_N
#define KCACHE_N 1024
#endif
constexpr int KCACHE = KCACHE_N;
struct KeyCache {
    unsigned long long *e;
    int ax, ay, az;
    // entry: bit 63 valid | bits 21..59 relative coords (13 bits each) | bits 0..20 slot + 2
    __device__ __forceinline__ bool rel(int rx, int ry, int rz, unsigned long long &tag,
                                        unsigned &idx) const {
        const unsigned ux = (unsigned)(rx - ax), uy = (unsigned)(ry - ay), uz = (unsigned)(rz - az);
        if ((ux | uy | uz) >= (1u << 13)) return false;
        tag = (unsigned long long)ux | ((unsigned long long)uy << 13) | ((unsigned long long)uz << 26);
        idx = (ux * 73856093u ^ uy * 19349663u ^ uz * 83492791u) & (KCACHE - 1);
        return true;
    }
    // slot, or -3 on a miss (-1/-2 are valid cached answers: absent / exhausted)
    __device__ __forceinline__ int find(int rx, int ry, int rz) const {
        unsigned long long tag;
        unsigned idx;
        if (!rel(rx, ry, rz, tag, idx)) return -3;
        const unsigned long long v = e[idx];
        if ((v >> 63) && ((v >> 21) & ((1ULL << 39) - 1)) == tag) return (int)(v & 0x1FFFFFu) - 2;
        return -3;
    }
    __device__ __forceinline__ void put(int rx, int ry, int rz, int slot) const {
        unsigned long long tag;
        unsigned idx;
        if (!rel(rx, ry, rz, tag, idx) || slot < -2 || slot >= (1 << 21) - 2) return;
        e[idx] = (1ULL << 63) | (tag << 21) | (unsigned long long)(slot + 2);
    }
};

__device__ __forceinline__ int cached_slot(const DevMap &m, const KeyCache &kc, int rx, int ry,
                                           int rz, bool *fresh) {
    int slot = kc.find(rx, ry, rz);
    *fresh = false;
    if (slot == -3) {
        slot = region_slot(m, pack_region(rx, ry, rz));
        kc.put(rx, ry, rz, slot);
        *fresh = true;
    }
    return slot;
}

// Coarse region DDA visitor (walk_regions, traversal.py:134-137).
struct PrefetchVisitor {
    const DevMap *m;
    const KeyCache *kc;
    int *sset;
    int lo[3], hi[3];
    __device__ __forceinline__ void begin(int, int, int) {}
    __device__ __forceinline__ void moved(int, int) {}
    __device__ __forceinline__ void jump(int, int, int) {}
    __device__ __forceinline__ void visit(int x, int y, int z, double, double, bool) {
        lo[0] = min(lo[0], x); lo[1] = min(lo[1], y); lo[2] = min(lo[2], z);
        hi[0] = max(hi[0], x); hi[1] = max(hi[1], y); hi[2] = max(hi[2], z);
        bool fresh;
        const int slot = cached_slot(*m, *kc, x, y, z, &fresh);
        if (slot == SLOT_SPILLED) {
            // a region evicted to disk: the batch must wait for its reload
            const unsigned long long k = atomicAdd(m->stats + S_SPILLED, 1ULL);
            if (m->reload && k < (unsigned long long)m->reload_cap) m->reload[k] = pack_region(x, y, z);
            return;
        }
        if (slot < 0 || !fresh) return;
        if (m->slot_last) m->slot_last[slot] = m->batch_no;
        if (!slotset_insert(sset, slot)) return;  // first sight of the region in this block only
        if (stamp_epoch(m->slot_pref + slot, m->epoch))
            atomicAdd(m->stats + S_PREF_TOUCHED, 1ULL);
        if (slot < m->cap && stamp_epoch(m->slot_touch + slot, m->epoch)) {
            unsigned long long t = atomicAdd(m->stats + S_WALK_TOUCHED, 1ULL);
            if (t < (unsigned long long)m->touched_cap) m->touched[t] = slot;
        }
    }
};

#ifndef DISC_BT
#define DISC_BT 512  // k_discover block size: more rays share a block's key cache
                     // (C2 discover: 128 -> 23.6, 256 -> 19.5, 512 -> 17.6 ms per step)
#endif

#ifndef DISC_MINB
#define DISC_MINB 2  // 2 x 512 threads per SM: the 64-register build (96 registers / 1 block: 17.5 -> 22.7 ms)
#endif

template <class Src>
__global__ void __launch_bounds__(DISC_BT, DISC_MINB) k_discover(const __grid_constant__ DevMap m, Src src,
                                                    long long n, int mode, int det, int emit,
                                                    int count_stats = 1) {
    if (m.chain && *((volatile int *)m.chain)) return;  // an earlier batch of the sequence failed
    __shared__ unsigned long long kcache[KCACHE];
    __shared__ int sset[SLOTSET];
    __shared__ unsigned long long srec[DISC_BT];
    __shared__ int nrec;
    __shared__ unsigned long long rec_base;
    __shared__ unsigned shist[SEG_BUCKETS];
    for (int i = threadIdx.x; i < SEG_BUCKETS; i += blockDim.x) shist[i] = 0u;
    __shared__ int anchor[3];
    for (int i = threadIdx.x; i < KCACHE; i += blockDim.x) kcache[i] = 0ULL;
    for (int i = threadIdx.x; i < SLOTSET; i += blockDim.x) sset[i] = -1;
    if (threadIdx.x == 0) {
        nrec = 0;
        const long long i0 = (long long)blockIdx.x * blockDim.x;
        double o0[3], e0[3];
        int h0;
        float it0;
        src.load(m.ray_lo + (i0 < n ? i0 : 0), o0, e0, h0, it0);
        for (int a = 0; a < 3; ++a) {
            const double c = floor(o0[a] / m.rsize);
            anchor[a] = (c > -1e9 && c < 1e9 ? (int)c : 0) - (1 << 12);
        }
    }
    __syncthreads();
    const KeyCache kc{kcache, anchor[0], anchor[1], anchor[2]};
    const bool tsdf = mode == M_TSDF;
    const bool ndt = mode == M_NDT_OM || mode == M_NDT_TM;
    const int lane = threadIdx.x & 31;
    unsigned long long st[3] = {0, 0, 0};  // processed, segments, range errors
    unsigned long long nmark_local = 0;
    // ray index in the batch (sharded maps discover the slice [ray_lo, ray_lo + n))
    long long i = m.ray_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    Ray r;
    bool ok = false;
    if (i < m.ray_lo + n) {
        src.load(i, r.o, r.e, r.has, r.inten);
        ok = prep_ray(m, r, !tsdf);
        if (ok) {
            st[0] = 1;
            st[1] = r.nseg;
            if (!in_range(m, r.o) || !in_range(m, r.e)) {
                st[2] = 1;
                ok = false;
            }
        }
        if (m.ray_order && blockIdx.y == 0) {
            // the ray's voxel steps (Manhattan cell distance of the clipped
            // ray): its bucket in the walk's longest-first order
            unsigned steps = 0;
            if (ok)
                for (int a = 0; a < 3; ++a)
                    steps += (unsigned)abs((int)floor(r.e[a] / m.vox) - (int)floor(r.o[a] / m.vox));
            const int bk = seg_bucket(steps);
            atomicAdd(shist + bk, 1u);
            m.seg_bk[i] = (unsigned char)bk;
        }
    }
    // one thread per (ray, segment): blockIdx.y is the segment index
    const int s = blockIdx.y;
    const bool mine = ok && s < r.nseg;
    if (s != 0) st[0] = st[1] = st[2] = 0;  // ray statistics are counted once
    // a later-segment block none of whose rays reach that segment (most of the
    // third, degenerate-segment row) has nothing to count, record or stamp
    if (s != 0 && !__syncthreads_or(mine)) return;
    // warp-aggregated allocation of segment descriptors
    unsigned long long dbase = 0;
    if (emit) {
        const unsigned bal = __ballot_sync(0xffffffffu, mine);
        unsigned long long base = 0;
        if (lane == 0 && bal) base = atomicAdd(m.stats + S_SEGDESC, (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        dbase = base + __popc(bal & ((1u << lane) - 1u));
    }
    PrefetchVisitor pv{&m, &kc, sset, {INT_MAX, INT_MAX, INT_MAX}, {INT_MIN, INT_MIN, INT_MIN}};
    if (mine) {
        do {
            double so[3], se[3];
            int sh;
            segment_of(m, r, s, so, se, sh);
            double pe[3] = {se[0], se[1], se[2]};
            if (tsdf && sh) {
                double L = norm3(se[0] - so[0], se[1] - so[1], se[2] - so[2]);
                if (L > 0.0) {
                    for (int a = 0; a < 3; ++a) {
                        double d = (se[a] - so[a]) / L;
                        pe[a] = se[a] + d * m.tsdf_trunc;
                    }
                    if (!in_range(m, pe)) {
                        st[2] = 1;
                        break;
                    }
                }
            }
            walk(so, pe, m.rsize, pv);
            if (emit && dbase < m.seg_cap) {
                SegDesc sd;
                int c[3];
                dda_init(so, se, m.vox, sd, c);
                sd.order = (unsigned)(i * m.maxseg + s) << 1;
                sd.flags |= sh ? 1u : 0u;
                const int rx = floordiv(c[0], m.dim), ry = floordiv(c[1], m.dim),
                          rz = floordiv(c[2], m.dim);
                bool fresh;
                sd.slot0 = cached_slot(m, kc, rx, ry, rz, &fresh);
                sd.rkey = pack_region(rx, ry, rz);
                sd.lp0 = (unsigned)(c[0] - rx * m.dim + 1) | ((unsigned)(c[1] - ry * m.dim + 1) << 10) |
                         ((unsigned)(c[2] - rz * m.dim + 1) << 20);
                sd.L = norm3(se[0] - so[0], se[1] - so[1], se[2] - so[2]);
                const uint4 *src4 = reinterpret_cast<const uint4 *>(&sd);
                atomicAdd(shist + seg_bucket(sd.rem), 1u);
                m.seg_bk[dbase] = (unsigned char)seg_bucket(sd.rem);
                uint4 *dst4 = reinterpret_cast<uint4 *>(m.segs + dbase);
#pragma unroll
                for (int q = 0; q < (int)(sizeof(SegDesc) / 16); ++q) dst4[q] = src4[q];
            }
            if (sh && (det || ndt) && !tsdf) {
                // the sample voxel floor(end / vox) (reference.py:178-186)
                int g[3];
                for (int a = 0; a < 3; ++a) g[a] = (int)floor(se[a] / m.vox);
                RegionTrack rt;
                rt.rx = floordiv(g[0], m.dim);
                rt.ry = floordiv(g[1], m.dim);
                rt.rz = floordiv(g[2], m.dim);
                rt.lx = g[0] - rt.rx * m.dim;
                rt.ly = g[1] - rt.ry * m.dim;
                rt.lz = g[2] - rt.rz * m.dim;
                bool fresh;
                rt.slot = cached_slot(m, kc, rt.rx, rt.ry, rt.rz, &fresh);
                if (rt.slot >= 0 && rt.slot < m.cap) {
                    int li = rt.li(m);
                    if (ndt) {
                        // NDT phase 2: the sample, bucketed by the voxel's index
                        // (vm_ndt.cuh); phase 1 sorts before it
                        const unsigned mi = ndt_index(m, rt.slot, li);
                        int k = atomicAdd(&nrec, 1);
                        srec[k] = ndt_key(mi, 1u, (unsigned)(i * m.maxseg + s));
                    } else if (m.key_mi) {
                        // claim the sample voxel's index; k_stamp writes MARK_FLAG | mi
                        // into its scratch word and the brick summary once the
                        // previous batch has folded (pipelined sequences run this
                        // discover concurrently with that fold)
                        claim_sample_voxel(m, rt.slot, li);
                    } else {
                        // stamp the sample voxel: the walk turns its visits into records
                        unsigned *w = layer_at<unsigned>(m, L_SCRATCH, rt.slot) + li;
                        const bool was = (*((volatile unsigned *)w) & MARK_FLAG) ||
                                         (atomicOr(w, MARK_FLAG) & MARK_FLAG);
                        if (!was) {
                            ++nmark_local;
                            if (m.marked) {
                                // the batch's sample-voxel list: published by sharded
                                // maps; its index keys the records otherwise
                                const unsigned long long mi = atomicAdd(m.nmarked, 1ULL);
                                if (mi < m.marked_cap) {
                                    m.marked[mi] = make_int2(rt.slot, li);
                                    if (m.key_mi) *w = MARK_FLAG | (unsigned)mi;
                                }
                            }
                        }
                        // brick summary read by the walks (4 x 4 x 2 bricks); set
                        // for every stamp, also one left over from a dropped batch
                        const int bsh = m.brick_shift;
                        const unsigned bit = bsh >= 0
                            ? 1u << ((rt.lx >> bsh) | ((rt.ly >> bsh) << 2) | ((rt.lz >> (bsh + 1)) << 4))
                            : 0xFFFFFFFFu;
                        if (!(__ldcg(m.bmask + rt.slot) & bit)) atomicOr(m.bmask + rt.slot, bit);
                    }
                }
            }
        } while (0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (nrec) rec_base = atomicAdd(m.stats + S_RECORDS, (unsigned long long)nrec);
    }
    if (emit || m.ray_order)
        for (int i = threadIdx.x; i < SEG_BUCKETS; i += blockDim.x)
            if (shist[i]) atomicAdd(m.seg_hist + i, shist[i]);
    __syncthreads();
    for (int k = threadIdx.x; k < nrec; k += blockDim.x) {
        unsigned long long ri = rec_base + k;
        if (ri < m.rec_cap) {
            m.rec[ri] = srec[k];
            if (m.recval) m.recval[ri] = 0u;
        }
    }
    const int which[3] = {S_PROCESSED, S_SEGMENTS, S_RANGE_ERR};
    if (count_stats) block_add_stats(m, st, which);
    {
        unsigned long long mk[1] = {nmark_local};
        const int wm[1] = {S_MARKED};
        block_add_stats(m, mk, wm);
    }
    // batch bounding box of prefetched regions (+1 margin for walk-entered ones)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int lo = pv.lo[a], hi = pv.hi[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if ((threadIdx.x & 31) == 0 && lo <= hi) {
            atomicMin(m.rbox + a, lo - 1);
            atomicMax(m.rbox + 3 + a, hi + 1);
        }
    }
}

// Dense region-slot grid over the batch bbox (walk lookups become one
// shared-memory load).  Cells of absent regions hold -1.
__global__ void k_rgrid(const __grid_constant__ DevMap m) {
    if (!read_go(m)) return;
    const int *b = m.rbox;
    const long long nx = (long long)b[3] - b[0] + 1, ny = (long long)b[4] - b[1] + 1,
                    nz = (long long)b[5] - b[2] + 1;
    if (nx <= 0 || ny <= 0 || nz <= 0 || nx * ny * nz > m.rg_max) return;
    const long long total = nx * ny * nz;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / (nx * ny));
        long long key = pack_region(b[0] + x, b[1] + y, b[2] + z);
        unsigned long long h = mix_key(key) & m.tmask;
        int slot = -1;
        for (unsigned long long p = 0; p <= m.tmask; ++p) {
            long long k = m.tkeys[h];
            if (k == key) { slot = m.tvals[h]; break; }
            if (k == -1) break;
            h = (h + 1) & m.tmask;
        }
        m.rgrid[i] = slot;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch((unsigned long long *)(m.stats + S_RGRID), 1ULL);
}

// Refuse the batch if the pool could overflow or inputs were invalid.
__global__ void k_guard(const __grid_constant__ DevMap m, int margin) {
    if (m.chain && *((volatile int *)m.chain)) {
        *m.go = 0;
        return;
    }
    int used = *((volatile int *)m.cursor);
    unsigned long long rerr = ((volatile unsigned long long *)m.stats)[S_RANGE_ERR];
    unsigned long long nseg = ((volatile unsigned long long *)m.stats)[S_SEGDESC];
    unsigned long long spilled = ((volatile unsigned long long *)m.stats)[S_SPILLED];
    bool ok = used + margin <= m.cap && rerr == 0 && nseg <= m.seg_cap && spilled == 0;
    *m.go = ok ? 1 : 0;
    if (!ok && m.chain) atomicCAS(m.chain, 0, m.batch_idx + 1);
}

// Pipelined sequences: per-batch state reset (stats slot, region box, the
// sample-voxel list unless the batch is a replay that keeps its claims).
__global__ void k_batch_init(const __grid_constant__ DevMap m, int reset_marked) {
    if (*((volatile int *)m.chain)) return;
    const int t = threadIdx.x;
    if (t < NUM_STATS) m.stats[t] = 0ULL;
    if (t < 3) m.rbox[t] = INT_MAX;
    else if (t < 6) m.rbox[t] = INT_MIN;
    if (t < 2 && reset_marked && m.nmarked) m.nmarked[t] = 0ULL;
    if (t == 0 && reset_marked && m.nlost) *m.nlost = 0ULL;
}

// Occupancy sample voxels: MARK_FLAG | mi into the scratch word, the brick
// bit into the region's summary, the claim released.  Runs after the previous
// batch's fold (which clears its own stamps) and before this batch's walk.
__global__ void __launch_bounds__(BLOCK) k_stamp(const __grid_constant__ DevMap m) {
    if (!read_go(m)) return;
    const unsigned long long M = min(*((volatile unsigned long long *)m.nmarked), m.marked_cap);
    const int bsh = m.brick_shift;
    for (unsigned long long mi = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; mi < M;
         mi += (unsigned long long)gridDim.x * blockDim.x) {
        const int2 sl = m.marked[mi];
        if (sl.x < 0 || sl.x >= m.cap) continue;
        const unsigned long long vid = (unsigned long long)sl.x * m.vpr + sl.y;
        reinterpret_cast<unsigned *>(m.slab[L_SCRATCH])[vid] = MARK_FLAG | (unsigned)mi;
        reinterpret_cast<unsigned *>(m.slab[m.nidx])[vid] = 0u;
        const unsigned bit = bsh >= 0 ? 1u << brick_of(sl.y, m.bsh) : 0xFFFFFFFFu;
        if (!(__ldcg(m.bmask + sl.x) & bit)) atomicOr(m.bmask + sl.x, bit);
    }
}

// ... and its outcome: regions after the batch and whether it ran.
// The regions after the batch, snapshot right after its walk (the next
// batch's discover may already be creating regions while this one folds).
__global__ void k_batch_regions(const __grid_constant__ DevMap m) {
    m.stats[NUM_STATS] = (unsigned long long)*((volatile int *)m.cursor);
}

__global__ void k_batch_fin(const __grid_constant__ DevMap m) {
    // sample voxels of the batch: the list's live length (also counts claims a
    // refused first attempt left for the replay)
    // (NDT: the claimed voxel indices)
    if (m.nmarked)
        m.stats[S_MARKED] = *((volatile unsigned long long *)m.nmarked) -
                            (m.key_mi ? *((volatile unsigned long long *)(m.nmarked + 1))
                                      : (m.nlost ? *((volatile unsigned long long *)m.nlost) : 0ULL));
    // bit 0: the guard let the batch run; bit 1: neither this batch nor an
    // earlier one stopped the chain (a later batch's guard, running
    // concurrently with this fold, may already have set it)
    const int c = *((volatile int *)m.chain);
    m.stats[NUM_STATS + 1] = (unsigned long long)(*((volatile int *)m.go) != 0) |
                             ((unsigned long long)(c == 0 || c > m.batch_idx + 1) << 1);
}

// Counting sort of the batch's segments by step count, longest first: the
// walk then hands every warp 32 segments of nearly equal length.  k_discover
// built the histogram; one block turns it into bucket cursors.
__global__ void k_seg_scan(const __grid_constant__ DevMap m) {
    __shared__ unsigned h[SEG_BUCKETS];
    for (int b = threadIdx.x; b < SEG_BUCKETS; b += blockDim.x) {
        h[b] = m.seg_hist[b];
        m.seg_hist[b] = 0u;  // ready for the next batch (or the replay)
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned run = 0;
    for (int b = SEG_BUCKETS - 1; b >= 0; --b) {
        m.seg_cursor[b] = run;
        run += h[b];
    }
}

// count >= 0: order `count` rays (NDT walks) instead of the batch's segments
__global__ void __launch_bounds__(BLOCK) k_seg_scatter(const __grid_constant__ DevMap m,
                                                       long long count = -1) {
    __shared__ unsigned cnt[SEG_BUCKETS], base[SEG_BUCKETS];
    if (!read_go(m)) return;
    const unsigned long long n =
        count >= 0 ? (unsigned long long)count
                   : min(*((volatile unsigned long long *)(m.stats + S_SEGDESC)), m.seg_cap);
    for (int i = threadIdx.x; i < SEG_BUCKETS; i += blockDim.x) cnt[i] = 0u;
    __syncthreads();
    const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    int b = -1;
    unsigned r = 0;
    if (idx < n) {
        b = m.seg_bk[idx];
        r = atomicAdd(cnt + b, 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SEG_BUCKETS; i += blockDim.x)
        if (cnt[i]) base[i] = atomicAdd(m.seg_cursor + i, cnt[i]);
    __syncthreads();
    if (b >= 0) m.perm[base[b] + r] = (unsigned)idx;
}

// --------------------------------------------------------------- NDT phase 1

// Deterministic NDT phase 1: a miss on a Gaussian voxel (count >= 3 at the
// start of the batch; the walk never resets in this mode) becomes a record
// (voxel | phase 0 | ray order) -> value = |fl32(g * miss_delta)| bits with
// bit 31 = (g >= miss-likelihood threshold), folded in ray order by
// k_fold_ndt together with the reset (reference.py:67-94).
// Region-sharded NDT: a ghost voxel's scratch word carries GAUSS_FLAG when
// its owner holds a Gaussian there (count >= 3 at the start of the batch);
// the low bits count the order-free misses.
constexpr unsigned GAUSS_FLAG = 0x40000000u;

// 32-byte exchange item of the sharded NDT protocol
struct ShardItemN {
    long long rkey;
    unsigned li_kind;  // li | kind << 30: 0 miss count, 1 sample (phase 2), 2 visit (phase 1)
    unsigned val;      // count, or segment order ray * maxseg + seg
    double t0, t1;     // kind 2: the visit's chord on the segment
};
static_assert(sizeof(ShardItemN) == 32, "ShardItemN layout");

__device__ __forceinline__ void shard_ghost_visit(const DevMap &m, long long key, int li,
                                                  unsigned oi, double t0, double t1) {
    const unsigned long long k = atomicAdd(m.ngx, 1ULL);
    if (k < m.gx_cap)
        reinterpret_cast<ShardItemN *>(m.gx)[k] =
            ShardItemN{key, (unsigned)li | (2u << 30), oi, t0, t1};
}

struct NdtRecStage {
    unsigned long long *key;
    double2 *t;
    int *n;
};
constexpr int NDT_STAGE = 1024;

template <bool TM, bool DET = false, bool REC_ONLY = false>
struct NdtVisitor {
    const DevMap *m;
    RegionTrack rt;
    float *occ, *cov;
    unsigned *mean, *cnt, *scr, *miss, *hitc;
    float *inten;
    int sh;
    const double *so;
    double v[3];
    int *sset;
    unsigned *cube;
    int c0, c1, c2;
    unsigned order;
    NdtRecStage st;
    unsigned long long visits, rmiss, retries;
    // region-sharded maps: the current region is another rank's (ghost);
    // `unknown`: no Gaussian bitmap of it arrived this batch
    bool ghost, unknown;
    unsigned gm;  // the region's Gaussian brick summary (all ones: unknown)

    __device__ __forceinline__ void bind() {
        int s = rt.slot;
        ghost = false;
        gm = (m->gmask && m->brick_shift >= 0 && s >= 0 && s < m->cap) ? __ldcg(m->gmask + s)
                                                                        : 0xFFFFFFFFu;
        if (DET && m->shard_world > 1 && s >= 0 && s < m->cap) {
            const long long key = m->slot_keys[s];
            ghost = region_owner(key, m->shard_world) != m->shard_rank;
            unknown = ghost && __ldcg(m->slot_pref + s) != m->epoch;
        }
        if (s >= 0 && s < m->cap) {
            occ = layer_at<float>(*m, L_OCC, s);
            cov = layer_at<float>(*m, L_COV, s);
            mean = layer_at<unsigned>(*m, L_MEAN, s);
            cnt = layer_at<unsigned>(*m, L_COUNT, s);
            scr = layer_at<unsigned>(*m, L_SCRATCH, s);
            if (TM) {
                miss = layer_at<unsigned>(*m, L_MISS, s);
                hitc = layer_at<unsigned>(*m, L_HIT, s);
                inten = layer_at<float>(*m, L_INTENS, s);
            }
            touch_region(*m, sset, s);
        } else {
            occ = nullptr;
        }
    }
    __device__ __forceinline__ void begin(int x, int y, int z) {
        rt.locate(*m, x, y, z);
        bind();
    }
    __device__ __forceinline__ void moved(int axis, int s) {
        if (rt.step(*m, axis, s)) bind();
    }
    __device__ __forceinline__ void jump(int x, int y, int z) {
        rt.locate(*m, x, y, z);
        bind();
    }
    // reference.py:67-94 / _kernels.pyx:602-648
    __device__ __forceinline__ void visit(int x, int y, int z, double t0, double t1, bool last) {
        ++visits;
        if (last && sh) return;  // sample voxel: phase 2
        if (!occ) {
            ++rmiss;
            return;
        }
        const int li = rt.li(*m);
        if (DET && ghost) {
            // another rank's voxel: a Gaussian there (its bitmap bit, or no
            // bitmap) -> the visit goes to the owner, who weighs it; else a
            // miss count (vm_shard_ndt.cuh)
            if (REC_ONLY) return;
            if (unknown || (__ldcg(scr + li) & GAUSS_FLAG))
                shard_ghost_visit(*m, m->slot_keys[rt.slot], li, order >> 1, t0, t1);
            else
                atomicAdd(scr + li, 1u);
            return;
        }
        // a brick without a Gaussian: no count to load, g == 1
        const unsigned ns = ((gm >> brick_of(li, m->bsh)) & 1u) ? __ldcg(cnt + li) : 0u;
        if (DET && ns >= 3) {
            // a miss through a Gaussian: a phase-1 record with its chord; the
            // weight is computed after the walk, for all records at once
            // (k_ndt_weigh), so no lane of the walk stalls the others on it
            const unsigned long long key = ndt_key(ndt_index(*m, rt.slot, li), 0u, order >> 1);
            const int k = atomicAdd(st.n, 1);
            if (k < NDT_STAGE) {
                st.key[k] = key;
                st.t[k] = make_double2(t0, t1);
            } else {
                const unsigned long long g = atomicAdd(m->stats + S_RECORDS, 1ULL);
                if (g < m->rec_cap) {
                    m->rec[g] = key;
                    m->rec_t[g] = make_double2(t0, t1);
                }
            }
            return;
        }
        if (ns < 3) {
            if (REC_ONLY) return;
            // g == 1: identical deltas, order-free -> counted, resolved exactly
            unsigned ux = (unsigned)(x - c0), uy = (unsigned)(y - c1), uz = (unsigned)(z - c2);
            if ((ux | uy | uz) < (unsigned)CUBE)
                atomicAdd(cube + ux + CUBE * (uy + CUBE * uz), 1u);
            else
                atomicAdd(scr + li, 1u);
            return;
        }
        unsigned packed = __ldcg(mean + li);
        float c6[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) c6[j] = __ldcg(cov + li * 6 + j);
        double off[3], mu[3];
        unpack_mean(packed, off);
        mu[0] = ((double)x + off[0]) * m->vox;
        mu[1] = ((double)y + off[1]) * m->vox;
        mu[2] = ((double)z + off[2]) * m->vox;
        double gw = gaussian_weight(mu, c6, m->sigma2, so, v, t0, t1);
        float d32 = (float)(gw * m->miss_delta);
        {
            float *p = occ + li;
            unsigned old = __float_as_uint(__ldcg(p));
            for (;;) {
                unsigned nb = __float_as_uint(clamp_add(__uint_as_float(old), d32, m->cmin,
                                                        m->cmax));
                if (nb == old) break;
                unsigned prev = atomicCAS(reinterpret_cast<unsigned *>(p), old, nb);
                if (prev == old) break;
                old = prev;
                ++retries;
            }
        }
        if (TM && gw >= m->miss_check) atomicAdd(miss + li, 1u);
        float lnow = __ldcg(occ + li);
        if (lnow < m->fthresh && __ldcg(cnt + li) > 0) {
            atomicExch(cnt + li, 0u);
            atomicExch(mean + li, 0u);
#pragma unroll
            for (int j = 0; j < 6; ++j) atomicExch(reinterpret_cast<unsigned *>(cov) + li * 6 + j, 0u);
            if (TM) {
                atomicExch(hitc + li, 0u);
                atomicExch(miss + li, 0u);
                atomicExch(reinterpret_cast<unsigned *>(inten) + li * 2, 0u);
                atomicExch(reinterpret_cast<unsigned *>(inten) + li * 2 + 1, 0u);
            }
        }
    }
};

#ifndef NDT_MINB
#define NDT_MINB 2  // k_walk_ndt: 2 blocks per SM (128 registers; 151 / 1 block: C3 walk 18.3 -> 17.1 ms)
#endif

template <bool TM, bool DET, bool REC_ONLY, class Src>
__global__ void __launch_bounds__(BLOCK, NDT_MINB) k_walk_ndt(const __grid_constant__ DevMap m, Src src, long long n) {
    __shared__ unsigned cube[CUBE_N];
    __shared__ int sset[SLOTSET];
    __shared__ int corner[3];
    __shared__ unsigned long long skey[DET ? NDT_STAGE : 1];
    __shared__ double2 st_t[DET ? NDT_STAGE : 1];
    __shared__ int nrec;
    __shared__ unsigned long long rec_base;
    if (!read_go(m)) return;
    if (DET && !REC_ONLY && m.walk_det_launched && walk_det_ok(m)) return;  // k_walk_ndt_det walked it
    for (int k = threadIdx.x; k < CUBE_N; k += blockDim.x) cube[k] = 0;
    for (int k = threadIdx.x; k < SLOTSET; k += blockDim.x) sset[k] = -1;
    long long first = (long long)blockIdx.x * blockDim.x;
    if (threadIdx.x == 0) {
        double o[3], e[3];
        int h;
        float it;
        src.load(m.ray_lo + (first < n ? first : 0), o, e, h, it);
        for (int a = 0; a < 3; ++a) corner[a] = (int)floor(o[a] / m.vox) - CUBE / 2;
        nrec = 0;
    }
    __syncthreads();
    NdtVisitor<TM, DET, REC_ONLY> v;
    v.m = &m;
    v.sset = sset;
    v.cube = cube;
    v.c0 = corner[0];
    v.c1 = corner[1];
    v.c2 = corner[2];
    v.st = NdtRecStage{skey, st_t, &nrec};
    v.visits = v.rmiss = v.retries = 0;
    long long i = first + threadIdx.x;
    if (i < n) {
        if (m.ray_order) i = m.perm[i];  // longest rays first: a warp's lanes finish together
        i += m.ray_lo;                   // sharded maps walk the slice [ray_lo, ray_lo + n)
        Ray r;
        src.load(i, r.o, r.e, r.has, r.inten);
        if (prep_ray(m, r, true)) {
            for (int s = 0; s < r.nseg; ++s) {
                double so[3], se[3];
                segment_of(m, r, s, so, se, v.sh);
                v.so = so;
                v.order = (unsigned)(i * m.maxseg + s) << 1;
                for (int a = 0; a < 3; ++a) v.v[a] = se[a] - so[a];
                walk(so, se, m.vox, v);
            }
        }
    }
    __syncthreads();
    if (DET) {
        const int nl = nrec < NDT_STAGE ? nrec : NDT_STAGE;
        if (threadIdx.x == 0 && nl) rec_base = atomicAdd(m.stats + S_RECORDS, (unsigned long long)nl);
        __syncthreads();
        for (int k = threadIdx.x; k < nl; k += blockDim.x) {
            const unsigned long long ri = rec_base + k;
            if (ri < m.rec_cap) {
                m.rec[ri] = skey[k];
                m.rec_t[ri] = st_t[k];
            }
        }
    }
    if (REC_ONLY) return;
    unsigned long long flushed = 0;
    for (int k = threadIdx.x; k < CUBE_N; k += blockDim.x) {
        unsigned cnt = cube[k];
        if (!cnt) continue;
        ++flushed;
        int g[3] = {v.c0 + k % CUBE, v.c1 + (k / CUBE) % CUBE, v.c2 + k / (CUBE * CUBE)};
        RegionTrack rt;
        rt.locate(m, g[0], g[1], g[2]);
        touch_region(m, sset, rt.slot);
        atomicAdd(layer_at<unsigned>(m, L_SCRATCH, rt.slot) + rt.li(m), cnt);
    }
    unsigned long long st[4] = {v.visits, v.rmiss, v.retries, flushed};
    const int which[4] = {S_VISITS, S_RMISS, S_RETRIES, S_CUBE_FLUSH};
    block_add_stats(m, st, which);
}

// --------------------------------------------------------------- TSDF

template <bool DET>
struct TsdfVisitor {
    const DevMap *m;
    RegionTrack rt;
    float *buf;
    double o[3], d[3], L;
    unsigned ray;
    Stage<unsigned long long, REC_STAGE> *stage;
    unsigned long long visits, rmiss, retries;
    __device__ __forceinline__ void bind() {
        int s = rt.slot;
        buf = (s >= 0 && s < m->cap) ? layer_at<float>(*m, L_TSDF, s) : nullptr;
    }
    __device__ __forceinline__ void begin(int x, int y, int z) {
        rt.locate(*m, x, y, z);
        bind();
    }
    __device__ __forceinline__ void moved(int axis, int s) {
        if (rt.step(*m, axis, s)) bind();
    }
    __device__ __forceinline__ void jump(int x, int y, int z) {
        rt.locate(*m, x, y, z);
        bind();
    }
    __device__ __forceinline__ void visit(int x, int y, int z, double, double, bool) {
        ++visits;
        if (!buf) {
            ++rmiss;
            return;
        }
        const int li = rt.li(*m);
        if (DET) {
            // bucketed by the voxel's claimed index (vm_ndt.cuh), ray order
            stage->push(ndt_key(ndt_index(*m, rt.slot, li), 0u, ray), m->rec, m->stats + S_RECORDS,
                        m->rec_cap);
            return;
        }
        // reference.py:167-174
        double c[3] = {((double)x + 0.5) * m->vox - o[0], ((double)y + 0.5) * m->vox - o[1],
                       ((double)z + 0.5) * m->vox - o[2]};
        double dv = L - dot3(c, d);
        if (dv < -m->tsdf_trunc) dv = -m->tsdf_trunc;
        if (dv > m->tsdf_trunc) dv = m->tsdf_trunc;
        unsigned long long *p = reinterpret_cast<unsigned long long *>(buf + 2 * li);
        unsigned long long old = __ldcg(p);
        for (;;) {
            float fd = __uint_as_float((unsigned)(old & 0xffffffffu));
            float fw = __uint_as_float((unsigned)(old >> 32));
            double w = fw;
            float nd = (float)((w * (double)fd + dv) / (w + 1.0));
            double nwd = w + 1.0;
            if (nwd > m->tsdf_maxw) nwd = m->tsdf_maxw;
            float nw = (float)nwd;
            unsigned long long nb = ((unsigned long long)__float_as_uint(nw) << 32) |
                                    __float_as_uint(nd);
            unsigned long long prev = atomicCAS(p, old, nb);
            if (prev == old) break;
            old = prev;
            ++retries;
        }
    }
};

// band geometry of integrate_tsdf_ray (reference.py:153-165)
__device__ __forceinline__ bool tsdf_band(const DevMap &m, const Ray &r, double d[3],
                                          double p0[3], double p1[3]) {
    if (!r.has || r.L == 0.0) return false;
    for (int a = 0; a < 3; ++a) d[a] = (r.e[a] - r.o[a]) / r.L;
    double ts = r.L - m.tsdf_trunc;
    if (!(ts > 0.0)) ts = 0.0;
    double te = r.L + m.tsdf_trunc;
    for (int a = 0; a < 3; ++a) {
        p0[a] = r.o[a] + d[a] * ts;
        p1[a] = r.o[a] + d[a] * te;
    }
    return true;
}

template <bool DET, class Src>
__global__ void __launch_bounds__(BLOCK) k_walk_tsdf(const __grid_constant__ DevMap m, Src src, long long n) {
    __shared__ unsigned long long srec[REC_STAGE];
    __shared__ int nrec;
    __shared__ unsigned long long rec_base;
    if (!read_go(m)) return;
    if (threadIdx.x == 0) nrec = 0;
    __syncthreads();
    Stage<unsigned long long, REC_STAGE> stage{srec, &nrec};
    TsdfVisitor<DET> v;
    v.m = &m;
    v.stage = &stage;
    v.visits = v.rmiss = v.retries = 0;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        Ray r;
        src.load(i, r.o, r.e, r.has, r.inten);
        double p0[3], p1[3];
        if (prep_ray(m, r, false) && tsdf_band(m, r, v.d, p0, p1)) {
            for (int a = 0; a < 3; ++a) v.o[a] = r.o[a];
            v.L = r.L;
            v.ray = (unsigned)i;
            walk(p0, p1, m.vox, v);
        }
    }
    if (DET) {
        __syncthreads();
        int nl = nrec < REC_STAGE ? nrec : REC_STAGE;
        if (threadIdx.x == 0 && nl) rec_base = atomicAdd(m.stats + S_RECORDS, (unsigned long long)nl);
        __syncthreads();
        for (int k = threadIdx.x; k < nl; k += blockDim.x) {
            unsigned long long ri = rec_base + k;
            if (ri < m.rec_cap) m.rec[ri] = srec[k];
        }
    }
    unsigned long long st[3] = {v.visits, v.rmiss, v.retries};
    const int which[3] = {S_VISITS, S_RMISS, S_RETRIES};
    block_add_stats(m, st, which);
}

// --------------------------------------------------------------- resolve

// f_miss^k for every voxel that received k order-free misses this batch;
// NDT adds the NDT-TM miss count and the transient reset
// (reference.py:86-93).  One block per touched region.
// Resolve region `slot`, voxels [v0, v1): f_miss^k per counted voxel.
#ifndef RES_U
#define RES_U 2     // scratch quads in flight per thread
#endif
#ifndef RES_PIPE
#define RES_PIPE 0  // software-pipelined scratch loads (experiment knob)
#endif
#ifndef RES_MINB
#define RES_MINB 8  // k_resolve resident blocks per SM: 8 x 2 quads in flight beat
                    // 4 x 4 and 2 x 8 (C2 resolve 10.0 / 10.5 / 11.6 ms per step)
#endif

template <bool NDT, bool TM>
__device__ __forceinline__ void resolve_range(const DevMap &m, int slot, int v0, int v1) {
    unsigned *scr = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH] + (size_t)slot * m.bpr[L_SCRATCH]);
    float *occ = reinterpret_cast<float *>(m.slab[L_OCC] + (size_t)slot * m.bpr[L_OCC]);
    if (!NDT && ((v0 | v1) & 3) == 0) {
        // 8 independent 16-byte scratch loads in flight per thread, then the
        // occupancy quads of the non-zero ones, also all in flight
        const uint4 *s4 = reinterpret_cast<const uint4 *>(scr);
        float4 *o4 = reinterpret_cast<float4 *>(occ);
#if RES_PIPE
        // the next chunk's scratch loads are issued before this chunk's
        // occupancy round trip (two dependent loads per chunk otherwise)
        uint4 wn[RES_U];
#pragma unroll
        for (int u = 0; u < RES_U; ++u) {
            const int q = (v0 >> 2) + threadIdx.x + u * blockDim.x;
            wn[u] = q < (v1 >> 2) ? __ldcs(s4 + q) : make_uint4(0, 0, 0, 0);
        }
#endif
        for (int q0 = (v0 >> 2) + threadIdx.x; q0 < (v1 >> 2); q0 += RES_U * blockDim.x) {
            uint4 w[RES_U];
            float4 l[RES_U];
            unsigned nz = 0;
#if RES_PIPE
#pragma unroll
            for (int u = 0; u < RES_U; ++u) {
                w[u] = wn[u];
                const int q = q0 + RES_U * blockDim.x + u * blockDim.x;
                wn[u] = q < (v1 >> 2) ? __ldcs(s4 + q) : make_uint4(0, 0, 0, 0);
            }
#else
#pragma unroll
            for (int u = 0; u < RES_U; ++u) {
                const int q = q0 + u * blockDim.x;
                w[u] = q < (v1 >> 2) ? __ldcs(s4 + q) : make_uint4(0, 0, 0, 0);
            }
#endif
#pragma unroll
            for (int u = 0; u < RES_U; ++u) {
                // counted voxels (MARK'ed words -- sample voxels -- are the fold's)
                const unsigned ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
                bool any = false;
#pragma unroll
                for (int j = 0; j < 4; ++j) any = any || (ws[j] != 0u && !(ws[j] & MARK_FLAG));
                if (any) {
                    nz |= 1u << u;
                    l[u] = o4[q0 + u * blockDim.x];
                }
            }
#pragma unroll
            for (int u = 0; u < RES_U; ++u) {
                if (!((nz >> u) & 1u)) continue;
                const int q = q0 + u * blockDim.x;
                unsigned ks[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
                float ls[4] = {l[u].x, l[u].y, l[u].z, l[u].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (ks[j] == 0 || (ks[j] & MARK_FLAG)) continue;
                    ls[j] = miss_k(ls[j], ks[j], m.miss32, m.cmin, m.cmax);
                    ks[j] = 0;
                }
                o4[q] = make_float4(ls[0], ls[1], ls[2], ls[3]);
                reinterpret_cast<uint4 *>(scr)[q] = make_uint4(ks[0], ks[1], ks[2], ks[3]);
            }
        }
        return;
    }
    for (int li = v0 + threadIdx.x; li < v1; li += blockDim.x) {
        const unsigned k = scr[li];
        if (k == 0 || (k & MARK_FLAG)) continue;
        scr[li] = 0;
        float l = occ[li];
        if (!NDT) {
            occ[li] = miss_k(l, k, m.miss32, m.cmin, m.cmax);
            continue;
        }
        // NDT phase 1, g == 1 (reference.py:86-93): each miss is followed by
        // the TM miss count and the transient reset check; with identical
        // deltas the reset fires at the first miss j with l < threshold.
        unsigned *cnt = layer_at<unsigned>(m, L_COUNT, slot);
        unsigned j = 0;
        if (cnt[li] > 0) {
            for (unsigned i = 1; i <= k; ++i) {
                const float nl = clamp_add(l, m.miss32, m.cmin, m.cmax);
                const bool same = __float_as_uint(nl) == __float_as_uint(l);
                l = nl;
                if (l < m.fthresh) {
                    j = i;
                    break;
                }
                if (same) break;  // fixed point above the threshold: never resets
            }
        }
        if (j) {
            l = miss_k(l, k - j, m.miss32, m.cmin, m.cmax);
            cnt[li] = 0;
            layer_at<unsigned>(m, L_MEAN, slot)[li] = 0;
            float *cov = layer_at<float>(m, L_COV, slot);
            for (int q = 0; q < 6; ++q) cov[li * 6 + q] = 0.0f;
            if (TM) {
                layer_at<unsigned>(m, L_HIT, slot)[li] = 0;
                layer_at<unsigned>(m, L_MISS, slot)[li] = k - j;
                float *it = layer_at<float>(m, L_INTENS, slot);
                it[li * 2] = 0.0f;
                it[li * 2 + 1] = 0.0f;
            }
        } else {
            l = miss_k(occ[li], k, m.miss32, m.cmin, m.cmax);
            if (TM) layer_at<unsigned>(m, L_MISS, slot)[li] += k;
        }
        occ[li] = l;
    }
}

// Resolve the order-free miss counts of every region the walk touched:
// the dense-grid regions plus touched-list regions outside the grid.
// Work item = (region, tile of RES_TILE voxels).
constexpr int RES_TILE = 8192;

template <bool NDT, bool TM>
__global__ void __launch_bounds__(BLOCK, RES_MINB) k_resolve(const __grid_constant__ DevMap m) {
    if (!read_go(m)) return;
    unsigned long long nt = *((volatile unsigned long long *)(m.stats + S_WALK_TOUCHED));
    if (nt > (unsigned long long)m.touched_cap) nt = m.touched_cap;
    const bool grid = *((volatile unsigned long long *)(m.stats + S_RGRID)) != 0;
    const int *b = m.rbox;
    const long long gx = grid ? b[3] - b[0] + 1 : 0, gy = grid ? b[4] - b[1] + 1 : 0,
                    gz = grid ? b[5] - b[2] + 1 : 0;
    const unsigned long long ncell = (unsigned long long)(gx * gy * gz);
    const int tiles = (m.vpr + RES_TILE - 1) / RES_TILE;
    for (unsigned long long w = blockIdx.x; w < (ncell + nt) * tiles; w += gridDim.x) {
        const unsigned long long t = w / tiles;
        const int tile = (int)(w % tiles);
        int slot;
        if (t < ncell) {
            slot = m.rgrid[t];
            if (slot < 0 || slot >= m.cap) continue;
        } else {
            slot = m.touched[t - ncell];
            if (grid) {
                int r[3];
                unpack_region(m.slot_keys[slot], r);
                const long long ux = r[0] - b[0], uy = r[1] - b[1], uz = r[2] - b[2];
                if (ux >= 0 && ux < gx && uy >= 0 && uy < gy && uz >= 0 && uz < gz &&
                    m.rgrid[ux + gx * (uy + gy * uz)] == slot)
                    continue;  // covered by its grid cell
            }
        }
        const int v0 = tile * RES_TILE;
        const int v1 = min(m.vpr, v0 + RES_TILE);
        resolve_range<NDT, TM>(m, slot, v0, v1);
    }
}

// --------------------------------------------------------------- folds

__device__ __forceinline__ long long lower_bound_u64(const unsigned long long *a, long long n,
                                                     unsigned long long key) {
    long long lo = 0, hi = n;
    while (lo < hi) {
        long long mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// voxel id of an occupancy record's key field (sample-voxel index or voxel id)
__device__ __forceinline__ unsigned record_vid(const DevMap &m, unsigned long long vk) {
    if (!m.key_mi) return (unsigned)vk;
    const int2 sl = m.marked[vk];
    return (unsigned)sl.x * (unsigned)m.vpr + (unsigned)sl.y;
}

// Apply one sample voxel's records [s, e) in ray order (reference.py:35-64
// restricted to that voxel): misses between hits collapse to f_miss^k.
// Clears the voxel's MARK'ed scratch word.
template <class Src>
__device__ __forceinline__ void fold_voxel_serial(const DevMap &m, const Src &src,
                                                  const unsigned long long *keys, long long s,
                                                  long long e, unsigned vid) {
    const unsigned long long omask = (1ULL << m.order_bits) - 1;
    float *occ = reinterpret_cast<float *>(m.slab[L_OCC]) + vid;
    unsigned *mean = m.slab[L_MEAN] ? reinterpret_cast<unsigned *>(m.slab[L_MEAN]) + vid : nullptr;
    unsigned *cnt = m.slab[L_COUNT] ? reinterpret_cast<unsigned *>(m.slab[L_COUNT]) + vid : nullptr;
    float l = *occ;
    unsigned packed = mean ? *mean : 0u, count = cnt ? *cnt : 0u;
    int g[3];
    slot_li_to_g(m, (int)(vid / (unsigned)m.vpr), (int)(vid % (unsigned)m.vpr), g);
    unsigned misses = 0;
    for (long long i = s; i < e; ++i) {
        const unsigned long long k = keys[i];
        if (!(k & 1ULL)) {
            ++misses;
            continue;
        }
        l = miss_k(l, misses, m.miss32, m.cmin, m.cmax);
        misses = 0;
        l = clamp_add(l, m.hit32, m.cmin, m.cmax);
        if (mean) {
            const long long ray = (long long)(((k & omask) >> 1) / (unsigned long long)m.maxseg);
            double ep[3];
            float it;
            src.load_end(ray, ep, it);
            const double off[3] = {ep[0] / m.vox - (double)g[0], ep[1] / m.vox - (double)g[1],
                                   ep[2] / m.vox - (double)g[2]};
            fold_mean(packed, count, off);
        }
    }
    l = miss_k(l, misses, m.miss32, m.cmin, m.cmax);
    *occ = l;
    if (mean) {
        *mean = packed;
        *cnt = count;
    }
    reinterpret_cast<unsigned *>(m.slab[L_SCRATCH])[vid] = 0u;
    m.bmask[vid / (unsigned)m.vpr] = 0u;
}

constexpr int FOLD_SERIAL_MAX = 64;

// One thread per record-run head (= sample voxel); runs longer than
// FOLD_SERIAL_MAX are handed to k_fold_occ_big (one warp each).
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_fold_occ(const __grid_constant__ DevMap m, Src src,
                                                    const unsigned long long *keys, long long R,
                                                    long long *big, unsigned long long *nbig) {
    if (!read_go(m)) return;
    const int ob = m.order_bits;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long vk = keys[i] >> ob;
        if (i > 0 && (keys[i - 1] >> ob) == vk) continue;
        if (vk == m.rec_invalid) continue;  // records a sharded map handed to their owner
        long long e = i + 1;
        while (e < R && e - i <= FOLD_SERIAL_MAX && (keys[e] >> ob) == vk) ++e;
        if (e < R && (keys[e] >> ob) == vk) {
            big[atomicAdd(nbig, 1ULL)] = i;
            continue;
        }
        fold_voxel_serial(m, src, keys, i, e, record_vid(m, vk));
    }
}

// Long runs: one warp scans 32 records at a time; misses between hits are
// counted with ballots and applied as f_miss^k.
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_fold_occ_big(const __grid_constant__ DevMap m, Src src,
                                                        const unsigned long long *keys, long long R,
                                                        const long long *big,
                                                        const unsigned long long *nbig) {
    if (!read_go(m)) return;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x / 32);
    const unsigned long long omask = (1ULL << m.order_bits) - 1;
    const int ob = m.order_bits;
    const long long nb = (long long)*nbig;
    for (long long w = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < nb;
         w += warps) {
        const long long s = big[w];
        const unsigned long long vk = keys[s] >> ob;
        const unsigned vid = record_vid(m, vk);
        float *occ = reinterpret_cast<float *>(m.slab[L_OCC]) + vid;
        unsigned *mean = m.slab[L_MEAN] ? reinterpret_cast<unsigned *>(m.slab[L_MEAN]) + vid : nullptr;
        unsigned *cnt = m.slab[L_COUNT] ? reinterpret_cast<unsigned *>(m.slab[L_COUNT]) + vid : nullptr;
        float l = *occ;
        unsigned packed = mean ? *mean : 0u, count = cnt ? *cnt : 0u;
        int g[3];
        slot_li_to_g(m, (int)(vid / (unsigned)m.vpr), (int)(vid % (unsigned)m.vpr), g);
        for (long long pos = s;; pos += 32) {
            const long long p = pos + lane;
            const unsigned long long key = p < R ? keys[p] : ~0ULL;
            const bool mine = p < R && (key >> ob) == vk;
            const unsigned vmask = __ballot_sync(0xffffffffu, mine);
            const unsigned hmask = __ballot_sync(0xffffffffu, mine && (key & 1ULL));
            const int nvalid = __popc(vmask);  // run records are a prefix of the window
            int cur = 0;
            while (cur < nvalid) {
                const unsigned rem = (hmask >> cur) & (nvalid - cur >= 32 ? 0xffffffffu
                                                                          : ((1u << (nvalid - cur)) - 1u));
                if (!rem) {
                    l = miss_k(l, (unsigned)(nvalid - cur), m.miss32, m.cmin, m.cmax);
                    break;
                }
                const int nh = cur + __ffs(rem) - 1;
                l = miss_k(l, (unsigned)(nh - cur), m.miss32, m.cmin, m.cmax);
                const unsigned long long hk = __shfl_sync(0xffffffffu, key, nh);
                l = clamp_add(l, m.hit32, m.cmin, m.cmax);
                if (mean) {
                    const long long ray = (long long)(((hk & omask) >> 1) / (unsigned long long)m.maxseg);
                    double ep[3];
                    float it;
                    src.load_end(ray, ep, it);
                    const double off[3] = {ep[0] / m.vox - (double)g[0], ep[1] / m.vox - (double)g[1],
                                           ep[2] / m.vox - (double)g[2]};
                    fold_mean(packed, count, off);
                }
                cur = nh + 1;
            }
            if (nvalid < 32) break;
        }
        if (lane == 0) {
            *occ = l;
            if (mean) {
                *mean = packed;
                *cnt = count;
            }
            reinterpret_cast<unsigned *>(m.slab[L_SCRATCH])[vid] = 0u;
            m.bmask[vid / (unsigned)m.vpr] = 0u;
        }
    }
}

// Deterministic TSDF: one thread per voxel merges its band visits in ray
// order (reference.py:153-175).
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_fold_tsdf(const __grid_constant__ DevMap m, Src src,
                                                     const unsigned long long *keys, long long R) {
    if (!read_go(m)) return;
    const unsigned long long omask = (1ULL << m.order_bits) - 1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long vid = keys[i] >> m.order_bits;
        if (i > 0 && (keys[i - 1] >> m.order_bits) == vid) continue;
        int slot = (int)(vid / (unsigned long long)m.vpr), li = (int)(vid % (unsigned long long)m.vpr);
        int g[3];
        slot_li_to_g(m, slot, li, g);
        float *buf = layer_at<float>(m, L_TSDF, slot);
        float fd = buf[2 * li], fw = buf[2 * li + 1];
        for (long long j = i; j < R && (keys[j] >> m.order_bits) == vid; ++j) {
            long long ray = (long long)(keys[j] & omask);
            Ray r;
            src.load(ray, r.o, r.e, r.has, r.inten);
            prep_ray(m, r, false);
            double d[3];
            for (int a = 0; a < 3; ++a) d[a] = (r.e[a] - r.o[a]) / r.L;
            double c[3] = {((double)g[0] + 0.5) * m.vox - r.o[0],
                           ((double)g[1] + 0.5) * m.vox - r.o[1],
                           ((double)g[2] + 0.5) * m.vox - r.o[2]};
            double dv = r.L - dot3(c, d);
            if (dv < -m.tsdf_trunc) dv = -m.tsdf_trunc;
            if (dv > m.tsdf_trunc) dv = m.tsdf_trunc;
            double w = fw;
            fd = (float)((w * (double)fd + dv) / (w + 1.0));
            double nw = w + 1.0;
            if (nw > m.tsdf_maxw) nw = m.tsdf_maxw;
            fw = (float)nw;
        }
        buf[2 * li] = fd;
        buf[2 * li + 1] = fw;
    }
}

// Error path: a refused batch leaves its sample-voxel stamps behind; clear
// every MARK'ed scratch word of the first nreg regions (no walk ran, so
// MARK'ed words hold nothing else).
__global__ void k_clear_marks(const __grid_constant__ DevMap m, long long words) {
    unsigned *scr = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < words;
         k += (long long)gridDim.x * blockDim.x) {
        if (scr[k] & MARK_FLAG) scr[k] = 0u;
        if (k % m.vpr == 0) m.bmask[k / m.vpr] = 0u;
    }
}

// --------------------------------------------------------------- single walk

struct CollectVisitor {
    long long *coords;
    double *t0, *t1;
    long long cap, n;
    __device__ __forceinline__ void begin(int, int, int) {}
    __device__ __forceinline__ void moved(int, int) {}
    __device__ __forceinline__ void jump(int, int, int) {}
    __device__ __forceinline__ void visit(int x, int y, int z, double a, double b, bool) {
        if (n < cap) {
            coords[3 * n] = x;
            coords[3 * n + 1] = y;
            coords[3 * n + 2] = z;
            t0[n] = a;
            t1[n] = b;
        }
        ++n;
    }
};

__global__ void k_walk_one(double ox, double oy, double oz, double ex, double ey, double ez,
                           double cell, long long *coords, double *t0, double *t1, long long cap,
                           long long *n_out) {
    double o[3] = {ox, oy, oz}, e[3] = {ex, ey, ez};
    CollectVisitor v{coords, t0, t1, cap, 0};
    walk(o, e, cell, v);
    *n_out = v.n;
}

}  // namespace vm
