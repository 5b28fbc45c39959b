// vm_walk.cuh -- the persistent occupancy/decay walk (the hot kernel).
//
// One warp = 32 independent walkers over the batch's preprocessed segments
// (SegDesc, written by k_discover with the exact fp64 DDA initial state).
// Every step each active lane takes exactly one DDA step of its segment
// (traversal.py:80-111) = one voxel visit.
//
// Lean per-step state: the three t_max / t_delta doubles, the voxel's
// local index `li` inside its region plus the region's voxel base
// (slot * region_dim^3), the biased packed local coordinates (region-face
// detection on the stepped axis only) and the packed region key (a region
// crossing adds +-1 to one 21-bit field, keys.py:76-86).  A crossing looks
// the new region up in the batch's dense region grid (shared memory), the
// hash table only outside it.  The axis choice and the t_max update are
// three fp64 compares and three predicated fp64 adds (no selects).
//
// Deterministic mode: every visit is ONE atomic add with return on the
// voxel's scratch counter (order-free miss count, resolved as f_miss^k by
// k_resolve).  k_discover stamped MARK_FLAG into the scratch word of every
// sample voxel, so the returned old value says whether the visit must
// instead become an order-keyed record (voxel id, ray order, hit) for the
// in-order fold.  The returned values are only inspected every WK_INNER
// steps, all together (one memory latency per WK_INNER steps instead of one
// per step); the candidate record keys wait in shared memory meanwhile.
// Visits around the sensor land in a small shared-memory cube first (the
// sensor voxel is visited by every ray of the batch); the cube carries its
// own sample-voxel bitmap.
//
// CAS mode: the paper's clamped compare-and-swap update (_kernels.pyx:233-
// 271); the load is issued one step ahead of the CAS.
//
// Work: segments are walked longest first (k_seg_scan / k_seg_scatter
// counting-sort them by step count), 32 per warp claim, so the lanes of a
// warp run segments of nearly equal length and the batch ends on short
// ones.  Lanes whose segment ends swap in the descriptor they prefetched
// into their own smem slot (cp.async).
#pragma once

#include <cuda_pipeline.h>

#include "vm_kernels.cuh"

namespace vm {

constexpr int WK_INNER = 8;     // DDA steps between warp-level bookkeeping (= max candidates)
constexpr int WK_BLOCKS = 3;    // resident blocks per SM
// dense region grid cells held in shared memory (larger boxes read the grid
// through L1): sized so three blocks of each walk fit an SM next to the 16^3
// sensor cube.  k_walk_det with 2048 cells (73 KB per block) measured 4%
// slower on C2 than with 1024 (65 KB); 64..1024 are equal.
constexpr int RG_SMEM = 1024;      // k_walk (generic / CAS)
#ifndef VM_RG_SMEM_DET
#define VM_RG_SMEM_DET 1024
#endif
constexpr int RG_SMEM_DET = VM_RG_SMEM_DET;  // k_walk_det
constexpr int WK_WBUF = 64;     // per-warp record ring (flushed 32 at a time)
// Sensor cube: the voxels next to the sensor, which every ray of the batch
// crosses, count in shared memory instead of as same-address L2 atomics.
// 16^3 instead of 8^3: C2 walk 63.7 -> 61.0 ms per step.
#ifndef VM_WCB
#define VM_WCB 4
#endif
constexpr int WCB = VM_WCB;           // log2 of the sensor cube edge
constexpr int WCUBE = 1 << WCB;       // sensor cube edge (voxels)
constexpr int WCUBE_N = WCUBE * WCUBE * WCUBE;
// cube coordinates packed one per byte in cp: cube cell index, and the
// bits that are set once a coordinate leaves [0, WCUBE)
__device__ __forceinline__ unsigned cube_cell(unsigned cp) {
    return (cp & (WCUBE - 1u)) | ((cp >> (8 - WCB)) & ((WCUBE - 1u) << WCB)) |
           ((cp >> (16 - 2 * WCB)) & ((WCUBE - 1u) << (2 * WCB)));
}
constexpr unsigned CUBE_OUT = (0xFFu & ~(WCUBE - 1u)) * 0x010101u;

struct WalkSmem {
    unsigned cube[WCUBE_N];                  // miss counts around the sensor
    unsigned cmark[WCUBE_N / 32];            // sample-voxel bitmap of the cube
    int2 grid[RG_SMEM];                      // (slot, brick mask of sample voxels)
    unsigned long long wbuf[BLOCK / 32][WK_WBUF];
    unsigned long long cand[WK_INNER][BLOCK];  // candidate visits (record keys) per lane
    SegDesc pf[BLOCK];
    int endc[BLOCK][3];    // end cell of the lane's current segment
    int gb[3], gn[3];      // dense region grid origin / extents; gn[0] = 0: no grid
    int anchor[3];         // cube corner (voxels)
    int gsmem;             // grid held in smem
};

// Region slot of region key (dense grid first, hash table otherwise) and
// its brick summary of sample voxels (bit b: brick b holds a sample voxel).
__device__ __forceinline__ int walk_region(const DevMap &m, const WalkSmem &sm, long long key,
                                           unsigned &bm, bool insert = true) {
    int r[3];
    unpack_region(key, r);
    const unsigned ux = (unsigned)(r[0] - sm.gb[0]), uy = (unsigned)(r[1] - sm.gb[1]),
                   uz = (unsigned)(r[2] - sm.gb[2]);
    if (ux < (unsigned)sm.gn[0] && uy < (unsigned)sm.gn[1] && uz < (unsigned)sm.gn[2]) {
        const int gi = ux + sm.gn[0] * (uy + sm.gn[1] * uz);
        if (sm.gsmem) {
            const int2 e = sm.grid[gi];
            if (e.x >= 0) {
                bm = (unsigned)e.y;
                return e.x;
            }
        } else {
            const int s = __ldg(m.rgrid + gi);
            if (s >= 0 && s < m.cap) {
                bm = __ldcg(m.bmask + s);
                return s;
            }
        }
    }
    const int slot = insert ? region_slot(m, key) : region_find(m, key);
    bm = 0xFFFFFFFFu;
    if (slot >= 0 && slot < m.cap) {
        bm = __ldcg(m.bmask + slot);
        if (stamp_epoch(m.slot_touch + slot, m.epoch)) {
            // regions reached outside the dense grid are resolved from the touched list
            const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
            if (t < (unsigned long long)m.touched_cap) m.touched[t] = slot;
        }
    }
    return slot;
}

// global voxel offset (slot * vpr + li) of global cell g; 0xFFFFFFFF if absent
__device__ __forceinline__ unsigned walk_vid(const DevMap &m, const WalkSmem &sm, int gx, int gy,
                                             int gz, bool insert = true) {
    const int rx = floordiv(gx, m.dim), ry = floordiv(gy, m.dim), rz = floordiv(gz, m.dim);
    unsigned bm;
    const int s = walk_region(m, sm, pack_region(rx, ry, rz), bm, insert);
    if (s < 0 || s >= m.cap) return 0xFFFFFFFFu;
    return (unsigned)s * (unsigned)m.vpr +
           (unsigned)((gx - rx * m.dim) + m.dim * ((gy - ry * m.dim) + m.dim * (gz - rz * m.dim)));
}

// DDA step of traversal._walk_grid (traversal.py:96-108): axis = 0; if
// t[1] < t[0]: 1; if t[2] < t[axis]: 2; t[axis] += delta[axis].  Three
// compares, three predicated adds; returns the axis.
__device__ __forceinline__ int dda_advance(double &tx, double &ty, double &tz, double dx, double dy,
                                           double dz) {
    int ax;
    asm("{\n\t.reg .pred py, pzx, pzy, pz, qx, qy, t0;\n\t"
        "setp.lt.f64 py, %1, %0;\n\t"
        "setp.lt.f64 pzx, %2, %0;\n\t"
        "setp.lt.f64 pzy, %2, %1;\n\t"
        "and.pred t0, py, pzy;\n\t"
        "not.pred qx, py;\n\t"
        "and.pred qx, qx, pzx;\n\t"
        "or.pred pz, t0, qx;\n\t"
        "not.pred t0, pz;\n\t"
        "and.pred qy, py, t0;\n\t"
        "not.pred qx, py;\n\t"
        "and.pred qx, qx, t0;\n\t"
        "@qx add.rn.f64 %0, %0, %4;\n\t"
        "@qy add.rn.f64 %1, %1, %5;\n\t"
        "@pz add.rn.f64 %2, %2, %6;\n\t"
        "selp.b32 %3, 1, 0, qy;\n\t"
        "@pz mov.b32 %3, 2;\n\t"
        "}"
        : "+d"(tx), "+d"(ty), "+d"(tz), "=r"(ax)
        : "d"(dx), "d"(dy), "d"(dz));
    return ax;
}

template <int MODE, bool DET, bool REC_ONLY, class Src>
__global__ void __launch_bounds__(BLOCK, WK_BLOCKS) k_walk(const __grid_constant__ DevMap m, Src src) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WalkSmem &sm = *reinterpret_cast<WalkSmem *>(smem_raw);
    if (!read_go(m)) return;
    if (DET && MODE == M_OCC && m.walk_det_launched && m.rbox[3] - m.rbox[0] < 509 &&
        m.rbox[4] - m.rbox[1] < 509 && m.rbox[5] - m.rbox[2] < 509)
        return;  // k_walk_det handled the batch
    const unsigned long long nseg_total =
        min(*((volatile unsigned long long *)(m.stats + S_SEGDESC)), m.seg_cap);
    const bool have_grid = *((volatile unsigned long long *)(m.stats + S_RGRID)) != 0;
    if (threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a) {
            sm.gb[a] = m.rbox[a];
            sm.gn[a] = have_grid ? m.rbox[3 + a] - m.rbox[a] + 1 : 0;
        }
        sm.gsmem = sm.gn[0] * sm.gn[1] * sm.gn[2] <= RG_SMEM;
        if (nseg_total) {
            const SegDesc &d0 = m.segs[0];
            int r0[3];
            unpack_region(d0.rkey, r0);
            for (int a = 0; a < 3; ++a)
                sm.anchor[a] = r0[a] * m.dim + (int)((d0.lp0 >> (10 * a)) & 1023u) - 1 - WCUBE / 2;
        } else {
            sm.anchor[0] = sm.anchor[1] = sm.anchor[2] = 1 << 29;
        }
    }
    for (int k = threadIdx.x; k < WCUBE_N / 32; k += blockDim.x) sm.cmark[k] = 0u;
    __syncthreads();
    if (sm.gsmem) {
        const int ncell = sm.gn[0] * sm.gn[1] * sm.gn[2];
        for (int k = threadIdx.x; k < ncell; k += blockDim.x) {
            const int sl = m.rgrid[k];
            sm.grid[k] = make_int2(sl, sl >= 0 && sl < m.cap ? (int)__ldcg(m.bmask + sl) : -1);
        }
    }
    __syncthreads();
    unsigned *const scr = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);
    float *const occ = reinterpret_cast<float *>(m.slab[L_OCC]);
    for (int k = threadIdx.x; k < WCUBE_N; k += blockDim.x) {
        sm.cube[k] = 0u;
        if (DET) {
            const unsigned vid = walk_vid(m, sm, sm.anchor[0] + k % WCUBE,
                                          sm.anchor[1] + (k / WCUBE) % WCUBE,
                                          sm.anchor[2] + k / (WCUBE * WCUBE), false);
            if (vid != 0xFFFFFFFFu && (__ldcg(scr + vid) & MARK_FLAG))
                atomicOr(sm.cmark + (k >> 5), 1u << (k & 31));
        }
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const int dim = m.dim;
    const unsigned vpr = (unsigned)m.vpr;
    const int dim2 = dim * dim;
    const int bs = m.brick_shift;
    unsigned long long *const wbuf = sm.wbuf[threadIdx.x >> 5];
    unsigned wcnt = 0, wflushed = 0;  // warp-uniform record ring counters

    unsigned visits = 0, rmiss = 0, retries = 0;
    // segment state
    double tx = 0, ty = 0, tz = 0, dx = 0, dy = 0, dz = 0, tprev = 0, L = 0;
    long long rkey = 0;
    unsigned lp = 0, vbase = 0xFFFFFFFFu, codes = 0, order = 0, cp = 0, bm = 0;
    int li = 0, rem = 0;
    bool active = false, in_cube = false;
    // deterministic path: visits in bricks holding a sample voxel wait as
    // candidates until the next retire (<= WK_INNER per lane)
    int ncand = 0;
    // CAS path: one visit in flight
    bool c_pend = false;
    unsigned c_old = 0;
    unsigned *c_ptr = nullptr;
    // prefetch + warp work pool
    bool pf_valid = false, exhausted = false;
    unsigned pool_next = 0, pool_end = 0;  // work indices (< 2^32 segments per batch)
    SegDesc *my_pf = &sm.pf[threadIdx.x];

    // record append (warp-aggregated; all lanes of the warp call it together)
    auto push_records = [&](bool rec, unsigned long long key) {
        const unsigned rb = __ballot_sync(0xffffffffu, rec);
        if (!rb) return;
        if (rec) wbuf[(wcnt + __popc(rb & lanemask_lt)) & (WK_WBUF - 1)] = key;
        wcnt += __popc(rb);
        if (wcnt - wflushed >= 32) {
            __syncwarp();
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(m.stats + S_RECORDS, 32ULL);
            b = __shfl_sync(0xffffffffu, b, 0);
            if (b + lane < m.rec_cap) m.rec[b + lane] = wbuf[(wflushed + lane) & (WK_WBUF - 1)];
            wflushed += 32;
            __syncwarp();
        }
    };

    // resolve the candidates: one batch of loads of their scratch words
    // (MARK_FLAG = sample voxel -> record; otherwise the delayed miss count).
    // key_mi: the word of a sample voxel holds MARK_FLAG | its index in the
    // batch's sample-voxel list, which then keys the record.
    auto retire = [&]() {
        if (!DET) return;
        if (!__any_sync(0xffffffffu, ncand != 0)) return;
        unsigned long long key[WK_INNER];
        unsigned w[WK_INNER];
        const unsigned long long omask = (1ULL << m.order_bits) - 1;
#pragma unroll
        for (int q = 0; q < WK_INNER; ++q) {
            key[q] = q < ncand ? sm.cand[q][threadIdx.x] : ~0ULL;
            w[q] = 0u;
            // cube candidates (bit 63) are sample voxels already
            if (q < ncand && (m.key_mi || !(key[q] & (1ULL << 63))))
                w[q] = __ldcg(scr + (unsigned)((key[q] & ~(1ULL << 63)) >> m.order_bits));
        }
#pragma unroll
        for (int q = 0; q < WK_INNER; ++q) {
            const bool valid = q < ncand;
            const bool cube_rec = valid && (key[q] & (1ULL << 63));
            const bool rec = cube_rec || (valid && (w[q] & MARK_FLAG));
            if (valid && !rec && !REC_ONLY) red_add(scr + (unsigned)(key[q] >> m.order_bits), 1u);
            const unsigned long long k = key[q] & ~(1ULL << 63);
            push_records(rec, m.key_mi ? ((unsigned long long)(w[q] & ~MARK_FLAG) << m.order_bits) |
                                             (k & omask)
                                       : k);
        }
        ncand = 0;
    };

    // one DDA step = one voxel visit
    auto step = [&]() {
        // ---- idle lanes start their prefetched segment ----
        if (!active && pf_valid) {
            __pipeline_wait_prior(0);
            const SegDesc &d = *my_pf;
            tx = d.t[0]; ty = d.t[1]; tz = d.t[2];
            dx = d.d[0]; dy = d.d[1]; dz = d.d[2];
            codes = d.flags;
            order = d.order;
            rem = (int)d.rem;
            lp = d.lp0;
            li = (int)(lp & 1023u) - 1 +
                 dim * ((int)((lp >> 10) & 1023u) - 1 + dim * ((int)(lp >> 20) - 1));
            rkey = d.rkey;
            {
                unsigned b2;
                const int s0 = walk_region(m, sm, rkey, b2);
                vbase = s0 >= 0 && s0 < m.cap ? (unsigned)s0 * vpr : 0xFFFFFFFFu;
                bm = b2;
            }
            L = d.L;
            sm.endc[threadIdx.x][0] = d.e[0];
            sm.endc[threadIdx.x][1] = d.e[1];
            sm.endc[threadIdx.x][2] = d.e[2];
            tprev = 0.0;
            // a straight segment leaves the (convex) cube for good
            int r0[3];
            unpack_region(rkey, r0);
            const unsigned ux = (unsigned)(r0[0] * dim + (int)(lp & 1023u) - 1 - sm.anchor[0]);
            const unsigned uy = (unsigned)(r0[1] * dim + (int)((lp >> 10) & 1023u) - 1 - sm.anchor[1]);
            const unsigned uz = (unsigned)(r0[2] * dim + (int)(lp >> 20) - 1 - sm.anchor[2]);
            in_cube = (ux | uy | uz) < (unsigned)WCUBE;
            cp = ux | (uy << 8) | (uz << 16);
            pf_valid = false;
            active = true;
        }
        if (!DET && c_pend) {
            c_pend = false;
            unsigned old = c_old;
            for (;;) {
                const unsigned nb = __float_as_uint(
                    clamp_add(__uint_as_float(old), m.miss32, m.cmin, m.cmax));
                if (nb == old) break;
                const unsigned prev = atomicCAS(c_ptr, old, nb);
                if (prev == old) break;
                old = prev;
                ++retries;
            }
        }
        if (!active) return;

        const bool last = rem == 0;
        if (last) {
            int r[3];
            unpack_region(rkey, r);
            const int gx = r[0] * dim + (int)(lp & 1023u) - 1;
            const int gy = r[1] * dim + (int)((lp >> 10) & 1023u) - 1;
            const int gz = r[2] * dim + (int)(lp >> 20) - 1;
            const int ex = sm.endc[threadIdx.x][0], ey = sm.endc[threadIdx.x][1],
                      ez = sm.endc[threadIdx.x][2];
            if (gx != ex || gy != ey || gz != ez) {
                // numerical fallback: the walk jumps to the end cell (traversal.py:88-92)
                const unsigned vid = walk_vid(m, sm, ex, ey, ez);
                vbase = vid == 0xFFFFFFFFu ? vid : vid - vid % vpr;
                li = vid == 0xFFFFFFFFu ? 0 : (int)(vid % vpr);
                bm = 0xFFFFFFFFu;  // conservative: the end voxel is a candidate
                in_cube = false;
            }
        }
        double t1 = 1.0;
        if (MODE == M_DECAY && !last) {
            // t_next = min over axes with the same tie-break, clamped to [t_prev, 1]
            const double ta = ty < tx ? ty : tx;
            t1 = tz < ta ? tz : ta;
            if (t1 < tprev) t1 = tprev;
            if (t1 > 1.0) t1 = 1.0;
        }
        ++visits;
        if (vbase == 0xFFFFFFFFu) {
            ++rmiss;
        } else {
            const unsigned vid = vbase + (unsigned)li;
            const bool hit = last && (codes & 1u);
            if (MODE == M_DECAY && !REC_ONLY) {
                red_add(reinterpret_cast<double *>(m.slab[L_DDIST]) + vid, (t1 - tprev) * L);
                if (hit) red_add(reinterpret_cast<unsigned *>(m.slab[L_DHITS]) + vid, 1u);
            }
            const unsigned ck = cube_cell(cp);
            if (DET) {
                const unsigned long long rk =
                    ((unsigned long long)vid << m.order_bits) | order | (hit ? 1u : 0u);
                if (in_cube) {
                    if ((sm.cmark[ck >> 5] >> (ck & 31)) & 1u) {
                        // sample voxel in the cube: a record for sure (bit 63 tags it)
                        sm.cand[ncand++][threadIdx.x] = rk | (1ULL << 63);
                    } else if (!REC_ONLY) {
                        atomicAdd(sm.cube + ck, 1u);
                    }
                } else {
                    int b = 0;
                    if (bs >= 0) {
                        const unsigned u = lp - 0x00100401u;  // unbiased lx | ly << 10 | lz << 20
                        b = (int)(((u >> bs) & 3u) | ((u >> (8 + bs)) & 0xCu) |
                                  ((u >> (17 + bs)) & 0x10u));
                    }
                    if ((bm >> b) & 1u) sm.cand[ncand++][threadIdx.x] = rk;
                    else if (!REC_ONLY) red_add(scr + vid, 1u);
                }
            } else if (hit) {
                float *p = occ + vid;
                unsigned old = __float_as_uint(__ldcg(p));
                for (;;) {
                    const unsigned nb = __float_as_uint(
                        clamp_add(__uint_as_float(old), m.hit32, m.cmin, m.cmax));
                    if (nb == old) break;
                    const unsigned prev = atomicCAS(reinterpret_cast<unsigned *>(p), old, nb);
                    if (prev == old) break;
                    old = prev;
                    ++retries;
                }
                if (m.slab[L_MEAN]) {
                    // a hit ends a has_sample segment: its end is the ray end
                    double e[3];
                    float it;
                    src.load_end((long long)((order >> 1) / (unsigned)m.maxseg), e, it);
                    const int ex = sm.endc[threadIdx.x][0], ey = sm.endc[threadIdx.x][1],
                              ez = sm.endc[threadIdx.x][2];
                    const double off[3] = {e[0] / m.vox - (double)ex, e[1] / m.vox - (double)ey,
                                           e[2] / m.vox - (double)ez};
                    retries += cas_mean(reinterpret_cast<unsigned *>(m.slab[L_MEAN]) + vid,
                                        reinterpret_cast<unsigned *>(m.slab[L_COUNT]) + vid, off);
                }
            } else if (in_cube) {
                atomicAdd(sm.cube + ck, 1u);
            } else {
                c_pend = true;
                c_ptr = reinterpret_cast<unsigned *>(occ + vid);
                c_old = __float_as_uint(__ldcg(occ + vid));
            }
        }
        if (last) {
            active = false;
            return;
        }
        // ---- advance (t_max[axis] += t_delta[axis]) ----
        tprev = t1;
        --rem;
        const int ax = dda_advance(tx, ty, tz, dx, dy, dz);
        const int sh = 10 * ax;
        const int st = (int)((codes >> (1 + 2 * ax)) & 3u) - 1;
        const int stride = ax == 2 ? dim2 : (ax == 1 ? dim : 1);
        lp += (unsigned)st << sh;
        li += st * stride;
        if (in_cube) {
            cp += (unsigned)st << (8 * ax);
            in_cube = (cp & CUBE_OUT) == 0;
        }
        const unsigned f = (lp >> sh) & 1023u;
        if (f - 1u >= (unsigned)dim) {
            // region crossing: wrap the local coordinate, step the region key
            lp += (unsigned)(-st * dim) << sh;
            li -= st * dim * stride;
            rkey += (long long)st << (21 * (2 - ax));
            unsigned b2;
            const int s = walk_region(m, sm, rkey, b2);
            vbase = s >= 0 && s < m.cap ? (unsigned)s * vpr : 0xFFFFFFFFu;
            bm = b2;
        }
    };

    for (;;) {
        retire();
        // ---- claim work for lanes without a prefetched descriptor ----
        unsigned need = __ballot_sync(0xffffffffu, !pf_valid && !exhausted);
        while (need) {
            if (pool_next >= pool_end) {
                unsigned b = 0;
                if (lane == 0) b = (unsigned)atomicAdd(m.work, 32ULL);
                b = __shfl_sync(0xffffffffu, b, 0);
                pool_next = b;
                pool_end = b + 32;
                if (b >= nseg_total) {
                    if ((need >> lane) & 1u) exhausted = true;
                    break;
                }
            }
            const unsigned avail = pool_end - pool_next;
            const unsigned rank = __popc(need & lanemask_lt);
            const bool served = ((need >> lane) & 1u) && rank < avail;
            if (served) {
                const unsigned long long w = (unsigned long long)pool_next + rank;
                if (w < nseg_total) {
                    // longest segments first (k_seg_order)
                    const char *g = reinterpret_cast<const char *>(m.segs + m.perm[w]);
#pragma unroll
                    for (int q = 0; q < (int)(sizeof(SegDesc) / 16); ++q)
                        __pipeline_memcpy_async(reinterpret_cast<char *>(my_pf) + 16 * q,
                                                g + 16 * q, 16);
                    __pipeline_commit();
                    pf_valid = true;
                } else {
                    exhausted = true;
                }
            }
            const unsigned served_mask = __ballot_sync(0xffffffffu, served);
            pool_next += __popc(served_mask);
            need &= ~served_mask;
        }
        if (!__any_sync(0xffffffffu, active || pf_valid || !exhausted || c_pend)) break;
#pragma unroll 1
        for (int q = 0; q < WK_INNER; ++q) step();
    }
    retire();
    // flush the warp's remaining records
    if (DET) {
        __syncwarp();
        const unsigned left = wcnt - wflushed;
        if (left) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(m.stats + S_RECORDS, (unsigned long long)left);
            b = __shfl_sync(0xffffffffu, b, 0);
            if ((unsigned)lane < left && b + lane < m.rec_cap)
                m.rec[b + lane] = wbuf[(wflushed + lane) & (WK_WBUF - 1)];
        }
    }

    __syncthreads();
    unsigned long long flushed = 0;
    if (!REC_ONLY) {
        for (int k = threadIdx.x; k < WCUBE_N; k += blockDim.x) {
            const unsigned cntk = sm.cube[k];
            if (!cntk) continue;
            ++flushed;
            const unsigned vid = walk_vid(m, sm, sm.anchor[0] + k % WCUBE,
                                          sm.anchor[1] + (k / WCUBE) % WCUBE,
                                          sm.anchor[2] + k / (WCUBE * WCUBE), true);
            if (vid == 0xFFFFFFFFu) continue;
            if (DET) red_add(scr + vid, cntk);
            else retries += cas_apply_k(occ + vid, m.miss32, cntk, m.cmin, m.cmax);
        }
    }
    if (!REC_ONLY) {
        unsigned long long st[4] = {visits, rmiss, retries, flushed};
        const int which[4] = {S_VISITS, S_RMISS, S_RETRIES, S_CUBE_FLUSH};
        block_add_stats(m, st, which);
    }
}

}  // namespace vm
