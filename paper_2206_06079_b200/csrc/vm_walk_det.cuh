// vm_walk_det.cuh -- the deterministic occupancy walk (the hot kernel of the
// default path).
//
// Same walk as k_walk (vm_walk.cuh): one warp = 32 lanes, each walking one
// preprocessed segment with the exact fp64 DDA of traversal._walk_grid
// (traversal.py:80-111), longest segments first.  What differs is the visit:
// a visit is a fire-and-forget RED.ADD on the voxel's scratch counter (the
// order-free miss count, resolved as f_miss^k by k_resolve) unless the
// voxel's brick (8 x 8 x 16 voxels at dim 32) holds one of the batch's sample
// voxels -- a bit test against the region's brick summary, which k_discover
// built while stamping MARK_FLAG into the sample voxels' counters.  Visits in
// such bricks are candidates: their voxel ids wait in shared memory and are
// resolved together at the end of the eight-step window (one batch of loads
// of their counters: MARK_FLAG -> an order-keyed record (voxel id, ray order,
// hit) for the in-order fold, otherwise the delayed miss count).  Around the
// sensor, visits count into the block's shared-memory cube, which carries its
// own sample-voxel bitmap.
//
// The step is written for the common case and the eight steps of a window
// are unrolled.  Region crossings step a grid index
// through the batch's dense region grid (shared memory); only a crossing out
// of the grid probes the hash table.  Segment starts happen at window
// boundaries.
#pragma once

#include "vm_walk.cuh"

namespace vm {

#ifndef VM_WD_STEPS
#define VM_WD_STEPS 8
#endif
constexpr int WD_STEPS = VM_WD_STEPS;  // steps per window (in-flight visits per lane)
#ifndef VM_WD_UNROLL
#define VM_WD_UNROLL 1  // steps of the window loop unrolled
#endif
constexpr int WD_UNROLL = VM_WD_UNROLL;
#ifndef VM_WD_AGG
#define VM_WD_AGG 0  // measured: 31% fewer REDs but +16% instructions and MATCH latency
                     // (short-scoreboard stalls): C2 walk 60.9 -> 94.2 ms per step
#endif
constexpr bool WD_AGG = VM_WD_AGG;       // warp-merged miss counts (match_any per step)
constexpr unsigned long long WD_NONE = ~0ULL;
constexpr unsigned long long WD_CUBE_TAG = 1ULL << 40;  // key = cube cell, not a voxel id
#ifndef VM_WD_BLOCKS
#define VM_WD_BLOCKS 3
#endif
constexpr int WD_BLOCKS = VM_WD_BLOCKS;  // resident blocks per SM
#ifndef VM_WD_DEFER
#define VM_WD_DEFER 0
#endif
// 1: a window's candidate counter loads are consumed one window later (the
// L2 round trip overlaps the next eight steps instead of stalling the warp)
constexpr int WD_DEFER = VM_WD_DEFER;

struct WalkDetSmem {
    unsigned cube[WCUBE_N];          // miss counts around the sensor
    unsigned cmark[WCUBE_N / 32];    // sample-voxel bitmap of the cube
    int2 grid[RG_SMEM_DET];          // (slot, brick summary of sample voxels)
    unsigned long long wbuf[BLOCK / 32][WK_WBUF];
    unsigned vids[1 + WD_DEFER][WD_STEPS][BLOCK];  // voxel id of each in-flight visit
    SegDesc pf[BLOCK];
    int endc[BLOCK][3];
    int gb[3], gn[3], gs[3];  // grid origin, extents, strides (1, nx, nx*ny)
    int anchor[3];
    int gmode;                // 1: grid in smem, 2: grid in global memory, 0: hash only
};

// region slot for grid-relative coordinates packed in rp (fields biased by
// RP_BIAS); inserts walk-entered regions like the generic walk
__device__ __noinline__ int wd_slow_region(const DevMap &m, const WalkDetSmem &sm, unsigned rp,
                                           unsigned *bm) {
    const int rx = sm.gb[0] + (int)(rp & 1023u) - RP_BIAS;
    const int ry = sm.gb[1] + (int)((rp >> 10) & 1023u) - RP_BIAS;
    const int rz = sm.gb[2] + (int)(rp >> 20) - RP_BIAS;
    const unsigned ux = (unsigned)(rx - sm.gb[0]), uy = (unsigned)(ry - sm.gb[1]),
                   uz = (unsigned)(rz - sm.gb[2]);
    if (sm.gmode && ux < (unsigned)sm.gn[0] && uy < (unsigned)sm.gn[1] && uz < (unsigned)sm.gn[2]) {
        const int gi = ux + sm.gs[1] * uy + sm.gs[2] * uz;
        const int s = sm.gmode == 1 ? sm.grid[gi].x : __ldg(m.rgrid + gi);
        if (s >= 0 && s < m.cap) {
            *bm = sm.gmode == 1 ? (unsigned)sm.grid[gi].y : __ldg(m.bmask + s);
            return s;
        }
    }
    const int slot = region_slot_inl(m, pack_region(rx, ry, rz));
    *bm = slot >= 0 && slot < m.cap ? __ldcg(m.bmask + slot) : 0xFFFFFFFFu;
    if (slot >= 0 && slot < m.cap && stamp_epoch(m.slot_touch + slot, m.epoch)) {
        const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
        if (t < (unsigned long long)m.touched_cap) m.touched[t] = slot;
    }
    return slot;
}

template <int DIM>
__device__ __noinline__ unsigned wd_vid_of(const DevMap &m, const WalkDetSmem &sm, int gx, int gy,
                                           int gz, bool insert) {
    // DIM = 32: floor division by the region edge is an arithmetic shift
    const int rx = DIM == 32 ? gx >> 5 : floordiv(gx, m.dim);
    const int ry = DIM == 32 ? gy >> 5 : floordiv(gy, m.dim);
    const int rz = DIM == 32 ? gz >> 5 : floordiv(gz, m.dim);
    int s;
    const unsigned ux = (unsigned)(rx - sm.gb[0]), uy = (unsigned)(ry - sm.gb[1]),
                   uz = (unsigned)(rz - sm.gb[2]);
    if (sm.gmode && ux < (unsigned)sm.gn[0] && uy < (unsigned)sm.gn[1] && uz < (unsigned)sm.gn[2]) {
        const int gi = ux + sm.gs[1] * uy + sm.gs[2] * uz;
        s = sm.gmode == 1 ? sm.grid[gi].x : __ldg(m.rgrid + gi);
        if (s < 0) s = insert ? region_slot_inl(m, pack_region(rx, ry, rz)) : -1;
    } else {
        s = insert ? region_slot_inl(m, pack_region(rx, ry, rz))
                   : region_find_probe(m, pack_region(rx, ry, rz));
        if (s >= 0 && s < m.cap && stamp_epoch(m.slot_touch + s, m.epoch)) {
            const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
            if (t < (unsigned long long)m.touched_cap) m.touched[t] = s;
        }
    }
    if (s < 0 || s >= m.cap) return 0xFFFFFFFFu;
    return (unsigned)s * (unsigned)m.vpr +
           (unsigned)((gx - rx * m.dim) + m.dim * ((gy - ry * m.dim) + m.dim * (gz - rz * m.dim)));
}

// brick bit of local index li; DIM = 32 (the default region) folds the shifts
template <int DIM>
__device__ __forceinline__ unsigned wd_brick(int li, const int bsh[3]) {
    if (DIM == 32)
        return (((unsigned)li >> 3) & 3u) | (((unsigned)li >> 6) & 0xCu) |
               (((unsigned)li >> 10) & 0x10u);
    return brick_of(li, bsh);
}

// DIM: compile-time region edge (32), or 0 for any other region_dim.
// SHARD: a region-sharded map (walk-created regions force records); single
// GPU maps compile that bookkeeping out.
template <bool REC_ONLY, class Src, int DIM = 0, bool SHARD = true>
__global__ void __launch_bounds__(BLOCK, WD_BLOCKS) k_walk_det(const __grid_constant__ DevMap m,
                                                               Src src) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WalkDetSmem &sm = *reinterpret_cast<WalkDetSmem *>(smem_raw);
    if (!read_go(m) || !walk_det_ok(m)) return;
    const unsigned long long nseg_total =
        min(*((volatile unsigned long long *)(m.stats + S_SEGDESC)), m.seg_cap);
    const bool have_grid = *((volatile unsigned long long *)(m.stats + S_RGRID)) != 0;
    if (threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a) {
            sm.gb[a] = m.rbox[a];
            sm.gn[a] = have_grid ? m.rbox[3 + a] - m.rbox[a] + 1 : 0;
        }
        sm.gs[0] = 1;
        sm.gs[1] = sm.gn[0];
        sm.gs[2] = sm.gn[0] * sm.gn[1];
        const int ncell = sm.gn[0] * sm.gn[1] * sm.gn[2];
        sm.gmode = !have_grid ? 0 : (ncell <= RG_SMEM_DET ? 1 : 2);
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
    __syncthreads();
    if (sm.gmode == 1) {
        const int ncell = sm.gn[0] * sm.gn[1] * sm.gn[2];
        for (int k = threadIdx.x; k < ncell; k += blockDim.x) {
            const int sl = m.rgrid[k];
            sm.grid[k] = make_int2(sl, sl >= 0 && sl < m.cap ? (int)__ldcg(m.bmask + sl) : 0);
        }
    }
    __syncthreads();
    unsigned *const scr = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);
    {
        // the cube's sample-voxel bitmap: every voxel id first, then all the
        // scratch loads in flight together, one ballot per 32 cells
        static_assert(WCUBE_N % BLOCK == 0, "cube cells per thread");
        constexpr int PER = WCUBE_N / BLOCK;
        unsigned vid[PER], c[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int k = threadIdx.x + j * BLOCK;
            vid[j] = wd_vid_of<DIM>(m, sm, sm.anchor[0] + k % WCUBE, sm.anchor[1] + (k / WCUBE) % WCUBE,
                                    sm.anchor[2] + k / (WCUBE * WCUBE), false);
            sm.cube[k] = 0u;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) c[j] = vid[j] != 0xFFFFFFFFu ? __ldcg(scr + vid[j]) : 0u;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const unsigned word = __ballot_sync(0xffffffffu, (c[j] & MARK_FLAG) != 0u);
            if ((threadIdx.x & 31) == 0) sm.cmark[(threadIdx.x + j * BLOCK) >> 5] = word;
        }
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const int dim = DIM ? DIM : m.dim;
    const unsigned vpr = DIM ? (unsigned)(DIM * DIM * DIM) : (unsigned)m.vpr;
    const int ob = m.order_bits;
    unsigned long long *const wbuf = sm.wbuf[threadIdx.x >> 5];
    unsigned wcnt = 0, wflushed = 0;  // warp-uniform record ring counters
    unsigned rmiss = 0, visits = 0;

    // segment state
    double tx = 0, ty = 0, tz = 0, dx = 0, dy = 0, dz = 0;
    unsigned lp = 0, rp = 0, vbase = 0xFFFFFFFFu, okey = 0, cp = 0, bm = 0;
    const bool bricks = m.brick_shift >= 0;
    int li = 0, gi = 0, rem = 0;
    int dli0 = 0, dli1 = 0, dli2 = 0;       // local-index step per axis (DIM != 32)
    unsigned dlp0 = 0, dlp1 = 0, dlp2 = 0;  // packed-coordinate step per axis (DIM != 32)
    unsigned sg3 = 0;  // DIM 32: the step direction codes, 2 bits per axis (step + 1)
    bool active = false, in_cube = false, ingrid = false;
    // rare events park the lane until the window boundary, where they are
    // resolved outside the unrolled steps (no call inside them)
    int parked = 0;  // 1: region lookup after a crossing, 2: fallback jump to the end cell
    bool jumped = false;
    // sharded maps: a region created during the walk was not stamped with the
    // other ranks' sample voxels, so every visit in it is kept as a record
    bool forced = false;
    // candidates of the window: bit q of `live` -- slot q holds a candidate
    // (voxel id in sm.vids); `sure` -- known record (cube sample voxel / forced)
    unsigned live = 0, hits = 0, sure = 0;
    // WD_DEFER: the previous window's candidates (vids[par ^ 1]), their
    // counter words in flight, and its segment's order key
    unsigned par = 0;
    unsigned plive = 0, phits = 0, psure = 0, pokey = 0;
    unsigned pw[WD_STEPS];
#pragma unroll
    for (int q = 0; q < WD_STEPS; ++q) pw[q] = 0u;
    // WD_AGG (off): the step's miss count applied after the step by the warp
    // as a whole -- lanes counting the same voxel at the same step merge into
    // one atomic (~46% of C2's per-step counts outside the sensor cube share
    // a voxel with another lane); the MATCH per step costs more than it saves
    unsigned long long pend = WD_NONE;
    // prefetch + warp work pool
    bool pf_valid = false, exhausted = false;
    unsigned pool_next = 0, pool_end = 0;
    SegDesc *my_pf = &sm.pf[threadIdx.x];

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

    auto set_region = [&](int s, unsigned b) {
        vbase = s >= 0 && s < m.cap ? (unsigned)s * vpr : 0xFFFFFFFFu;
        bm = bricks ? b : 0xFFFFFFFFu;
        if (SHARD) forced = m.shard_world > 1 && s >= m.walk_slot0;
    };

    auto start = [&]() {
        __pipeline_wait_prior(0);
        const SegDesc &d = *my_pf;
        tx = d.t[0]; ty = d.t[1]; tz = d.t[2];
        dx = d.d[0]; dy = d.d[1]; dz = d.d[2];
        const unsigned codes = d.flags;
        okey = d.order | (codes & 1u);
        rem = (int)d.rem;
        visits += (unsigned)rem + 1u;
        lp = d.lp0;
        li = (int)(lp & 1023u) - 1 +
             dim * ((int)((lp >> 10) & 1023u) - 1 + dim * ((int)(lp >> 20) - 1));
        const int sx = (int)((codes >> 1) & 3u) - 1, sy = (int)((codes >> 3) & 3u) - 1,
                  sz = (int)((codes >> 5) & 3u) - 1;
        if (DIM == 32) {
            sg3 = (codes >> 1) & 63u;
        } else {
            dli0 = sx;
            dli1 = sy * dim;
            dli2 = sz * dim * dim;
            dlp0 = (unsigned)sx;
            dlp1 = (unsigned)sy << 10;
            dlp2 = (unsigned)sz << 20;
        }
        int r0[3];
        unpack_region(d.rkey, r0);
        const int u0 = r0[0] - sm.gb[0], u1 = r0[1] - sm.gb[1], u2 = r0[2] - sm.gb[2];
        rp = (unsigned)(u0 + RP_BIAS) | ((unsigned)(u1 + RP_BIAS) << 10) |
             ((unsigned)(u2 + RP_BIAS) << 20);
        ingrid = sm.gmode && (unsigned)u0 < (unsigned)sm.gn[0] && (unsigned)u1 < (unsigned)sm.gn[1] &&
                 (unsigned)u2 < (unsigned)sm.gn[2];
        gi = u0 + sm.gs[1] * u1 + sm.gs[2] * u2;
        {
            int s = -1;
            unsigned b = 0xFFFFFFFFu;
            if (ingrid) {
                if (sm.gmode == 1) {
                    const int2 ge = sm.grid[gi];
                    s = ge.x;
                    b = (unsigned)ge.y;
                } else {
                    s = __ldg(m.rgrid + gi);
                    if (s >= 0 && s < m.cap) b = __ldg(m.bmask + s);
                }
            }
            if (s < 0) s = wd_slow_region(m, sm, rp, &b);
            set_region(s, b);
        }
        sm.endc[threadIdx.x][0] = d.e[0];
        sm.endc[threadIdx.x][1] = d.e[1];
        sm.endc[threadIdx.x][2] = d.e[2];
        const unsigned ux = (unsigned)(r0[0] * dim + (int)(lp & 1023u) - 1 - sm.anchor[0]);
        const unsigned uy = (unsigned)(r0[1] * dim + (int)((lp >> 10) & 1023u) - 1 - sm.anchor[1]);
        const unsigned uz = (unsigned)(r0[2] * dim + (int)(lp >> 20) - 1 - sm.anchor[2]);
        in_cube = (ux | uy | uz) < (unsigned)WCUBE;
        cp = ux | (uy << 8) | (uz << 16);
        pf_valid = false;
        active = true;
        jumped = false;
    };

    // one DDA step = one voxel visit into in-flight slot Q (common case only)
    auto step = [&](const int Q) {  // Q: the window's step index (dynamic)
        if (!active) return;
        const bool last = rem == 0;
        if (last) {
            if (!jumped) {
                const int gx = sm.gb[0] + (int)(rp & 1023u) - RP_BIAS;
                const int gy = sm.gb[1] + (int)((rp >> 10) & 1023u) - RP_BIAS;
                const int gz = sm.gb[2] + (int)(rp >> 20) - RP_BIAS;
                const int cx = gx * dim + (int)(lp & 1023u) - 1;
                const int cy = gy * dim + (int)((lp >> 10) & 1023u) - 1;
                const int cz = gz * dim + (int)(lp >> 20) - 1;
                if (cx != sm.endc[threadIdx.x][0] || cy != sm.endc[threadIdx.x][1] ||
                    cz != sm.endc[threadIdx.x][2]) {
                    // numerical fallback: the walk jumps to the end cell (traversal.py:88-92)
                    parked = 2;
                    active = false;
                    return;
                }
            }
            if (okey & 1u) hits |= 1u << Q;
        }
        // ---- the visit: a miss count, or a candidate checked at the window's end ----
        const unsigned vid = vbase + (unsigned)li;
        if (vbase != 0xFFFFFFFFu) {
            if (in_cube) {
                const unsigned ck = cube_cell(cp);
                if (((sm.cmark[ck >> 5] >> (ck & 31)) & 1u) || (SHARD && forced)) {
                    sm.vids[par][Q][threadIdx.x] = vid;
                    live |= 1u << Q;
                    sure |= 1u << Q;
                } else if (!REC_ONLY) {
                    if (WD_AGG) pend = WD_CUBE_TAG | ck;
                    else atomicAdd(sm.cube + ck, 1u);
                }
            } else if (((bm >> wd_brick<DIM>(li, m.bsh)) & 1u) || (SHARD && forced)) {
                sm.vids[par][Q][threadIdx.x] = vid;
                live |= 1u << Q;
                if (SHARD && forced) sure |= 1u << Q;
            } else if (!REC_ONLY) {
                if (WD_AGG) pend = vid;
                else red_add(scr + vid, 1u);
            }
        } else {
            ++rmiss;
        }
        if (last) {
            active = false;
            return;
        }
        // ---- advance (t_max[axis] += t_delta[axis]) ----
        --rem;
        const int ax = dda_advance(tx, ty, tz, dx, dy, dz);
        const int sh = 10 * ax;
        int dl, sgn;
        unsigned dp;
        if (DIM == 32) {
            // branch-free: the axis' step from its 2-bit code; strides 1, 32, 1024
            sgn = (int)((sg3 >> (2 * ax)) & 3u) - 1;
            dl = (int)((unsigned)sgn << (5 * ax));
            dp = (unsigned)sgn << sh;
        } else {
            dl = ax == 2 ? dli2 : (ax == 1 ? dli1 : dli0);
            dp = ax == 2 ? dlp2 : (ax == 1 ? dlp1 : dlp0);
            sgn = (int)dp >> sh;
        }
        lp += dp;
        li += dl;
        if (in_cube) {
            cp += (unsigned)sgn << (8 * ax);  // the step (+-1) into the cube field
            in_cube = (cp & CUBE_OUT) == 0;
        }
        if (((lp >> sh) & 1023u) - 1u >= (unsigned)dim) {
            // region crossing: wrap the local coordinate, step the grid index
            lp -= (unsigned)dim * dp;
            li -= dim * dl;
            rp += dp;
            const unsigned f = ((rp >> sh) & 1023u) - RP_BIAS;
            gi += sgn * sm.gs[ax];
            ingrid = ingrid && f < (unsigned)sm.gn[ax];
            int s = -1;
            unsigned b = 0xFFFFFFFFu;
            if (ingrid) {
                if (sm.gmode == 1) {
                    const int2 ge = sm.grid[gi];
                    s = ge.x;
                    b = (unsigned)ge.y;
                } else {
                    s = __ldg(m.rgrid + gi);
                    if (s >= 0 && s < m.cap) b = __ldg(m.bmask + s);
                }
            }
            if (s >= 0) {
                set_region(s, b);
            } else {
                parked = 1;  // outside the grid or a region the prefetch did not create
                active = false;
            }
        }
    };

    // window boundary: resolve parked lanes (no visit in flight)
    auto unpark = [&]() {
        if (parked == 1) {
            unsigned b = 0xFFFFFFFFu;
            const int s = wd_slow_region(m, sm, rp, &b);
            set_region(s, b);
        } else if (parked == 2) {
            const unsigned vid = wd_vid_of<DIM>(m, sm, sm.endc[threadIdx.x][0], sm.endc[threadIdx.x][1],
                                           sm.endc[threadIdx.x][2], true);
            vbase = vid == 0xFFFFFFFFu ? vid : vid - vid % vpr;
            li = vid == 0xFFFFFFFFu ? 0 : (int)(vid % vpr);
            if (SHARD) forced = m.shard_world > 1 && vid != 0xFFFFFFFFu && (int)(vid / vpr) >= m.walk_slot0;
            bm = 0xFFFFFFFFu;  // the end voxel is a candidate
            in_cube = false;
            jumped = true;
        }
        parked = 0;
        active = true;
    };

    // candidates of one window (bit q of lv: slot q of vids[pp] holds one;
    // w: their counter words): records or the delayed miss count
    auto retire = [&](unsigned lv, unsigned sr, unsigned ht, unsigned ok, const unsigned(&w)[WD_STEPS],
                      unsigned pp) {
        unsigned v[WD_STEPS];
        // key_mi: the counter of a sample voxel holds MARK_FLAG | its index in
        // the batch's sample-voxel list, which then keys the record
#pragma unroll
        for (int q = 0; q < WD_STEPS; ++q) v[q] = ((lv >> q) & 1u) ? sm.vids[pp][q][threadIdx.x] : 0u;
        unsigned recm = 0u;
#pragma unroll
        for (int q = 0; q < WD_STEPS; ++q) {
            const bool cand = (lv >> q) & 1u;
            const bool rec = cand && (((sr >> q) & 1u) || (w[q] & MARK_FLAG));
            if (cand && !rec && !REC_ONLY) red_add(scr + v[q], 1u);
            recm |= (unsigned)rec << q;
        }
        // records (a few per window at most): only the steps some lane holds one
        const unsigned wrec = __reduce_or_sync(0xffffffffu, recm);
        if (wrec) {
#pragma unroll
            for (int q = 0; q < WD_STEPS; ++q) {
                if (!((wrec >> q) & 1u)) continue;  // warp-uniform
                const unsigned long long kf = m.key_mi ? (w[q] & ~MARK_FLAG) : v[q];
                push_records((recm >> q) & 1u, (kf << ob) | (ok & ~1u) | ((ht >> q) & 1u));
            }
        }
    };

    for (;;) {
        // ---- retire the window: candidates become records or miss counts ----
        if (__any_sync(0xffffffffu, (live | plive) != 0u)) {
            if (WD_DEFER) {
                retire(plive, psure, phits, pokey, pw, par ^ 1u);
                // issue this window's loads; they are read at the next retire
                const unsigned need = m.key_mi ? live : (live & ~sure);
#pragma unroll
                for (int q = 0; q < WD_STEPS; ++q)
                    pw[q] = ((need >> q) & 1u) ? __ldcg(scr + sm.vids[par][q][threadIdx.x]) : 0u;
                plive = live;
                psure = sure;
                phits = hits;
                pokey = okey;
                par ^= 1u;
            } else {
                unsigned w[WD_STEPS];
                const unsigned need = m.key_mi ? live : (live & ~sure);
#pragma unroll
                for (int q = 0; q < WD_STEPS; ++q)
                    w[q] = ((need >> q) & 1u) ? __ldcg(scr + sm.vids[0][q][threadIdx.x]) : 0u;
                retire(live, sure, hits, okey, w, 0u);
            }
            live = 0u;
            hits = 0u;
            sure = 0u;
        }
        if (parked) unpark();
        if (!active && pf_valid) start();
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
        if (!__any_sync(0xffffffffu, active || pf_valid || !exhausted || parked)) break;
        if (!__any_sync(0xffffffffu, active)) continue;
#pragma unroll WD_UNROLL
        for (int q = 0; q < WD_STEPS; ++q) {
            step(q);
            if (WD_AGG && !REC_ONLY) {
                const unsigned long long key = pend;
                pend = WD_NONE;
                const unsigned grp = __match_any_sync(0xffffffffu, key);
                if (key != WD_NONE && (grp & lanemask_lt) == 0u) {  // the group's lowest lane
                    const unsigned c = __popc(grp);
                    if (key & WD_CUBE_TAG) atomicAdd(sm.cube + (unsigned)key, c);
                    else red_add(scr + (unsigned)key, c);
                }
            }
        }
    }
    if (WD_DEFER && __any_sync(0xffffffffu, plive != 0u)) retire(plive, psure, phits, pokey, pw, par ^ 1u);
    // flush the warp's remaining records
    __syncwarp();
    {
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
            const unsigned c = sm.cube[k];
            if (!c) continue;
            ++flushed;
            const unsigned vid = wd_vid_of<DIM>(m, sm, sm.anchor[0] + k % WCUBE,
                                           sm.anchor[1] + (k / WCUBE) % WCUBE,
                                           sm.anchor[2] + k / (WCUBE * WCUBE), true);
            if (vid != 0xFFFFFFFFu) red_add(scr + vid, c);
        }
        unsigned long long st[3] = {visits, rmiss, flushed};
        const int which[3] = {S_VISITS, S_RMISS, S_CUBE_FLUSH};
        block_add_stats(m, st, which);
    }
}

}  // namespace vm
