// vm_walk_ndt_det.cuh -- the deterministic NDT phase-1 walk over segment
// descriptors (the hot kernel of NDT-OM / NDT-TM).
//
// k_walk_det's machinery (vm_walk_det.cuh) with NDT's visit: one warp = 32
// lanes, each walking one preprocessed segment (SegDesc from k_discover, the
// exact fp64 DDA of traversal._walk_grid), longest segments first, new
// segments claimed from a warp pool at window boundaries.  A visit
// (reference.py:67-94 / _kernels.pyx:602-648) is
//   * the segment's sample voxel: nothing (phase 2, a record k_discover filed);
//   * a miss through a voxel holding a Gaussian (count >= 3 at the start of
//     the batch): a phase-1 record (voxel index | ray order) with its chord
//     (t0, t1), weighed after the walk (k_ndt_weigh) and folded in ray order;
//   * any other miss: g = 1, an order-free count on the voxel's scratch word
//     (k_resolve applies f_miss^k with the transient reset).
// Whether a voxel holds a Gaussian is only asked in bricks whose Gaussian
// summary bit (gmask, set by the fold when a count reaches 3) is set; those
// visits are candidates whose counts are loaded together at the end of the
// window.  Around the sensor, visits count into the block's shared-memory
// cube, whose Gaussian bitmap is loaded once per block.
//
// The chord of a visit is walk()'s (vm_device.cuh): t0 = the previous
// visit's exit, t1 = min(t_max) clamped to [t0, 1], and 1 for the segment's
// last visit -- the same doubles the generic walk (k_walk_ndt) computes.
// Sharded maps (ghost regions), record re-emission after an overflow and
// batches whose region box is too large for the packed grid coordinates take
// k_walk_ndt.
#pragma once

#include "vm_walk_det.cuh"

namespace vm {

#ifndef VM_WN_STEPS
#define VM_WN_STEPS 8
#endif
constexpr int WN_STEPS = VM_WN_STEPS;  // steps per window (in-flight candidates per lane)
#ifndef VM_WN_BLOCKS
#define VM_WN_BLOCKS 2
#endif
constexpr int WN_BLOCKS = VM_WN_BLOCKS;  // resident blocks per SM
constexpr int WN_WBUF = 64;              // per-warp record ring (flushed 32 at a time)

// the sensor cube of this walk (log2 edge; 4 = k_walk_det's 16^3)
#ifndef VM_WN_CB
#define VM_WN_CB 4
#endif
constexpr int NCB = VM_WN_CB;
constexpr int NCUBE = 1 << NCB;
constexpr int NCUBE_N = NCUBE * NCUBE * NCUBE;
__device__ __forceinline__ unsigned ncube_cell(unsigned cp) {
    return (cp & (NCUBE - 1u)) | ((cp >> (8 - NCB)) & ((NCUBE - 1u) << NCB)) |
           ((cp >> (16 - 2 * NCB)) & ((NCUBE - 1u) << (2 * NCB)));
}
constexpr unsigned NCUBE_OUT = (0xFFu & ~(NCUBE - 1u)) * 0x010101u;
static_assert(NCUBE_N % BLOCK == 0, "cube cells per thread");

struct WalkNdtSmem {
    unsigned cube[NCUBE_N];            // order-free miss counts around the sensor
    unsigned cgauss[NCUBE_N / 32];     // cube voxels holding a Gaussian
    int2 grid[RG_SMEM_DET];            // (slot, Gaussian brick summary)
    unsigned long long wkey[BLOCK / 32][WN_WBUF];
    double2 wt[BLOCK / 32][WN_WBUF];
    unsigned vids[WN_STEPS][BLOCK];    // voxel id of each candidate visit
    double2 tv[WN_STEPS][BLOCK];       // its chord
    SegDesc pf[BLOCK];
    int endc[BLOCK][3];
    int gb[3], gn[3], gs[3];
    int anchor[3];
    int gmode;  // 1: grid in smem, 2: grid in global memory, 0: hash only
};

// Axis choice of traversal._walk_grid (axis = 0; if t[1] < t[0]: 1; if
// t[2] < t[axis]: 2), the chosen t_max value (walk()'s `ta`) and the
// t_max[axis] += t_delta[axis] update: dda_advance plus the selected value.
__device__ __forceinline__ int dda_advance_t(double &tx, double &ty, double &tz, double dx,
                                             double dy, double dz, double &ta) {
    int ax;
    asm("{\n\t.reg .pred py, pzx, pzy, pz, qx, qy, t0;\n\t"
        "setp.lt.f64 py, %1, %0;\n\t"
        "setp.lt.f64 pzx, %2, %0;\n\t"
        "setp.lt.f64 pzy, %2, %1;\n\t"
        "and.pred t0, py, pzy;\n\t"
        "not.pred qx, py;\n\t"
        "and.pred qx, qx, pzx;\n\t"
        "or.pred pz, t0, qx;\n\t"
        "selp.f64 %4, %1, %0, py;\n\t"
        "@pz mov.f64 %4, %2;\n\t"
        "not.pred t0, pz;\n\t"
        "and.pred qy, py, t0;\n\t"
        "not.pred qx, py;\n\t"
        "and.pred qx, qx, t0;\n\t"
        "@qx add.rn.f64 %0, %0, %5;\n\t"
        "@qy add.rn.f64 %1, %1, %6;\n\t"
        "@pz add.rn.f64 %2, %2, %7;\n\t"
        "selp.b32 %3, 1, 0, qy;\n\t"
        "@pz mov.b32 %3, 2;\n\t"
        "}"
        : "+d"(tx), "+d"(ty), "+d"(tz), "=r"(ax), "=d"(ta)
        : "d"(dx), "d"(dy), "d"(dz));
    return ax;
}

// region slot (and Gaussian brick summary) for grid-relative coordinates rp
__device__ __noinline__ int wn_slow_region(const DevMap &m, const WalkNdtSmem &sm, unsigned rp,
                                           unsigned *gm) {
    const int rx = sm.gb[0] + (int)(rp & 1023u) - RP_BIAS;
    const int ry = sm.gb[1] + (int)((rp >> 10) & 1023u) - RP_BIAS;
    const int rz = sm.gb[2] + (int)(rp >> 20) - RP_BIAS;
    const unsigned ux = (unsigned)(rx - sm.gb[0]), uy = (unsigned)(ry - sm.gb[1]),
                   uz = (unsigned)(rz - sm.gb[2]);
    if (sm.gmode && ux < (unsigned)sm.gn[0] && uy < (unsigned)sm.gn[1] && uz < (unsigned)sm.gn[2]) {
        const int gi = ux + sm.gs[1] * uy + sm.gs[2] * uz;
        const int s = sm.gmode == 1 ? sm.grid[gi].x : __ldg(m.rgrid + gi);
        if (s >= 0 && s < m.cap) {
            *gm = sm.gmode == 1 ? (unsigned)sm.grid[gi].y : __ldg(m.gmask + s);
            return s;
        }
    }
    const int slot = region_slot_inl(m, pack_region(rx, ry, rz));
    *gm = slot >= 0 && slot < m.cap ? __ldcg(m.gmask + slot) : 0xFFFFFFFFu;
    if (slot >= 0 && slot < m.cap && stamp_epoch(m.slot_touch + slot, m.epoch)) {
        const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
        if (t < (unsigned long long)m.touched_cap) m.touched[t] = slot;
    }
    return slot;
}

template <int DIM>
__device__ __noinline__ unsigned wn_vid_of(const DevMap &m, const WalkNdtSmem &sm, int gx, int gy,
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

// DIM: compile-time region edge (32), or 0 for any other region_dim
template <class Src, int DIM = 0>
__global__ void __launch_bounds__(BLOCK, WN_BLOCKS) k_walk_ndt_det(const __grid_constant__ DevMap m,
                                                                   Src src) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WalkNdtSmem &sm = *reinterpret_cast<WalkNdtSmem *>(smem_raw);
    if (!read_go(m) || !walk_det_ok(m)) return;
    const unsigned long long nseg_total =
        min(*((volatile unsigned long long *)(m.stats + S_SEGDESC)), m.seg_cap);
    const bool have_grid = *((volatile unsigned long long *)(m.stats + S_RGRID)) != 0;
    const bool bricks = m.brick_shift >= 0 && m.gmask;
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
                sm.anchor[a] = r0[a] * m.dim + (int)((d0.lp0 >> (10 * a)) & 1023u) - 1 - NCUBE / 2;
        } else {
            sm.anchor[0] = sm.anchor[1] = sm.anchor[2] = 1 << 29;
        }
    }
    __syncthreads();
    if (sm.gmode == 1) {
        const int ncell = sm.gn[0] * sm.gn[1] * sm.gn[2];
        for (int k = threadIdx.x; k < ncell; k += blockDim.x) {
            const int sl = m.rgrid[k];
            sm.grid[k] = make_int2(sl, !bricks ? -1 : (sl >= 0 && sl < m.cap ? (int)__ldcg(m.gmask + sl) : 0));
        }
    }
    __syncthreads();
    unsigned *const scr = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);
    const unsigned *const cntl = reinterpret_cast<const unsigned *>(m.slab[L_COUNT]);
    {
        // the cube's Gaussian bitmap: every voxel id first, then all count
        // loads in flight together, one ballot per 32 cells
        constexpr int PER = NCUBE_N / BLOCK;
        unsigned vid[PER], c[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int k = threadIdx.x + j * BLOCK;
            vid[j] = wn_vid_of<DIM>(m, sm, sm.anchor[0] + k % NCUBE, sm.anchor[1] + (k / NCUBE) % NCUBE,
                               sm.anchor[2] + k / (NCUBE * NCUBE), false);
            sm.cube[k] = 0u;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) c[j] = vid[j] != 0xFFFFFFFFu ? __ldcg(cntl + vid[j]) : 0u;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const unsigned word = __ballot_sync(0xffffffffu, c[j] >= 3u);
            if ((threadIdx.x & 31) == 0) sm.cgauss[(threadIdx.x + j * BLOCK) >> 5] = word;
        }
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const int dim = DIM ? DIM : m.dim;
    const unsigned vpr = DIM ? (unsigned)(DIM * DIM * DIM) : (unsigned)m.vpr;
    unsigned long long *const wkey = sm.wkey[threadIdx.x >> 5];
    double2 *const wt = sm.wt[threadIdx.x >> 5];
    unsigned wcnt = 0, wflushed = 0;  // warp-uniform record ring counters
    unsigned rmiss = 0, visits = 0;

    // segment state
    double tx = 0, ty = 0, tz = 0, dx = 0, dy = 0, dz = 0, tprev = 0;
    unsigned lp = 0, rp = 0, vbase = 0xFFFFFFFFu, oi = 0, cp = 0, gm = 0;
    bool sample = false;
    int li = 0, gi = 0, rem = 0;
    int dli0 = 0, dli1 = 0, dli2 = 0;       // DIM != 32
    unsigned dlp0 = 0, dlp1 = 0, dlp2 = 0;  // DIM != 32
    unsigned sg3 = 0;  // DIM 32: the step direction codes, 2 bits per axis (step + 1)
    bool active = false, in_cube = false, ingrid = false;
    int parked = 0;  // 1: region lookup after a crossing, 2: fallback jump to the end cell
    bool jumped = false;
    unsigned live = 0, sure = 0;  // candidate slots of the window; known Gaussian (cube)
    bool pf_valid = false, exhausted = false;
    unsigned pool_next = 0, pool_end = 0;
    SegDesc *my_pf = &sm.pf[threadIdx.x];

    auto push_records = [&](bool rec, unsigned long long key, double2 t) {
        const unsigned rb = __ballot_sync(0xffffffffu, rec);
        if (!rb) return;
        if (rec) {
            const unsigned k = (wcnt + __popc(rb & lanemask_lt)) & (WN_WBUF - 1);
            wkey[k] = key;
            wt[k] = t;
        }
        wcnt += __popc(rb);
        if (wcnt - wflushed >= 32) {
            __syncwarp();
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(m.stats + S_RECORDS, 32ULL);
            b = __shfl_sync(0xffffffffu, b, 0);
            const unsigned k = (wflushed + lane) & (WN_WBUF - 1);
            if (b + lane < m.rec_cap) {
                m.rec[b + lane] = wkey[k];
                m.rec_t[b + lane] = wt[k];
            }
            wflushed += 32;
            __syncwarp();
        }
    };

    auto set_region = [&](int s, unsigned g) {
        vbase = s >= 0 && s < m.cap ? (unsigned)s * vpr : 0xFFFFFFFFu;
        gm = bricks ? g : 0xFFFFFFFFu;
    };

    auto start = [&]() {
        __pipeline_wait_prior(0);
        const SegDesc &d = *my_pf;
        tx = d.t[0]; ty = d.t[1]; tz = d.t[2];
        dx = d.d[0]; dy = d.d[1]; dz = d.d[2];
        tprev = 0.0;
        const unsigned codes = d.flags;
        oi = d.order >> 1;
        sample = codes & 1u;
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
            unsigned g = 0xFFFFFFFFu;
            if (ingrid) {
                if (sm.gmode == 1) {
                    const int2 ge = sm.grid[gi];
                    s = ge.x;
                    g = (unsigned)ge.y;
                } else {
                    s = __ldg(m.rgrid + gi);
                    if (s >= 0 && s < m.cap) g = __ldg(m.gmask + s);
                }
            }
            if (s < 0) s = wn_slow_region(m, sm, rp, &g);
            set_region(s, g);
        }
        sm.endc[threadIdx.x][0] = d.e[0];
        sm.endc[threadIdx.x][1] = d.e[1];
        sm.endc[threadIdx.x][2] = d.e[2];
        const unsigned ux = (unsigned)(r0[0] * dim + (int)(lp & 1023u) - 1 - sm.anchor[0]);
        const unsigned uy = (unsigned)(r0[1] * dim + (int)((lp >> 10) & 1023u) - 1 - sm.anchor[1]);
        const unsigned uz = (unsigned)(r0[2] * dim + (int)(lp >> 20) - 1 - sm.anchor[2]);
        in_cube = (ux | uy | uz) < (unsigned)NCUBE;
        cp = ux | (uy << 8) | (uz << 16);
        pf_valid = false;
        active = true;
        jumped = false;
    };

    // one DDA step = one voxel visit into in-flight slot Q
    auto step = [&](const int Q) {
        if (!active) return;
        const bool last = rem == 0;
        if (last && !jumped) {
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
        // the visit's chord (walk(): tn = ta clamped to [tprev, 1]; 1 on the last visit)
        int ax = 0;
        double tn = 1.0;
        if (!last) {
            double ta;
            ax = dda_advance_t(tx, ty, tz, dx, dy, dz, ta);
            tn = ta < tprev ? tprev : ta;
            tn = tn > 1.0 ? 1.0 : tn;
        }
        // ---- the visit ----
        if (!(last && sample)) {  // the sample voxel itself: phase 2 (k_discover's record)
            const unsigned vid = vbase + (unsigned)li;
            if (vbase != 0xFFFFFFFFu) {
                if (in_cube) {
                    const unsigned ck = ncube_cell(cp);
                    if ((sm.cgauss[ck >> 5] >> (ck & 31)) & 1u) {
                        sm.vids[Q][threadIdx.x] = vid;
                        sm.tv[Q][threadIdx.x] = make_double2(tprev, tn);
                        live |= 1u << Q;
                        sure |= 1u << Q;
                    } else {
                        atomicAdd(sm.cube + ck, 1u);
                    }
                } else if ((gm >> wd_brick<DIM>(li, m.bsh)) & 1u) {
                    sm.vids[Q][threadIdx.x] = vid;
                    sm.tv[Q][threadIdx.x] = make_double2(tprev, tn);
                    live |= 1u << Q;
                } else {
                    red_add(scr + vid, 1u);
                }
            } else {
                ++rmiss;
            }
        }
        if (last) {
            active = false;
            return;
        }
        tprev = tn;
        --rem;
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
            cp += (unsigned)sgn << (8 * ax);
            in_cube = (cp & NCUBE_OUT) == 0;
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
            unsigned g = 0xFFFFFFFFu;
            if (ingrid) {
                if (sm.gmode == 1) {
                    const int2 ge = sm.grid[gi];
                    s = ge.x;
                    g = (unsigned)ge.y;
                } else {
                    s = __ldg(m.rgrid + gi);
                    if (s >= 0 && s < m.cap) g = __ldg(m.gmask + s);
                }
            }
            if (s >= 0) {
                set_region(s, g);
            } else {
                parked = 1;
                active = false;
            }
        }
    };

    auto unpark = [&]() {
        if (parked == 1) {
            unsigned g = 0xFFFFFFFFu;
            const int s = wn_slow_region(m, sm, rp, &g);
            set_region(s, g);
        } else if (parked == 2) {
            const unsigned vid = wn_vid_of<DIM>(m, sm, sm.endc[threadIdx.x][0], sm.endc[threadIdx.x][1],
                                           sm.endc[threadIdx.x][2], true);
            vbase = vid == 0xFFFFFFFFu ? vid : vid - vid % vpr;
            li = vid == 0xFFFFFFFFu ? 0 : (int)(vid % vpr);
            gm = 0xFFFFFFFFu;  // the end voxel is a candidate
            in_cube = false;
            jumped = true;
        }
        parked = 0;
        active = true;
    };

    for (;;) {
        // ---- retire the window: candidates become records or miss counts ----
        if (__any_sync(0xffffffffu, live != 0u)) {
            unsigned w[WN_STEPS], v[WN_STEPS];
            const unsigned need = live & ~sure;
#pragma unroll
            for (int q = 0; q < WN_STEPS; ++q) {
                w[q] = 0u;
                v[q] = 0u;
                if ((live >> q) & 1u) v[q] = sm.vids[q][threadIdx.x];
                if ((need >> q) & 1u) w[q] = __ldcg(cntl + v[q]);
            }
            // candidates without a Gaussian: the delayed miss count
            unsigned recm = 0u;
#pragma unroll
            for (int q = 0; q < WN_STEPS; ++q) {
                const bool cand = (live >> q) & 1u;
                const bool rec = cand && (((sure >> q) & 1u) || w[q] >= 3u);
                if (cand && !rec) red_add(scr + v[q], 1u);
                recm |= (unsigned)rec << q;
            }
            // phase-1 records: only the steps some lane holds one (warp-uniform)
            const unsigned wrec = __reduce_or_sync(0xffffffffu, recm);
            if (wrec) {
#pragma unroll
                for (int q = 0; q < WN_STEPS; ++q) {
                    if (!((wrec >> q) & 1u)) continue;
                    const bool rec = (recm >> q) & 1u;
                    unsigned long long key = 0;
                    double2 t = make_double2(0.0, 0.0);
                    if (rec) {
                        const int s = (int)(v[q] / vpr), l = (int)(v[q] % vpr);
                        key = ndt_key(ndt_index(m, s, l), 0u, oi);
                        t = sm.tv[q][threadIdx.x];
                    }
                    push_records(rec, key, t);
                }
            }
            live = 0u;
            sure = 0u;
        }
        if (parked) unpark();
        if (!active && pf_valid) start();
        // ---- claim work for lanes without a prefetched descriptor ----
        unsigned needw = __ballot_sync(0xffffffffu, !pf_valid && !exhausted);
        while (needw) {
            if (pool_next >= pool_end) {
                unsigned b = 0;
                if (lane == 0) b = (unsigned)atomicAdd(m.work, 32ULL);
                b = __shfl_sync(0xffffffffu, b, 0);
                pool_next = b;
                pool_end = b + 32;
                if (b >= nseg_total) {
                    if ((needw >> lane) & 1u) exhausted = true;
                    break;
                }
            }
            const unsigned avail = pool_end - pool_next;
            const unsigned rank = __popc(needw & lanemask_lt);
            const bool served = ((needw >> lane) & 1u) && rank < avail;
            if (served) {
                const unsigned long long wi = (unsigned long long)pool_next + rank;
                if (wi < nseg_total) {
                    const char *g = reinterpret_cast<const char *>(m.segs + m.perm[wi]);
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
            needw &= ~served_mask;
        }
        if (!__any_sync(0xffffffffu, active || pf_valid || !exhausted || parked)) break;
        if (!__any_sync(0xffffffffu, active)) continue;
#pragma unroll 1
        for (int q = 0; q < WN_STEPS; ++q) step(q);
    }
    // flush the warp's remaining records
    __syncwarp();
    {
        const unsigned left = wcnt - wflushed;
        if (left) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(m.stats + S_RECORDS, (unsigned long long)left);
            b = __shfl_sync(0xffffffffu, b, 0);
            const unsigned k = (wflushed + lane) & (WN_WBUF - 1);
            if ((unsigned)lane < left && b + lane < m.rec_cap) {
                m.rec[b + lane] = wkey[k];
                m.rec_t[b + lane] = wt[k];
            }
        }
    }
    __syncthreads();
    unsigned long long flushed = 0;
    for (int k = threadIdx.x; k < NCUBE_N; k += blockDim.x) {
        const unsigned c = sm.cube[k];
        if (!c) continue;
        ++flushed;
        const unsigned vid = wn_vid_of<DIM>(m, sm, sm.anchor[0] + k % NCUBE,
                                       sm.anchor[1] + (k / NCUBE) % NCUBE,
                                       sm.anchor[2] + k / (NCUBE * NCUBE), true);
        if (vid != 0xFFFFFFFFu) red_add(scr + vid, c);
    }
    unsigned long long st[3] = {visits, rmiss, flushed};
    const int which[3] = {S_VISITS, S_RMISS, S_CUBE_FLUSH};
    block_add_stats(m, st, which);
}

}  // namespace vm
