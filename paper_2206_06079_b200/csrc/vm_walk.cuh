// vm_walk.cuh -- the persistent occupancy/decay walk (the hot kernel).
//
// One warp = 32 independent walkers over the batch's preprocessed segments
// (SegDesc, written by k_discover with the DDA initial state).  Every loop
// iteration each active lane takes exactly one DDA step of its segment
// (traversal.py:80-111) = one voxel visit:
//
//   * the end test is `remaining == 0` (exact: Manhattan distance to the
//     end cell never drops below `remaining`, so cur == last can only hold
//     there; otherwise it is the numerical-fallback jump);
//   * local/region coordinates advance incrementally; a region crossing is
//     one shared-memory load from the dense per-batch region grid
//     (slot | 32-bit brick summary of sample voxels), hash probe only for
//     regions outside it;
//   * deterministic mode: a visit whose brick holds no sample voxel is a
//     miss with the identical delta: +1 in the block's smem cube (voxels
//     around the sensor) or RED.ADD into the scratch layer, finished at
//     once.  A visit in a marked brick issues the mark-word / marked-index
//     loads and is finished one iteration later (software pipeline), when
//     it becomes an order-keyed record if the voxel is a sample voxel.
//   * CAS mode: the paper's clamped atomicCAS update (load issued one
//     iteration ahead).
//
// Lanes whose segment ends swap in the descriptor they prefetched into
// their own smem slot (cp.async); work is pulled 32 segments at a time.
#pragma once

#include <cuda_pipeline.h>

#include "vm_kernels.cuh"

namespace vm {

constexpr int WK_STAGE = 3072;  // staged records per block (24 KiB)
constexpr int RG_MAX = 4096;    // dense region grid cells held in smem (32 KiB)
constexpr int WK_INNER = 8;     // DDA steps between warp-level work bookkeeping

struct WalkSmem {
    unsigned cube[CUBE_N];
    unsigned long long grid[RG_MAX];
    unsigned long long rec[WK_STAGE];
    SegDesc pf[BLOCK];
    int gb[3], gn[3];      // grid origin / extents (regions); gn[0] = 0: no grid
    int anchor[3];         // cube corner (voxels)
    int nrec;
    unsigned long long rec_base;
};

// brick of a local coordinate: 4 x 4 x 2 bricks (32 bits) for power-of-two dims
__device__ __forceinline__ int brick32(int lx, int ly, int lz, int bs) {
    return (lx >> bs) | ((ly >> bs) << 2) | ((lz >> (bs + 1)) << 4);
}

// slot (low 32 bits, signed) + brick summary (high 32 bits) of region r
struct GridView {
    int b0, b1, b2, n0, n1, n2;
};

__device__ __forceinline__ unsigned long long region_entry(const DevMap &m, const WalkSmem &sm,
                                                           const GridView &gv, int rx, int ry,
                                                           int rz) {
    const int ux = rx - gv.b0, uy = ry - gv.b1, uz = rz - gv.b2;
    if ((unsigned)ux < (unsigned)gv.n0 && (unsigned)uy < (unsigned)gv.n1 &&
        (unsigned)uz < (unsigned)gv.n2) {
        const unsigned long long e = sm.grid[ux + gv.n0 * (uy + gv.n1 * uz)];
        if ((int)(unsigned)e >= 0) return e;
    }
    const int slot = region_slot(m, pack_region(rx, ry, rz));
    unsigned bm = 0xFFFFFFFFu;
    if (slot >= 0 && slot < m.cap) {
        bm = (unsigned)m.bmask[slot];
        // regions reached outside the dense grid are resolved from the touched list
        if (atomicExch(m.slot_touch + slot, m.epoch) != m.epoch) {
            const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
            if (t < (unsigned long long)m.touched_cap) m.touched[t] = slot;
        }
    }
    return ((unsigned long long)bm << 32) | (unsigned)slot;
}

template <int MODE, bool DET, bool REC_ONLY, class Src>
__global__ void __launch_bounds__(BLOCK, 2) k_walk(const __grid_constant__ DevMap m, Src src) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WalkSmem &sm = *reinterpret_cast<WalkSmem *>(smem_raw);
    if (!read_go(m)) return;
    const unsigned long long nseg_total =
        min(*((volatile unsigned long long *)(m.stats + S_SEGDESC)), m.seg_cap);
    for (int k = threadIdx.x; k < CUBE_N; k += blockDim.x) sm.cube[k] = 0;
    const bool have_grid = *((volatile unsigned long long *)(m.stats + S_RGRID)) != 0;
    if (threadIdx.x == 0) {
        sm.nrec = 0;
        for (int a = 0; a < 3; ++a) {
            sm.gb[a] = m.rbox[a];
            sm.gn[a] = have_grid ? m.rbox[3 + a] - m.rbox[a] + 1 : 0;
            sm.anchor[a] = nseg_total ? m.segs[0].c[a] - CUBE / 2 : (1 << 29);
        }
    }
    __syncthreads();
    const int ncell = sm.gn[0] * sm.gn[1] * sm.gn[2];
    for (int k = threadIdx.x; k < ncell; k += blockDim.x) {
        const int s = m.rgrid[k];
        unsigned bm = 0xFFFFFFFFu;
        if (s >= 0 && s < m.cap) bm = (unsigned)m.bmask[s];
        sm.grid[k] = ((unsigned long long)bm << 32) | (unsigned)s;
    }
    __syncthreads();

    const int c0 = sm.anchor[0], c1 = sm.anchor[1], c2 = sm.anchor[2];
    const GridView gv{sm.gb[0], sm.gb[1], sm.gb[2], sm.gn[0], sm.gn[1], sm.gn[2]};
    const int lane = threadIdx.x & 31;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const int dim = m.dim, bs = m.brick_shift, cap = m.cap;
    const unsigned long long vpr = (unsigned long long)m.vpr;
    float *const occ_base = reinterpret_cast<float *>(m.slab[L_OCC]);
    unsigned *const scr_base = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);

    unsigned long long visits = 0, rmiss = 0, retries = 0;
    // segment state
    double tx = 0, ty = 0, tz = 0, dx = 0, dy = 0, dz = 0, tprev = 0, L = 0;
    int cx = 0, cy = 0, cz = 0, ex = 0, ey = 0, ez = 0, remaining = 0;
    int lx = 0, ly = 0, lz = 0, rx = 0, ry = 0, rz = 0;
    unsigned codes = 0, order = 0, bm = 0;
    int cube_left = 0;          // steps the segment may still spend in the smem cube
    bool active = false;
    // current region: base pointers (null when the region is unavailable)
    unsigned *scr_r = nullptr;
    float *occ_r = nullptr;
    const unsigned *mk_r = nullptr;
    int slot = -1;
    // pipelined visit (issued loads, finished next step)
    bool pend = false;
    unsigned *p_scr = nullptr;  // counter word (det) / log-odds word (cas)
    unsigned p_key = 0, p_w1 = 0, p_w2 = 0, p_bit = 0;
    int p_cube = -1;
    // prefetch + warp work pool
    bool pf_valid = false, exhausted = false;
    unsigned long long pool_next = 0, pool_end = 0;
    SegDesc *my_pf = &sm.pf[threadIdx.x];

    auto set_region = [&](unsigned long long e) {
        slot = (int)(unsigned)e;
        bm = (unsigned)(e >> 32);
        if ((unsigned)slot < (unsigned)cap) {
            const unsigned long long base = (unsigned long long)slot * vpr;
            scr_r = scr_base + base;
            occ_r = occ_base + base;
            mk_r = m.marks + (size_t)slot * m.mark_words;
        } else {
            scr_r = nullptr;
        }
    };

    for (;;) {
        // ---- claim work for lanes without a prefetched descriptor ----
        unsigned need = __ballot_sync(0xffffffffu, !pf_valid && !exhausted);
        while (need) {
            if (pool_next >= pool_end) {
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(m.work, 32ULL);
                b = __shfl_sync(0xffffffffu, b, 0);
                pool_next = b;
                pool_end = b + 32;
                if (b >= nseg_total) {
                    if ((need >> lane) & 1u) exhausted = true;
                    break;
                }
            }
            const unsigned long long avail = pool_end - pool_next;
            const unsigned rank = __popc(need & lanemask_lt);
            const bool served = ((need >> lane) & 1u) && rank < avail;
            if (served) {
                const unsigned long long idx = pool_next + rank;
                if (idx < nseg_total) {
                    const char *g = reinterpret_cast<const char *>(m.segs + idx);
#pragma unroll
                    for (int q = 0; q < 7; ++q)
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
        if (!__any_sync(0xffffffffu, active || pf_valid || !exhausted || pend)) break;

        // ---- up to WK_INNER steps without warp-level bookkeeping ----
#pragma unroll 1
        for (int inner = 0; inner < WK_INNER; ++inner) {
            // idle lanes start their prefetched segment
            if (!active && pf_valid) {
                __pipeline_wait_prior(0);
                const SegDesc &d = *my_pf;
                tx = d.t[0]; ty = d.t[1]; tz = d.t[2];
                dx = d.d[0]; dy = d.d[1]; dz = d.d[2];
                cx = d.c[0]; cy = d.c[1]; cz = d.c[2];
                ex = d.e[0]; ey = d.e[1]; ez = d.e[2];
                codes = d.flags;
                order = d.order;
                L = d.L;
                lx = (int)(d.local0 & 1023u);
                ly = (int)((d.local0 >> 10) & 1023u);
                lz = (int)(d.local0 >> 20);
                rx = d.r0[0]; ry = d.r0[1]; rz = d.r0[2];
                tprev = 0.0;
                remaining = abs(cx - ex) + abs(cy - ey) + abs(cz - ez);
                set_region(region_entry(m, sm, gv, rx, ry, rz));
                // a straight segment leaves the (convex) cube within 3*CUBE steps
                // and never re-enters it
                const unsigned ux = (unsigned)(cx - c0), uy = (unsigned)(cy - c1),
                               uz = (unsigned)(cz - c2);
                cube_left = (ux | uy | uz) < (unsigned)CUBE ? 3 * CUBE : 0;
                pf_valid = false;
                active = true;
            }
            // finish the visit pipelined from the previous step
            if (pend) {
                pend = false;
                if (DET) {
                    if (p_w1 & p_bit) {
                        const unsigned long long key =
                            ((unsigned long long)(p_w2 & ~MARK_FLAG) << m.order_bits) | p_key;
                        const int k = atomicAdd(&sm.nrec, 1);
                        if (k < WK_STAGE) {
                            sm.rec[k] = key;
                        } else {
                            const unsigned long long g = atomicAdd(m.stats + S_RECORDS, 1ULL);
                            if (g < m.rec_cap) m.rec[g] = key;
                        }
                    } else if (!REC_ONLY) {
                        if (p_cube >= 0) atomicAdd(sm.cube + p_cube, 1u);
                        else red_add(p_scr, 1u);
                    }
                } else {
                    unsigned old = p_w1;
                    for (;;) {
                        const unsigned nb = __float_as_uint(
                            clamp_add(__uint_as_float(old), m.miss32, m.cmin, m.cmax));
                        if (nb == old) break;
                        const unsigned prev = atomicCAS(p_scr, old, nb);
                        if (prev == old) break;
                        old = prev;
                        ++retries;
                    }
                }
            }
            if (!active) continue;

            // ---- one DDA step = one voxel visit ----
            const bool last = remaining == 0;
            if (last && !(cx == ex && cy == ey && cz == ez)) {
                // numerical fallback: the walk jumps to the end cell (traversal.py:88-92)
                cx = ex;
                cy = ey;
                cz = ez;
                rx = floordiv(cx, dim);
                ry = floordiv(cy, dim);
                rz = floordiv(cz, dim);
                lx = cx - rx * dim;
                ly = cy - ry * dim;
                lz = cz - rz * dim;
                set_region(region_entry(m, sm, gv, rx, ry, rz));
                cube_left = 1;
            }
            // axis = 0; if tmax[1] < tmax[axis]: 1; if tmax[2] < tmax[axis]: 2
            const bool py = ty < tx;
            const double ta = py ? ty : tx;
            const bool pz = tz < ta;
            double t1 = 1.0;
            if (MODE == M_DECAY && !last) {
                t1 = pz ? tz : ta;
                if (t1 < tprev) t1 = tprev;
                if (t1 > 1.0) t1 = 1.0;
            }
            ++visits;
            if (!scr_r) {
                ++rmiss;
            } else {
                const int li = lx + dim * (ly + dim * lz);
                const bool hit = last && (codes & 1u);
                if (MODE == M_DECAY && !REC_ONLY) {
                    const unsigned long long vidx = (unsigned long long)slot * vpr + (unsigned)li;
                    red_add(reinterpret_cast<double *>(m.slab[L_DDIST]) + vidx, (t1 - tprev) * L);
                    if (hit) red_add(reinterpret_cast<unsigned *>(m.slab[L_DHITS]) + vidx, 1u);
                }
                int cube = -1;
                if (cube_left > 0) {
                    const unsigned ux = (unsigned)(cx - c0), uy = (unsigned)(cy - c1),
                                   uz = (unsigned)(cz - c2);
                    if ((ux | uy | uz) < (unsigned)CUBE) {
                        cube = (int)(ux + CUBE * (uy + CUBE * uz));
                        --cube_left;
                    } else {
                        cube_left = 0;  // left the cube for good
                    }
                }
                if (DET) {
                    const int b = bs >= 0 ? brick32(lx, ly, lz, bs) : 0;
                    if ((bm >> b) & 1u) {
                        pend = true;
                        p_scr = scr_r + li;
                        p_bit = 1u << (li & 31);
                        p_key = order | (hit ? 1u : 0u);
                        p_cube = cube;
                        p_w1 = __ldg(mk_r + ((unsigned)li >> 5));
                        p_w2 = __ldcg(scr_r + li);
                    } else if (!REC_ONLY) {
                        if (cube >= 0) atomicAdd(sm.cube + cube, 1u);
                        else red_add(scr_r + li, 1u);
                    }
                } else if (hit) {
                    float *p = occ_r + li;
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
                        const double off[3] = {e[0] / m.vox - (double)cx, e[1] / m.vox - (double)cy,
                                               e[2] / m.vox - (double)cz};
                        const unsigned long long vidx = (unsigned long long)slot * vpr + (unsigned)li;
                        retries += cas_mean(reinterpret_cast<unsigned *>(m.slab[L_MEAN]) + vidx,
                                            reinterpret_cast<unsigned *>(m.slab[L_COUNT]) + vidx, off);
                    }
                } else if (cube >= 0) {
                    atomicAdd(sm.cube + cube, 1u);
                } else {
                    pend = true;
                    p_scr = reinterpret_cast<unsigned *>(occ_r + li);
                    p_w1 = __float_as_uint(__ldcg(occ_r + li));
                }
            }
            if (last) {
                active = false;
                continue;
            }
            // ---- advance (t_max[axis] += t_delta[axis]), branch-free ----
            tprev = t1;
            --remaining;
            const bool ax = !py && !pz, ay = py && !pz;
            const int shift = pz ? 5 : (py ? 3 : 1);
            const int st = (int)((codes >> shift) & 3u) - 1;
            const double tn = (pz ? tz : ta) + (pz ? dz : (py ? dy : dx));
            tx = ax ? tn : tx;
            ty = ay ? tn : ty;
            tz = pz ? tn : tz;
            cx += ax ? st : 0;
            cy += ay ? st : 0;
            cz += pz ? st : 0;
            lx += ax ? st : 0;
            ly += ay ? st : 0;
            lz += pz ? st : 0;
            const int lnew = pz ? lz : (py ? ly : lx);
            if ((unsigned)lnew >= (unsigned)dim) {
                // region crossing (rare): wrap the local coordinate
                const int wrapped = st > 0 ? 0 : dim - 1;
                if (ax) { lx = wrapped; rx += st; }
                if (ay) { ly = wrapped; ry += st; }
                if (pz) { lz = wrapped; rz += st; }
                set_region(region_entry(m, sm, gv, rx, ry, rz));
            }
        }
    }

    __syncthreads();
    unsigned long long flushed = 0;
    if (!REC_ONLY) {
        for (int k = threadIdx.x; k < CUBE_N; k += blockDim.x) {
            const unsigned cntk = sm.cube[k];
            if (!cntk) continue;
            ++flushed;
            RegionTrack r2;
            r2.locate(m, c0 + k % CUBE, c1 + (k / CUBE) % CUBE, c2 + k / (CUBE * CUBE));
            const unsigned long long vidx = (unsigned long long)r2.slot * vpr + r2.li(m);
            if (DET) red_add(scr_base + vidx, cntk);
            else retries += cas_apply_k(occ_base + vidx, m.miss32, cntk, m.cmin, m.cmax);
        }
    }
    if (DET) {
        __syncthreads();
        const int nl = sm.nrec < WK_STAGE ? sm.nrec : WK_STAGE;
        if (threadIdx.x == 0 && nl)
            sm.rec_base = atomicAdd(m.stats + S_RECORDS, (unsigned long long)nl);
        __syncthreads();
        for (int k = threadIdx.x; k < nl; k += blockDim.x) {
            const unsigned long long ri = sm.rec_base + k;
            if (ri < m.rec_cap) m.rec[ri] = sm.rec[k];
        }
    }
    if (!REC_ONLY) {
        unsigned long long st[4] = {visits, rmiss, retries, flushed};
        const int which[4] = {S_VISITS, S_RMISS, S_RETRIES, S_CUBE_FLUSH};
        block_add_stats(m, st, which);
    }
}

}  // namespace vm
