// vm_compat.cuh -- one-to-one device replacement of the reference's
// `_kernels.integrate_occupancy` (_kernels.pyx:376-470).
//
// Same argument meaning as the Cython entry point: a chunk of pre-built
// segments (engine._segment_arrays, engine.py:153-162), the open-addressing
// region table of engine._build_region_table (engine.py:121-147) and
// per-layer arrays of per-region buffer pointers -- except every array is a
// device array.  One thread per segment; the walk is the exact fp64 DDA
// (walk_fill, _kernels.pyx:134-211) and every visit does the reference's
// clamped CAS log-odds update (:233-271), the native packed-mean fold with
// its `* (1 / (n + 1))` weight (:318-357) and the decay accumulators
// (:460-466).  The table is probed only when the walk crosses a region face
// (the reference probes on every visit; the table is read-only during the
// call, so the answers are identical).  There is no mutex fallback on the
// GPU: retries are counted, cas_failures stays 0.
#pragma once

#include "vm_kernels.cuh"

namespace vm {

struct CompatArgs {
    const double *o, *e;
    const unsigned char *has;
    long long n;
    const long long *tkeys;
    const int *tvals;
    unsigned long long tmask;
    void *const *occ, *const *mean, *const *cnt, *const *dhit, *const *ddist;
    double vox;
    int dim;
    float hit, miss, cmin, cmax;
    int walk_cap;
    unsigned long long *stats;  // retries, failures, region_misses, visits
};

// _kernels.pyx:113-124 (table_lookup): linear probing, -1 = empty
__device__ __forceinline__ int compat_lookup(const CompatArgs &a, long long key) {
    unsigned long long h = mix_key(key) & a.tmask;
    for (unsigned long long p = 0; p <= a.tmask; ++p) {
        const long long k = a.tkeys[h];
        if (k == key) return a.tvals[h];
        if (k == -1) return -1;
        h = (h + 1) & a.tmask;
    }
    return -1;
}

// _kernels.pyx:318-357 exactly (native weight form)
__device__ __forceinline__ unsigned compat_mean(unsigned *mean, unsigned *cnt, const double off[3]) {
    const unsigned n_old = atomicAdd(cnt, 1u);
    if (n_old == 0xFFFFFFFFu) {
        atomicExch(cnt, 0xFFFFFFFFu);
        return 0;
    }
    const double w = 1.0 / ((double)n_old + 1.0);
    unsigned retries = 0;
    unsigned old = __ldcg(mean);
    for (;;) {
        double mv[3];
        if (n_old == 0) {
            mv[0] = off[0]; mv[1] = off[1]; mv[2] = off[2];
        } else {
            unpack_mean(old, mv);
#pragma unroll
            for (int q = 0; q < 3; ++q) mv[q] = mv[q] + (off[q] - mv[q]) * w;
        }
        const unsigned nb = pack_mean(mv);
        const unsigned prev = atomicCAS(mean, old, nb);
        if (prev == old) return retries;
        old = prev;
        ++retries;
    }
}

struct CompatVisitor {
    const CompatArgs *a;
    int rx, ry, rz, lx, ly, lz, slot;
    double ex, ey, ez, length;
    bool has;
    unsigned long long retries, rmiss;

    __device__ __forceinline__ void locate(int x, int y, int z) {
        rx = floordiv(x, a->dim);
        ry = floordiv(y, a->dim);
        rz = floordiv(z, a->dim);
        lx = x - rx * a->dim;
        ly = y - ry * a->dim;
        lz = z - rz * a->dim;
        slot = compat_lookup(*a, pack_region(rx, ry, rz));
    }
    __device__ __forceinline__ void begin(int x, int y, int z) { locate(x, y, z); }
    __device__ __forceinline__ void jump(int x, int y, int z) { locate(x, y, z); }
    __device__ __forceinline__ void moved(int axis, int s) {
        int *l = axis == 0 ? &lx : (axis == 1 ? &ly : &lz);
        int *r = axis == 0 ? &rx : (axis == 1 ? &ry : &rz);
        const int nl = *l + s;
        if (nl >= 0 && nl < a->dim) {
            *l = nl;
            return;
        }
        *l = nl < 0 ? a->dim - 1 : 0;
        *r += s;
        slot = compat_lookup(*a, pack_region(rx, ry, rz));
    }
    __device__ __forceinline__ void visit(int x, int y, int z, double t0, double t1, bool last) {
        if (slot < 0) {
            ++rmiss;
            return;
        }
        const int li = lx + a->dim * (ly + a->dim * lz);
        const bool hit = has && last;
        unsigned *occ = reinterpret_cast<unsigned *>(a->occ[slot]) + li;
        const float d = hit ? a->hit : a->miss;
        unsigned old = __ldcg(occ);
        for (;;) {
            const unsigned nb = __float_as_uint(clamp_add(__uint_as_float(old), d, a->cmin, a->cmax));
            const unsigned prev = atomicCAS(occ, old, nb);
            if (prev == old) break;
            old = prev;
            ++retries;
        }
        if (hit && a->mean) {
            const double off[3] = {ex / a->vox - (double)x, ey / a->vox - (double)y,
                                   ez / a->vox - (double)z};
            retries += compat_mean(reinterpret_cast<unsigned *>(a->mean[slot]) + li,
                                   reinterpret_cast<unsigned *>(a->cnt[slot]) + li, off);
        }
        if (a->dhit) {
            red_add(reinterpret_cast<double *>(a->ddist[slot]) + li, (t1 - t0) * length);
            if (hit) red_add(reinterpret_cast<unsigned *>(a->dhit[slot]) + li, 1u);
        }
    }
};

__global__ void __launch_bounds__(BLOCK) k_compat_occupancy(const __grid_constant__ CompatArgs a) {
    unsigned long long visits = 0;
    CompatVisitor v;
    v.a = &a;
    v.retries = v.rmiss = 0;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < a.n;
         r += (long long)gridDim.x * blockDim.x) {
        const double o[3] = {a.o[3 * r], a.o[3 * r + 1], a.o[3 * r + 2]};
        const double e[3] = {a.e[3 * r], a.e[3 * r + 1], a.e[3 * r + 2]};
        // _kernels.pyx:432: naive sqrt of the squared differences (no FMA)
        const double dx = e[0] - o[0], dy = e[1] - o[1], dz = e[2] - o[2];
        v.length = sqrt(dx * dx + dy * dy + dz * dz);
        v.ex = e[0];
        v.ey = e[1];
        v.ez = e[2];
        v.has = a.has[r] != 0;
        // walk_fill returns -1 (segment skipped) when it needs more than cap
        // visits; the visit count is the Manhattan distance between the end
        // cells + 1
        long long need = 1;
#pragma unroll
        for (int q = 0; q < 3; ++q)
            need += llabs((long long)floor(o[q] / a.vox) - (long long)floor(e[q] / a.vox));
        if (need > a.walk_cap) continue;
        visits += (unsigned long long)need;
        walk(o, e, a.vox, v);
    }
    unsigned long long st[3] = {v.retries, v.rmiss, visits};
    const int which[3] = {0, 2, 3};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        unsigned long long x = st[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(a.stats + which[i], x);
    }
}

}  // namespace vm
