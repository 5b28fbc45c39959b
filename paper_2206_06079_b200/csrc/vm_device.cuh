// vm_device.cuh -- device-side building blocks of the B200 ray-integration
// path: exact fp64 arithmetic of the reference, ray preprocessing, the DDA
// walker, the HBM region table and the per-block aggregation helpers.
//
// Every translation unit that includes this file is compiled with
// -fmad=false: the reference never fuses a*b+c (numpy ufuncs and CPython
// floats round each operation), so neither may we.  The single place the
// reference *does* fuse -- OpenBLAS ddot inside np.linalg.norm / `@`
// (traversal.py:40-42, reference.py:170) -- is written out with fma().
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace vm {

enum Layer {
    L_SCRATCH = 0,  // private: per-voxel miss counter (deterministic resolve)
    L_OCC = 1, L_MEAN = 2, L_COUNT = 3, L_COV = 4, L_HIT = 5, L_MISS = 6,
    L_INTENS = 7, L_DHITS = 8, L_DDIST = 9, L_TSDF = 10,
    L_NIDX = 11,    // private: per-voxel bucket index of the batch's ordered records
    L_NIDX2 = 12,   // private (NDT maps): the same for odd batches of a pipelined sequence
    NUM_LAYERS = 13
};

enum Mode { M_OCC = 0, M_DECAY = 1, M_NDT_OM = 2, M_NDT_TM = 3, M_TSDF = 4 };

enum Stat {
    S_RAYS_IN = 0, S_PROCESSED, S_SEGMENTS, S_VISITS, S_RETRIES, S_FAILURES,
    S_RMISS, S_PREF_TOUCHED, S_RECORDS, S_MARKED, S_WALK_TOUCHED, S_RANGE_ERR,
    S_CUBE_FLUSH, S_SEGDESC, S_WORK, S_RGRID, S_SPILLED, NUM_STATS
};

constexpr unsigned MARK_FLAG = 0x80000000u;
constexpr int SLOT_SPILLED = -3;         // region-table value of a region spilled to disk
constexpr int CUBE = 16;                 // smem aggregation cube edge (voxels)
constexpr int CUBE_N = CUBE * CUBE * CUBE;
constexpr int SLOTSET = 256;             // per-block region dedupe set
constexpr int RG_MAX = 1 << 16;
constexpr int SEG_BUCKETS = 64;          // step-count buckets of the walk's longest-first order
__host__ __device__ __forceinline__ int seg_bucket(unsigned rem) {
    const unsigned b = rem >> 4;
    return b < (unsigned)SEG_BUCKETS ? (int)b : SEG_BUCKETS - 1;
}          // dense per-batch region grid cells (HBM, L1-cached)

// One preprocessed segment with its DDA initial state (k_discover writes
// it, the persistent walk consumes it): 96 bytes, 16-byte aligned.
struct __align__(16) SegDesc {
    double t[3];       // t_max per axis at the start cell (traversal.py:70-78)
    double d[3];       // t_delta per axis
    long long rkey;    // packed region key of the start cell (keys.py:76-86)
    double L;          // segment length (RaySample.length), for decay
    unsigned order;    // (ray * maxseg + seg) << 1
    unsigned flags;    // bit0 has_sample (last visit is a hit), bits 1-6 step + 1 per axis
    unsigned rem;      // Manhattan distance start cell -> end cell
    unsigned lp0;      // start cell local coords, biased: (lx+1) | (ly+1) << 10 | (lz+1) << 20
    int slot0;         // region slot of the start cell
    int e[3];          // end cell (global)
};
static_assert(sizeof(SegDesc) == 96, "SegDesc layout");

// All state a kernel needs, passed by value.
struct DevMap {
    double vox, rsize;                   // voxel size, region size (region_dim * vox)
    double hit_delta, miss_delta;
    double max_range, seg_len;
    double tsdf_trunc, tsdf_maxw;
    double sigma2, miss_check;
    float hit32, miss32, cmin, cmax, fthresh;
    int dim, vpr, maxseg;
    int order_bits;                      // bits of (ray*maxseg+seg)<<1|hit
    int cell_limit;                      // |global voxel coord| must stay below
    // region table (engine._build_region_table format, engine.py:121-147)
    long long *tkeys;
    int *tvals;
    unsigned long long tmask;
    int *cursor;                         // regions allocated (dense slot ids)
    int cap;                             // slots backed by HBM
    int max_slots;                       // slot id space (slot_keys size)
    int insert;                          // lookups may create regions
    long long *slot_keys;
    unsigned *slot_touch, *slot_pref;
    unsigned epoch;
    void *const *lptr[NUM_LAYERS];       // per layer: region base pointer per slot
    char *slab[NUM_LAYERS];              // pool slabs: region s at slab + s * bpr
    unsigned long long bpr[NUM_LAYERS];  // bytes per region per layer
    int *rgrid;                          // dense region-slot grid over the batch bbox
    unsigned *bmask;                     // per slot: brick summary of the batch's sample voxels
    unsigned *gmask;                     // per slot (NDT maps): bricks that may hold a Gaussian
                                         // (count >= 3); set by the fold, conservative
    int brick_shift;                     // log2(dim) - 2 for power-of-two dims >= 4, else -1
    int bsh[3];                          // brick index from the local index li (see brick_of)
    int *rbox;                           // [6]: min xyz, max xyz (regions) of the batch
    int rg_max;                          // capacity of rgrid (cells)
    SegDesc *segs;                       // preprocessed segments of the batch
    unsigned *perm;                      // walk order of the segments (longest first)
    unsigned char *seg_bk;               // step-count bucket of each segment
    unsigned *seg_hist, *seg_cursor;     // [SEG_BUCKETS] counting-sort state
    unsigned long long seg_cap;
    unsigned long long *work;            // persistent-walk work counter
    unsigned long long *stats;
    int *go;                             // batch guard (0 = skip, replay later)
    int walk_det_launched;               // k_walk_det runs before k_walk (deterministic occupancy)
    int ndt_segs;                        // NDT batch with segment descriptors (k_walk_ndt_det)
    int nidx;                            // the batch's index-claim layer (L_NIDX / L_NIDX2)
    unsigned long long *nlost;           // voxel-index claims lost to a concurrent claimer (NDT / TSDF)
    int ray_order;                       // NDT walks: k_discover buckets rays by step count and
                                         // the walk takes them through perm, longest first
    // region sharding (vm_shard_*): this map owns regions with owner(key) == shard_rank
    int shard_rank, shard_world;
    long long ray_lo;                    // first ray of this map's slice of the batch
    int2 *marked;                        // new sample voxels (slot, li) of the slice
    unsigned long long *nmarked;
    unsigned long long marked_cap;
    unsigned long long rec_invalid;      // voxel-id field of dropped records (skipped by the fold)
    int walk_slot0;                      // regions with slot >= this were created by the walk
    int key_mi;                          // occupancy records key on the sample-voxel index
                                         // (marked list) instead of the voxel id
    // pipelined batch sequences (vm_integrate_many): the first batch that is
    // refused or overflows its records sets *chain (batch + 1) and every later
    // batch of the sequence becomes a no-op; nullptr for single batches
    int *chain;
    int batch_idx;
    // batch outputs
    unsigned long long *rec;
    unsigned *recval;                    // per-record value (NDT deterministic phase 1)
    double2 *rec_t;                      // NDT phase-1 records: the visit's chord (t0, t1),
                                         // weighed after the walk (k_ndt_weigh)
    unsigned long long rec_cap;
    int *touched;                        // regions touched by the walk
    int touched_cap;
    // region-sharded NDT (vm_shard_ndt.cuh): the walk's visits through
    // Gaussian voxels of regions other ranks own, for their owners
    void *gx;
    unsigned long long *ngx;
    unsigned long long gx_cap;
    // eviction (vm_map_evict_regions): region key table values of spilled
    // regions are SLOT_SPILLED; the prefetch lists the ones a batch reaches
    // (the guard refuses it, the host reloads them and replays)
    long long *reload;
    int reload_cap;
    unsigned batch_no;                   // the batch counter (Region.last_access)
    unsigned *slot_last;                 // per slot: last batch whose prefetch touched it
};

// ---------------------------------------------------------------- arithmetic

// RaySample.length (traversal.py:40-42): np.linalg.norm -> OpenBLAS ddot
__device__ __forceinline__ double norm3(double x, double y, double z) {
    return sqrt(fma(z, z, fma(y, y, x * x)));
}
// float(a @ b) for 3-vectors (reference.py:170)
__device__ __forceinline__ double dot3(const double *a, const double *b) {
    return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

// _kernels.pyx:105-110 (splitmix64 finalizer)
__host__ __device__ __forceinline__ unsigned long long mix_key(long long key) {
    unsigned long long h = (unsigned long long)key + 0x9E3779B97F4A7C15ULL;
    h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ULL;
    h = (h ^ (h >> 27)) * 0x94D049BB133111EBULL;
    return h ^ (h >> 31);
}

// keys.py:76-86
__host__ __device__ __forceinline__ long long pack_region(long long rx, long long ry,
                                                          long long rz) {
    const long long B = 1LL << 20, M = (1LL << 21) - 1;
    return (((rx + B) & M) << 42) | (((ry + B) & M) << 21) | ((rz + B) & M);
}
__host__ __device__ __forceinline__ void unpack_region(long long p, int r[3]) {
    const long long B = 1LL << 20, M = (1LL << 21) - 1;
    r[0] = (int)(((p >> 42) & M) - B);
    r[1] = (int)(((p >> 21) & M) - B);
    r[2] = (int)((p & M) - B);
}

__device__ __forceinline__ int floordiv(int a, int d) {
    int q = a / d;
    if ((a % d != 0) && (a < 0)) q -= 1;
    return q;
}

// Fire-and-forget reductions (REDG): no return value, no scoreboard wait.
__device__ __forceinline__ void red_add(unsigned *p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or(unsigned *p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// reference.py:22-23 / _kernels.pyx:233-271 clamped log-odds step (f32)
__device__ __forceinline__ float clamp_add(float l, float d, float cmin, float cmax) {
    float v = __fadd_rn(l, d);
    if (v < cmin) v = cmin;
    if (v > cmax) v = cmax;
    return v;
}
// k identical misses: f^k with early exit at the fixed point (clamp_min)
__device__ __forceinline__ float miss_k(float l, unsigned k, float d, float cmin, float cmax) {
    for (unsigned i = 0; i < k; ++i) {
        float n = clamp_add(l, d, cmin, cmax);
        if (__float_as_uint(n) == __float_as_uint(l)) break;
        l = n;
    }
    return l;
}

// ---- verified fast division / square root (the serial folds' steps) ----
// IEEE `a / b` and `sqrt(x)` compile to an approximation, Newton steps and a
// branch to a slow path that needs the result first, so a thread's
// independent divisions run one after another.  These variants are
// branch-free: the Newton result q is checked to be THE correctly rounded
// value (the exact residual a - b*q, one FMA, is below half an ulp of q
// times |b|; operands and result well inside the normal range), and `ok`
// turns false otherwise -- the caller then redoes the step with the IEEE
// operators, so the values are always the IEEE ones.
__device__ __forceinline__ int xexp(double v) {
    return (int)((unsigned long long)__double_as_longlong(v) >> 52) & 0x7FF;
}
__device__ __forceinline__ bool xmid(double v) {
    const int e = xexp(v);
    return e > 200 && e < 1800;
}
__device__ __forceinline__ double xpow2(int biased) { return __longlong_as_double((long long)biased << 52); }
__device__ __forceinline__ double xrcp(double b) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    double e = fma(-b, y, 1.0);
    y = fma(y, e, y);
    e = fma(-b, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double xdiv(double a, double b, bool &ok) {
    const double y = xrcp(b);
    double q = a * y;
    q = fma(fma(-b, q, a), y, q);
    const double r = fma(-b, q, a);
    const double e = ((b < 0.0) != (q < 0.0)) ? -r : r;
    const double hb = fabs(b) * xpow2(xexp(q) - 53);
    const bool p2 = (__double_as_longlong(q) & 0xFFFFFFFFFFFFFLL) == 0;
    const bool good = xmid(q) && xmid(a) && xmid(b) && e < hb && -e < (p2 ? 0.5 * hb : hb);
    ok = ok && (good || (a == 0.0 && xmid(b)));
    return a == 0.0 ? a * y : q;
}
__device__ __forceinline__ double xsqrt(double x, bool &ok) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = fma(y, fma(-hx * y, y, 0.5), y);
    y = fma(y, fma(-hx * y, y, 0.5), y);
    double s = x * y;
    s = fma(fma(-s, s, x), 0.5 * y, s);
    const double r = fma(-s, s, x);
    const double su = s * xpow2(xexp(s) - 52);
    const bool p2 = (__double_as_longlong(s) & 0xFFFFFFFFFFFFFLL) == 0;
    const bool good = x > 0.0 && xmid(x) && xmid(s) && r <= su && -r < (p2 ? 0.5 * su : su);
    ok = ok && (good || x == 0.0);
    return x == 0.0 ? x : s;
}
// FAST: the verified operators (ok false = redo with IEEE); else IEEE
template <bool FAST>
__device__ __forceinline__ double vdiv(double a, double b, bool &ok) {
    if (FAST) return xdiv(a, b, ok);
    return a / b;
}
template <bool FAST>
__device__ __forceinline__ double vsqrt(double x, bool &ok) {
    if (FAST) return xsqrt(x, ok);
    return sqrt(x);
}
// subvoxel.py:16-23
__device__ __forceinline__ unsigned pack_mean(const double off[3]) {
    unsigned packed = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double f = floor(off[a] * 1024.0);
        int q = f < 0.0 ? 0 : (f > 1023.0 ? 1023 : (int)f);
        packed |= (unsigned)q << (10 * a);
    }
    return packed;
}
// subvoxel.py:26-31
__device__ __forceinline__ void unpack_mean(unsigned packed, double out[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) out[a] = ((double)((packed >> (10 * a)) & 1023u) + 0.5) / 1024.0;
}
// subvoxel.py:34-49 (the oracle's `/ (count + 1)` form, not the native `* w`)
// fold_mean with the division selectable (FAST: verified, `ok` false = redo)
template <bool FAST>
__device__ __forceinline__ void fold_mean_v(unsigned &packed, unsigned &count, const double s[3],
                                            bool &ok) {
    if (count >= 0xFFFFFFFFu) return;
    if (count == 0) {
        packed = pack_mean(s);
        count = 1;
        return;
    }
    double m[3];
    unpack_mean(packed, m);
    double div = (double)count + 1.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) m[a] = m[a] + vdiv<FAST>(s[a] - m[a], div, ok);
    packed = pack_mean(m);
    count += 1;
}

__device__ __forceinline__ void fold_mean(unsigned &packed, unsigned &count, const double s[3]) {
    if (count >= 0xFFFFFFFFu) return;
    if (count == 0) {
        packed = pack_mean(s);
        count = 1;
        return;
    }
    double m[3];
    unpack_mean(packed, m);
    double div = (double)count + 1.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) m[a] = m[a] + (s[a] - m[a]) / div;
    packed = pack_mean(m);
    count += 1;
}

// Brick (4 x 4 x 2 per region, i.e. 8 x 8 x 16 voxels at dim 32) of local
// index li = lx + dim * (ly + dim * lz), for power-of-two dims: bit index of
// the per-region sample-voxel summary.
__device__ __forceinline__ unsigned brick_of(int li, const int bsh[3]) {
    return (((unsigned)li >> bsh[0]) & 3u) | (((unsigned)li >> bsh[1]) & 0xCu) |
           (((unsigned)li >> bsh[2]) & 0x10u);
}

// ---------------------------------------------------------------- rays

struct SrcOHMB1 {  // rayset.py:19-27 40-byte records
    const unsigned char *p;
    __device__ __forceinline__ void load(long long i, double o[3], double e[3], int &has,
                                         float &inten) const {
        const float2 *q = reinterpret_cast<const float2 *>(p + i * 40 + 8);
        float2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
        o[0] = a.x; o[1] = a.y; o[2] = b.x;
        e[0] = b.y; e[1] = c.x; e[2] = c.y;
        inten = d.x;
        has = (int)(__float_as_uint(d.y) & 1u);
    }
    __device__ __forceinline__ void load_end(long long i, double e[3], float &inten) const {
        const float2 *q = reinterpret_cast<const float2 *>(p + i * 40 + 8);
        float2 b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
        e[0] = b.y; e[1] = c.x; e[2] = c.y;
        inten = d.x;
    }
};
struct SrcF64 {  // RaySample arrays (traversal.py:20-42)
    const double *o, *e;
    const unsigned char *h;
    const float *it;
    __device__ __forceinline__ void load(long long i, double oo[3], double ee[3], int &has,
                                         float &inten) const {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            oo[a] = __ldg(o + 3 * i + a);
            ee[a] = __ldg(e + 3 * i + a);
        }
        has = __ldg(h + i) ? 1 : 0;
        inten = it ? __ldg(it + i) : 0.0f;
    }
    __device__ __forceinline__ void load_end(long long i, double ee[3], float &inten) const {
#pragma unroll
        for (int a = 0; a < 3; ++a) ee[a] = __ldg(e + 3 * i + a);
        inten = it ? __ldg(it + i) : 0.0f;
    }
};

// engine._preprocess + clip_ray + segment_ray (engine.py:82-96,
// traversal.py:140-178), in registers: one ray -> nseg segments.
struct Ray {
    double o[3], e[3], d[3];
    double L;
    int has, nseg;
    float inten;
};

__device__ __forceinline__ bool prep_ray(const DevMap &m, Ray &r, bool segment) {
    double L = norm3(r.e[0] - r.o[0], r.e[1] - r.o[1], r.e[2] - r.o[2]);
    if (L == 0.0) return false;
    if (L > m.max_range) {
        double d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) d[a] = (r.e[a] - r.o[a]) / L;
#pragma unroll
        for (int a = 0; a < 3; ++a) r.e[a] = r.o[a] + d[a] * m.max_range;
        r.has = 0;
        L = norm3(r.e[0] - r.o[0], r.e[1] - r.o[1], r.e[2] - r.o[2]);
    }
    r.L = L;
    if (!segment || L <= m.seg_len) {
        r.nseg = 1;
        return true;
    }
    r.nseg = (int)ceil(L / m.seg_len);
#pragma unroll
    for (int a = 0; a < 3; ++a) r.d[a] = (r.e[a] - r.o[a]) / L;
    return true;
}

__device__ __forceinline__ void segment_of(const DevMap &m, const Ray &r, int s, double so[3],
                                           double se[3], int &sh) {
    if (r.nseg == 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            so[a] = r.o[a];
            se[a] = r.e[a];
        }
        sh = r.has;
        return;
    }
    double t0 = (double)s * m.seg_len;
    double t1 = (double)(s + 1) * m.seg_len;
    if (r.L < t1) t1 = r.L;
    bool last = s == r.nseg - 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        so[a] = r.o[a] + r.d[a] * t0;
        se[a] = last ? r.e[a] : r.o[a] + r.d[a] * t1;
    }
    sh = last ? r.has : 0;
}

// ---------------------------------------------------------------- region table

// _kernels.pyx:113-124 (table_lookup) + on-demand creation with the
// sequential oracle's get_or_create semantics (reference.py:31).
__device__ __forceinline__ int wait_slot(const DevMap &m, unsigned long long h) {
    volatile int *p = m.tvals + h;
    int v;
    while ((v = *p) == -1) __nanosleep(32);
    return v;
}

__device__ __forceinline__ int region_slot_probe(const DevMap &m, long long key) {
    unsigned long long h = mix_key(key) & m.tmask;
    for (unsigned long long probe = 0; probe <= m.tmask; ++probe) {
        long long k = ((volatile long long *)m.tkeys)[h];
        if (k == key) return wait_slot(m, h);
        if (k == -1) {
            if (!m.insert) return -1;
            long long prev = (long long)atomicCAS((unsigned long long *)(m.tkeys + h),
                                                  0xFFFFFFFFFFFFFFFFULL,
                                                  (unsigned long long)key);
            if (prev == -1) {
                int s = atomicAdd(m.cursor, 1);
                if (s < m.max_slots) m.slot_keys[s] = key;
                else s = -2;  // id space exhausted: permanent region miss
                __threadfence();
                atomicExch(m.tvals + h, s);
                return s;
            }
            if (prev == key) return wait_slot(m, h);
        }
        h = (h + 1) & m.tmask;
    }
    return -1;
}

// Lookup only (never creates): slot or -1.
__device__ __noinline__ int region_find(const DevMap &m, long long key) {
    unsigned long long h = mix_key(key) & m.tmask;
    for (unsigned long long probe = 0; probe <= m.tmask; ++probe) {
        const long long k = ((volatile long long *)m.tkeys)[h];
        if (k == key) return wait_slot(m, h);
        if (k == -1) return -1;
        h = (h + 1) & m.tmask;
    }
    return -1;
}

__device__ __noinline__ int region_slot_slow(const DevMap &m, long long key) {
    return region_slot_probe(m, key);
}

// Lookup only (never creates): slot or -1.
__device__ __forceinline__ int region_find_probe(const DevMap &m, long long key) {
    unsigned long long h = mix_key(key) & m.tmask;
    for (unsigned long long probe = 0; probe <= m.tmask; ++probe) {
        const long long k = ((volatile long long *)m.tkeys)[h];
        if (k == key) return wait_slot(m, h);
        if (k == -1) return -1;
        h = (h + 1) & m.tmask;
    }
    return -1;
}

// Same as region_slot, fully inlined (no call ABI inside register-heavy loops).
__device__ __forceinline__ int region_slot_inl(const DevMap &m, long long key) {
    unsigned long long h = mix_key(key) & m.tmask;
    long long k = m.tkeys[h];
    if (k == key) {
        int v = m.tvals[h];
        if (v >= 0) return v;
    }
    return region_slot_probe(m, key);
}

__device__ __forceinline__ int region_slot(const DevMap &m, long long key) {
    // fast path: plain (cached) probe of entries that existed before this kernel
    unsigned long long h = mix_key(key) & m.tmask;
    long long k = m.tkeys[h];
    if (k == key) {
        int v = m.tvals[h];
        if (v >= 0) return v;
    }
    return region_slot_slow(m, key);
}

// Region owner for sharded maps: blocks of 2 x 2 x 2
// regions hashed over the ranks, so the busy regions around a sensor spread
// over all GPUs while neighbouring regions mostly stay together.
__host__ __device__ __forceinline__ int region_owner(long long key, int world) {
    if (world <= 1) return 0;
    const long long B = 1LL << 20, M = (1LL << 21) - 1;
    const long long bx = (((key >> 42) & M) - B) >> 1, by = (((key >> 21) & M) - B) >> 1,
                    bz = ((key & M) - B) >> 1;
    return (int)(mix_key(pack_region(bx, by, bz)) % (unsigned long long)world);
}

// First stamp of `epoch` into a per-slot word: true for exactly one caller
// per epoch.  A plain load first, so the common already-stamped case costs
// no atomic on these hot words (every block touches the sensor's regions).
__device__ __forceinline__ bool stamp_epoch(unsigned *p, unsigned epoch) {
    if (*((volatile unsigned *)p) == epoch) return false;
    return atomicExch(p, epoch) != epoch;
}

// ---------------------------------------------------------------- block helpers

// Per-block set of region slots already recorded this kernel: turns the
// per-ray region bookkeeping into O(blocks x regions) global atomics.
__device__ __forceinline__ bool slotset_insert(int *set, int slot) {
    unsigned h = ((unsigned)slot * 2654435761u) >> 24;
    for (int i = 0; i < SLOTSET; ++i) {
        unsigned idx = (h + i) & (SLOTSET - 1);
        int v = set[idx];
        if (v == slot) return false;
        if (v == -1) {
            int prev = atomicCAS(set + idx, -1, slot);
            if (prev == -1) return true;
            if (prev == slot) return false;
        }
    }
    return true;  // set full: treat as new (global op stays correct)
}

template <int N>
__device__ __forceinline__ void block_add_stats(const DevMap &m, unsigned long long (&v)[N],
                                                const int (&which)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        unsigned long long x = v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(m.stats + which[i], x);
    }
}

// Track the region of the walker's current voxel: local coordinates are
// stepped incrementally and the table is probed only on face crossings.
// (Scalar fields only: dynamic array indexing would spill to local memory.)
struct RegionTrack {
    int rx, ry, rz, lx, ly, lz;
    int slot;
    __device__ __forceinline__ void locate(const DevMap &m, int gx, int gy, int gz) {
        rx = floordiv(gx, m.dim);
        ry = floordiv(gy, m.dim);
        rz = floordiv(gz, m.dim);
        lx = gx - rx * m.dim;
        ly = gy - ry * m.dim;
        lz = gz - rz * m.dim;
        slot = region_slot(m, pack_region(rx, ry, rz));
    }
    // returns true if the region changed
    __device__ __forceinline__ bool step(const DevMap &m, int axis, int s) {
        int *l = axis == 0 ? &lx : (axis == 1 ? &ly : &lz);
        int *r = axis == 0 ? &rx : (axis == 1 ? &ry : &rz);
        int nl = *l + s;
        if (nl == m.dim) {
            *l = 0;
            *r += 1;
        } else if (nl < 0) {
            *l = m.dim - 1;
            *r -= 1;
        } else {
            *l = nl;
            return false;
        }
        slot = region_slot(m, pack_region(rx, ry, rz));
        return true;
    }
    __device__ __forceinline__ int li(const DevMap &m) const {
        return lx + m.dim * (ly + m.dim * lz);
    }
};

// ---------------------------------------------------------------- the walk

// DDA initial state of traversal._walk_grid (traversal.py:58-78) into a
// descriptor (everything the persistent walk needs to start the segment).
// Returns the start cell in c[].
__device__ __forceinline__ void dda_init(const double o[3], const double e[3], double cell,
                                         SegDesc &sd, int c[3]) {
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    unsigned codes = 0;
    int rem = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double v = e[a] - o[a];
        c[a] = (int)floor(o[a] / cell);
        sd.e[a] = (int)floor(e[a] / cell);
        rem += abs(sd.e[a] - c[a]);
        double t = INF, d = INF;
        unsigned code = 1;  // step + 1
        if (v > 0) {
            code = 2;
            t = ((double)(c[a] + 1) * cell - o[a]) / v;
            d = cell / v;
        } else if (v < 0) {
            code = 0;
            t = ((double)c[a] * cell - o[a]) / v;
            d = -cell / v;
        }
        sd.t[a] = t;
        sd.d[a] = d;
        codes |= code << (2 * a);
    }
    sd.flags = codes << 1;
    sd.rem = (unsigned)rem;
}

// traversal._walk_grid (traversal.py:52-111) == _kernels.walk_fill
// (_kernels.pyx:134-211), streamed: the visitor sees every visit in order
// with (global cell, entry t, exit t, is_last).  Exact fp64 (no FMA).
// V::begin(g) is called once, V::moved(axis, step) after every DDA step,
// V::jump(g) before the numerical-fallback visit.  Scalar state only.
template <class V>
__device__ __forceinline__ void walk(const double o[3], const double e[3], double cell, V &vis) {
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const double vx = e[0] - o[0], vy = e[1] - o[1], vz = e[2] - o[2];
    int cx = (int)floor(o[0] / cell), cy = (int)floor(o[1] / cell), cz = (int)floor(o[2] / cell);
    const int ex = (int)floor(e[0] / cell), ey = (int)floor(e[1] / cell),
              ez = (int)floor(e[2] / cell);
    int sx = 0, sy = 0, sz = 0;
    double tx = INF, ty = INF, tz = INF, dx = INF, dy = INF, dz = INF;
    if (vx > 0) { sx = 1; tx = ((double)(cx + 1) * cell - o[0]) / vx; dx = cell / vx; }
    else if (vx < 0) { sx = -1; tx = ((double)cx * cell - o[0]) / vx; dx = -cell / vx; }
    if (vy > 0) { sy = 1; ty = ((double)(cy + 1) * cell - o[1]) / vy; dy = cell / vy; }
    else if (vy < 0) { sy = -1; ty = ((double)cy * cell - o[1]) / vy; dy = -cell / vy; }
    if (vz > 0) { sz = 1; tz = ((double)(cz + 1) * cell - o[2]) / vz; dz = cell / vz; }
    else if (vz < 0) { sz = -1; tz = ((double)cz * cell - o[2]) / vz; dz = -cell / vz; }
    int remaining = abs(cx - ex) + abs(cy - ey) + abs(cz - ez);
    double tprev = 0.0;
    vis.begin(cx, cy, cz);
    for (;;) {
        if (cx == ex && cy == ey && cz == ez) {
            vis.visit(cx, cy, cz, tprev, 1.0, true);
            return;
        }
        if (remaining <= 0) {
            vis.jump(ex, ey, ez);
            vis.visit(ex, ey, ez, tprev, 1.0, true);
            return;
        }
        // axis = 0; if tmax[1] < tmax[axis]: 1; if tmax[2] < tmax[axis]: 2
        int axis = ty < tx ? 1 : 0;
        double ta = axis ? ty : tx;
        if (tz < ta) { axis = 2; ta = tz; }
        double tn = ta;
        if (tn < tprev) tn = tprev;
        if (tn > 1.0) tn = 1.0;
        vis.visit(cx, cy, cz, tprev, tn, false);
        if (axis == 0) { cx += sx; tx += dx; vis.moved(0, sx); }
        else if (axis == 1) { cy += sy; ty += dy; vis.moved(1, sy); }
        else { cz += sz; tz += dz; vis.moved(2, sz); }
        tprev = tn;
        --remaining;
    }
}

}  // namespace vm
