// vm_runtime.cu -- device map runtime and the C ABI (include/voxmap_b200.h).
//
// Owns the HBM region pool (one slab per layer, region slot s at
// slab + s * bytes_per_region), the open-addressing region table in the
// format of engine._build_region_table (engine.py:121-147), and the batch
// pipeline of submit_batch (engine.py:175-210).  All work is enqueued on
// the map's stream; vm_integrate returns once the batch is complete.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <zlib.h>

#include "../../include/voxmap_b200.h"
#include "vm_walk.cuh"
#include "vm_compat.cuh"
#include "vm_walk_det.cuh"
#include "vm_walk_ndt_det.cuh"
#include "vm_shard.cuh"
#include "vm_bucket.cuh"
#include "vm_ndt.cuh"
#include "vm_shard_ndt.cuh"
#include "vm_export.cuh"

using namespace vm;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            return fail(e_ == cudaErrorMemoryAllocation ? VM_ERR_OOM : VM_ERR_CUDA,     \
                        std::string(#x) + ": " + cudaGetErrorString(e_));              \
    } while (0)

constexpr int RELOAD_CAP = 4096;  // spilled regions one refused attempt can list

const int LAYER_ELEM[NUM_LAYERS] = {4, 4, 4, 4, 4, 4, 4, 4, 4, 8, 4, 4, 4};
const int LAYER_COMP[NUM_LAYERS] = {1, 1, 1, 1, 6, 1, 1, 2, 1, 1, 2, 1, 1};

int bitlen(unsigned long long x) {
    int b = 0;
    while (x) {
        ++b;
        x >>= 1;
    }
    return b;
}

template <class T>
int dev_alloc(T **p, size_t count, int fill = 0) {
    *p = nullptr;
    if (count == 0) count = 1;
    CK(cudaMalloc((void **)p, count * sizeof(T)));
    CK(cudaMemset(*p, fill, count * sizeof(T)));
    return VM_OK;
}

}  // namespace

struct vm_map {
    vm_config cfg{};
    uint32_t mask = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int dim = 0, vpr = 0;
    long long max_slots = 0, cap = 0, nreg = 0, max_growth = 0;
    size_t bpr[NUM_LAYERS] = {};
    void *slab[NUM_LAYERS] = {};
    void **d_lptr[NUM_LAYERS] = {};
    long long *d_tkeys = nullptr;
    int *d_tvals = nullptr;
    unsigned long long tsize = 0;
    int *d_cursor = nullptr;
    long long *d_slot_keys = nullptr;
    unsigned *d_slot_touch = nullptr, *d_slot_pref = nullptr;
    SegDesc *d_segs = nullptr;
    size_t seg_cap = 0;
    unsigned *d_perm = nullptr;
    size_t perm_cap = 0;
    unsigned char *d_seg_bk = nullptr;
    size_t seg_bk_cap = 0;
    unsigned *d_seg_hist = nullptr, *d_seg_cursor = nullptr;
    unsigned long long *d_work = nullptr;
    int *d_rgrid = nullptr;
    unsigned *d_bmask = nullptr;
    unsigned *d_gmask = nullptr;     // NDT: bricks that may hold a Gaussian (walk skips the count load)
    int *d_rbox = nullptr;
    long long *d_big = nullptr;
    size_t big_cap = 0;
    unsigned long long *d_nbig = nullptr;
    unsigned long long *d_nmid = nullptr;  // occupancy bucket fold: medium buckets
    // bucketed fold of the deterministic occupancy records (vm_bucket.cuh)
    unsigned *d_bk_cnt = nullptr, *d_bk_off = nullptr;
    size_t bk_cap = 0;
    int *d_bk_big = nullptr;
    unsigned *d_bk_perm = nullptr;   // NDT buckets, most samples first (vm_ndt.cuh)
    unsigned *d_bk_cnt2 = nullptr;   // NDT: samples per bucket
    int *d_bk_big2 = nullptr;        // NDT: buckets for the block sort
    unsigned long long *d_nbk_ctr = nullptr;  // NDT: [mid, big] sort-list lengths
    double4 *d_nbk_pos = nullptr;    // NDT: sample end points beside their bucket slots
    size_t nbk_pos_cap = 0;
    double2 *d_rec_t = nullptr;      // NDT: chords of the phase-1 records (k_ndt_weigh)
    size_t rec_t_cap = 0;
    unsigned *d_nbk_small = nullptr; // NDT: size histogram, cursors, live count, slice cursor
    double4 *d_ndt_roots = nullptr;  // NDT: tabulated count roots (k_ndt_roots)
    unsigned *d_bk_bits = nullptr;
    size_t bk_bits_cap = 0;
    // pipelined sequences (vm_integrate_many)
    int *d_chain = nullptr;
    unsigned long long *d_mstats = nullptr, *h_mstats = nullptr;
    size_t mstats_cap = 0;  // batches
    std::vector<cudaEvent_t> mev;  // 6 per batch
    static constexpr int RING = 3;
    unsigned char *d_ring[RING] = {};
    size_t ring_bytes = 0;
    cudaEvent_t ev_ring[RING] = {}, ev_ring_up[RING] = {};
    // eviction / spill (vm_map_evict_regions): OHMS1 files in spill_dir
    std::string spill_dir;
    std::vector<int> spill_ids;      // user layers in the host map's order (payload order)
    std::set<long long> spilled;     // packed keys of the regions on disk
    long long *d_reload = nullptr;   // keys of spilled regions a refused batch reached
    unsigned *d_slot_last = nullptr; // per slot: last batch whose prefetch touched it
    unsigned batch_no = 0;           // Region.last_access value of the next batch
    long long rec_floor_override = 0;
    long long ndt_rec_override = 0;  // VOXMAP_B200_TEST_NDT_REC_CAP: force the NDT overflow path
    int no_ray_order = 0;  // VOXMAP_B200_NO_RAY_ORDER: NDT walk in input order (A/B runs)
    int no_pipeline = 0;   // VOXMAP_B200_NO_PIPELINE: sequences as one vm_integrate per batch (A/B runs)
    int ndt_generic = 0;   // VOXMAP_B200_NDT_GENERIC: NDT walks ray by ray (k_walk_ndt; A/B runs)
    int num_sms = 148;
    unsigned long long *d_stats = nullptr;
    int *d_go = nullptr;
    unsigned long long *d_rec = nullptr, *d_rec2 = nullptr;
    unsigned *d_val = nullptr, *d_val2 = nullptr;
    size_t rec_cap = 0;
    int *d_touched = nullptr;
    void *d_sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int sort_sized = 0;
    unsigned char *d_rays = nullptr;
    size_t rays_bytes = 0;
    // host rays of the batch: uploaded in chunks on copy_stream, each chunk's
    // discover waits only for its own chunk (the copy overlaps discover)
    cudaStream_t copy_stream = nullptr;
    // pipelined sequences: batch b+1's discover runs on disc_stream while batch
    // b resolves and folds; batch-scoped buffers alternate by batch parity
    cudaStream_t disc_stream = nullptr;
    cudaStream_t aux_stream = nullptr;  // NDT: bucket kernels next to k_resolve
    cudaEvent_t ev_seq0 = nullptr;
    int *d_touched2 = nullptr, *d_rgrid2 = nullptr, *d_rbox2 = nullptr, *d_go2 = nullptr;
    int2 *d_smarked2 = nullptr;
    size_t smarked2_cap = 0;
    SegDesc *d_segs2 = nullptr;      // (a batch's descriptors outlive the next discover:
    size_t segs2_cap = 0;            //  a records-overflow recovery re-walks them)
    unsigned *d_perm2 = nullptr;
    size_t perm2_cap = 0;
    unsigned char *d_seg_bk2 = nullptr;
    size_t seg_bk2_cap = 0;
    unsigned long long *d_mk2 = nullptr;  // parity-1 [nmarked, lost claims]
    static constexpr int UP_CHUNKS = 4;
    cudaEvent_t ev_up[UP_CHUNKS] = {};
    struct Upload {
        int pending = 0;            // 1: the first discover attempt uploads
        int format = 0;
        const unsigned char *rec = nullptr;  // OHMB1 host records
        const double *o = nullptr, *e = nullptr;
        const unsigned char *h = nullptr;
        const float *it = nullptr;
        size_t b_o = 0, b_h = 0;   // device layout of the f64 arrays
    } up;
    unsigned long long *h_stats = nullptr;  // pinned, NUM_STATS + 2
    // region sharding (vm_shard_*)
    int shard_rank = 0, shard_world = 1;
    int2 *d_smarked = nullptr;
    size_t smarked_cap = 0;
    unsigned long long *d_shard_cnt = nullptr;  // [2 + world]: nmarked, nreq, per-dest counts
    unsigned long long *d_nlost = nullptr;      // lost voxel-index claims of the batch (NDT / TSDF)
    unsigned long long *d_nlost2 = nullptr;     // ... of odd batches in a pipelined NDT sequence
    ShardItemN *d_gx = nullptr;      // sharded NDT: the walk's ghost visit items
    size_t gx_cap = 0;
    unsigned long long *d_ngx = nullptr;
    struct ShardBatch {
        bool open = false, walked = false;
        int format = 0;
        const void *rays = nullptr;  // device pointer of the batch (records or f64 arrays)
        const double *o = nullptr, *e = nullptr;
        const unsigned char *h = nullptr;
        const float *it = nullptr;
        long long n_all = 0, lo = 0, n = 0;
        int order_bits = 0, maxseg = 0, walk_slot0 = 0;
        long long nreg0 = 0, launches0 = 0;
        unsigned long long nmarks = 0, R = 0;
        int ndt = 0;                 // NDT-OM batch (vm_shard_ndt.cuh)
        float ms_disc = 0.f, ms_walk = 0.f;
    } sb;
    unsigned epoch = 0;
    long long launches = 0;
    cudaEvent_t ev_start{}, ev_end{}, ev_w0{}, ev_w1{}, ev_k1{}, ev_k2{}, ev_res{}, ev_sort{};
};

namespace {

DevMap make_dm(const vm_map *m) {
    DevMap d{};
    const vm_config &c = m->cfg;
    d.vox = c.voxel_size;
    d.rsize = (double)c.region_dim * c.voxel_size;  // config.py:54-57
    d.hit_delta = c.hit_delta;
    d.miss_delta = c.miss_delta;
    d.max_range = c.max_ray_range;
    d.seg_len = c.segment_length;
    d.tsdf_trunc = c.tsdf_truncation;
    d.tsdf_maxw = c.tsdf_max_weight;
    d.sigma2 = c.ndt_sensor_noise * c.ndt_sensor_noise;
    d.miss_check = c.ndt_miss_likelihood_threshold;
    d.hit32 = (float)c.hit_delta;
    d.miss32 = (float)c.miss_delta;
    d.cmin = (float)c.clamp_min;
    d.cmax = (float)c.clamp_max;
    d.fthresh = (float)c.ndt_reset_threshold;
    d.dim = m->dim;
    d.vpr = m->vpr;
    d.maxseg = (int)std::ceil(c.max_ray_range / c.segment_length) + 1;
    d.cell_limit = (int)std::min<long long>((1LL << 20) * (long long)m->dim - 1, (1LL << 30));
    d.tkeys = m->d_tkeys;
    d.tvals = m->d_tvals;
    d.tmask = m->tsize - 1;
    d.cursor = m->d_cursor;
    d.cap = (int)m->cap;
    d.max_slots = (int)m->max_slots;
    d.insert = 1;
    d.slot_keys = m->d_slot_keys;
    d.slot_touch = m->d_slot_touch;
    d.slot_pref = m->d_slot_pref;
    d.epoch = m->epoch;
    for (int l = 0; l < NUM_LAYERS; ++l) {
        d.lptr[l] = m->d_lptr[l];
        d.slab[l] = (char *)m->slab[l];
        d.bpr[l] = m->bpr[l];
    }
    d.rgrid = m->d_rgrid;
    d.bmask = m->d_bmask;
    d.gmask = m->d_gmask;
    {
        int bs = -1;
        if (m->dim >= 4 && (m->dim & (m->dim - 1)) == 0) {
            bs = 0;
            while ((1 << (bs + 2)) < m->dim) ++bs;
        }
        d.brick_shift = bs;
        int k = 0;
        while ((1 << k) < m->dim) ++k;
        // lx >> bs, (ly >> bs) << 2, (lz >> (bs + 1)) << 4 taken straight from li
        d.bsh[0] = bs < 0 ? 0 : bs;
        d.bsh[1] = bs < 0 ? 0 : k + bs - 2;
        d.bsh[2] = bs < 0 ? 0 : 2 * k + bs - 3;
    }
    d.rbox = m->d_rbox;
    d.rg_max = RG_MAX;
    d.segs = m->d_segs;
    d.perm = m->d_perm;
    d.seg_bk = m->d_seg_bk;
    d.seg_hist = m->d_seg_hist;
    d.seg_cursor = m->d_seg_cursor;
    d.seg_cap = m->seg_cap;
    d.work = m->d_work;
    d.stats = m->d_stats;
    d.go = m->d_go;
    d.rec = m->d_rec;
    d.recval = m->d_val;
    d.rec_t = m->d_rec_t;
    d.rec_cap = m->rec_cap;
    d.touched = m->d_touched;
    d.touched_cap = (int)m->max_slots;
    d.shard_rank = m->shard_rank;
    d.shard_world = m->shard_world;
    d.ray_lo = 0;
    d.marked = nullptr;
    d.nmarked = m->d_shard_cnt;
    d.marked_cap = 0;
    d.rec_invalid = ~0ULL;
    d.walk_slot0 = 1 << 30;
    d.key_mi = 0;
    d.nidx = L_NIDX;
    d.reload = m->d_reload;
    d.reload_cap = RELOAD_CAP;
    d.batch_no = m->batch_no;
    d.slot_last = m->d_slot_last;
    return d;
}

int grow_pool(vm_map *m, long long new_cap) {
    if (new_cap > m->max_slots) new_cap = m->max_slots;
    if (new_cap <= m->cap) return VM_OK;
    CK(cudaStreamSynchronize(m->stream));
    for (int l = 0; l < NUM_LAYERS; ++l) {
        if (!m->bpr[l]) continue;
        void *nw = nullptr;
        CK(cudaMalloc(&nw, (size_t)new_cap * m->bpr[l]));
        CK(cudaMemsetAsync((char *)nw + (size_t)m->cap * m->bpr[l], 0,
                           (size_t)(new_cap - m->cap) * m->bpr[l], m->stream));
        if (m->slab[l]) {
            CK(cudaMemcpyAsync(nw, m->slab[l], (size_t)m->cap * m->bpr[l],
                               cudaMemcpyDeviceToDevice, m->stream));
        }
        std::vector<void *> ptrs((size_t)new_cap);
        for (long long s = 0; s < new_cap; ++s) ptrs[s] = (char *)nw + (size_t)s * m->bpr[l];
        CK(cudaMemcpyAsync(m->d_lptr[l], ptrs.data(), ptrs.size() * sizeof(void *),
                           cudaMemcpyHostToDevice, m->stream));
        CK(cudaStreamSynchronize(m->stream));
        if (m->slab[l]) CK(cudaFree(m->slab[l]));
        m->slab[l] = nw;
    }
    m->cap = new_cap;
    return VM_OK;
}

template <class T>
int ensure_buf(T **p, size_t *cap, size_t need) {
    if (need <= *cap && *p) return VM_OK;
    size_t nc = std::max(need, *cap * 2);
    if (*p) CK(cudaFree(*p));
    *p = nullptr;
    CK(cudaMalloc((void **)p, nc * sizeof(T)));
    *cap = nc;
    return VM_OK;
}

int ensure_records(vm_map *m, size_t need) {
    if (need <= m->rec_cap && m->d_rec) return VM_OK;
    size_t nc = std::max(need, m->rec_cap * 2);
    if (m->d_rec) CK(cudaFree(m->d_rec));
    if (m->d_rec2) CK(cudaFree(m->d_rec2));
    if (m->d_val) CK(cudaFree(m->d_val));
    if (m->d_val2) CK(cudaFree(m->d_val2));
    m->d_rec = m->d_rec2 = nullptr;
    m->d_val = m->d_val2 = nullptr;
    CK(cudaMalloc((void **)&m->d_rec, nc * sizeof(unsigned long long)));
    CK(cudaMalloc((void **)&m->d_rec2, nc * sizeof(unsigned long long)));
    CK(cudaMalloc((void **)&m->d_val, nc * sizeof(unsigned)));
    CK(cudaMalloc((void **)&m->d_val2, nc * sizeof(unsigned)));
    m->rec_cap = nc;
    m->sort_sized = 0;  // CUB temp storage is sized lazily (ensure_sort_tmp)
    return VM_OK;
}

// CUB radix-sort temp storage for rec_cap records (the sorted NDT / TSDF /
// sharded paths; the bucketed occupancy fold never sorts).
int ensure_sort_tmp(vm_map *m) {
    if (m->sort_sized) return VM_OK;
    size_t bytes = 0, bytes2 = 0;
    cub::DoubleBuffer<unsigned long long> db(m->d_rec, m->d_rec2);
    cub::DoubleBuffer<unsigned> dv(m->d_val, m->d_val2);
    const int nc = (int)std::min<size_t>(m->rec_cap, INT32_MAX);
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, nc));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes2, db, dv, nc));
    bytes = std::max(bytes, bytes2);
    if (bytes > m->sort_tmp_bytes) {
        if (m->d_sort_tmp) CK(cudaFree(m->d_sort_tmp));
        CK(cudaMalloc(&m->d_sort_tmp, bytes));
        m->sort_tmp_bytes = bytes;
    }
    m->sort_sized = 1;
    return VM_OK;
}

// Initial record capacity of a deterministic occupancy batch.  The records
// overflow path is exercised by tests through VOXMAP_B200_TEST_REC_CAP
// (read when the map is created).
size_t rec_floor(const vm_map *m, long long n) {
    if (m->rec_floor_override > 0) return (size_t)m->rec_floor_override;
    return std::max<size_t>(1 << 20, (size_t)n * 4);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(VM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return VM_OK;
}

// One thread per (ray, segment): blockIdx.y is the segment index.  (A
// persistent variant with warp-claimed work items measured slower on C2:
// 28.9 vs 19.6 ms per step -- a block's region key cache then sees the whole
// batch instead of 256 neighbouring rays.)
template <class Src>
int launch_discover(vm_map *m, const DevMap &dm, const Src &src, long long n, int mode, int det,
                    int emit, int count_stats, cudaStream_t s) {
    const dim3 grid((unsigned)((n + DISC_BT - 1) / DISC_BT), mode == M_TSDF ? 1u : (unsigned)dm.maxseg);
    k_discover<<<grid, DISC_BT, 0, s>>>(dm, src, n, mode, det, emit, count_stats);
    m->launches += 1;
    return check_launch("discover");
}

// The dynamic shared-memory opt-in is a per-device (per-context) function
// attribute: set it once per device per kernel instantiation, checked.
// (One instantiation -- one `done` mask -- per kernel: the template parameter
// is the kernel itself, not its type, which several kernels share.)
template <auto Kernel>
cudaError_t opt_in_smem(size_t smem) {
    static unsigned long long done = 0;  // bit d: configured on device d
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && (done >> dev) & 1ULL) return cudaSuccess;
    e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && dev < 64) done |= 1ULL << dev;
    return e;
}

template <bool REC_ONLY, class Src, int DIM, bool SHARD>
cudaError_t launch_wd_sh(dim3 grid, cudaStream_t s, const DevMap &dm, const Src &src) {
    const size_t smem = sizeof(WalkDetSmem);
    cudaError_t e = opt_in_smem<k_walk_det<REC_ONLY, Src, DIM, SHARD>>(smem);
    if (e != cudaSuccess) return e;
    k_walk_det<REC_ONLY, Src, DIM, SHARD><<<grid, BLOCK, smem, s>>>(dm, src);
    return cudaSuccess;
}

template <bool REC_ONLY, class Src, int DIM>
cudaError_t launch_wd_dim(dim3 grid, cudaStream_t s, const DevMap &dm, const Src &src) {
    if (dm.shard_world > 1) return launch_wd_sh<REC_ONLY, Src, DIM, true>(grid, s, dm, src);
    return launch_wd_sh<REC_ONLY, Src, DIM, false>(grid, s, dm, src);
}

template <class Src, int DIM>
cudaError_t launch_wn_dim(dim3 grid, cudaStream_t s, const DevMap &dm, const Src &src) {
    const size_t smem = sizeof(WalkNdtSmem);
    cudaError_t e = opt_in_smem<k_walk_ndt_det<Src, DIM>>(smem);
    if (e != cudaSuccess) return e;
    k_walk_ndt_det<Src, DIM><<<grid, BLOCK, smem, s>>>(dm, src);
    return cudaSuccess;
}

template <class Src>
cudaError_t launch_wn(dim3 grid, cudaStream_t s, const DevMap &dm, const Src &src) {
    if (dm.dim == 32 && dm.brick_shift == 3) return launch_wn_dim<Src, 32>(grid, s, dm, src);
    return launch_wn_dim<Src, 0>(grid, s, dm, src);
}

template <bool REC_ONLY, class Src>
cudaError_t launch_wd(dim3 grid, cudaStream_t s, const DevMap &dm, const Src &src) {
    if (dm.dim == 32 && dm.brick_shift == 3) return launch_wd_dim<REC_ONLY, Src, 32>(grid, s, dm, src);
    return launch_wd_dim<REC_ONLY, Src, 0>(grid, s, dm, src);
}

template <int MODE, bool DET, bool REC_ONLY, class Src>
cudaError_t launch_w3(dim3 grid, size_t smem, cudaStream_t s, const DevMap &dm, const Src &src) {
    cudaError_t e = opt_in_smem<k_walk<MODE, DET, REC_ONLY, Src>>(smem);
    if (e != cudaSuccess) return e;
    k_walk<MODE, DET, REC_ONLY, Src><<<grid, BLOCK, smem, s>>>(dm, src);
    return cudaSuccess;
}

// kernel dispatch over (mode, exec, ray format)
template <class Src>
int launch_walk(vm_map *m, const DevMap &dm, const Src &src, long long n, int mode, bool det,
                bool rec_only) {
    dim3 grid((unsigned)((n + BLOCK - 1) / BLOCK)), block(BLOCK);
    cudaStream_t s = m->stream;
    // persistent grid: 2 resident blocks per SM, never more than the work needs
    dim3 pgrid((unsigned)std::max<long long>(
        1, std::min<long long>((long long)WK_BLOCKS * m->num_sms, (n * 3 + BLOCK - 1) / BLOCK)));
    // NDT batches with segment descriptors (ndt_segs) take the descriptor walk
    const bool ndt_seg = (mode == M_NDT_OM || mode == M_NDT_TM) && det && !rec_only && dm.ndt_segs;
    if (mode == M_OCC || mode == M_DECAY || ndt_seg) {
        cudaError_t e = cudaMemsetAsync(m->d_work, 0, sizeof(unsigned long long), s);
        if (e != cudaSuccess) return fail(VM_ERR_CUDA, cudaGetErrorString(e));
    }
    if (ndt_seg) {
        // the persistent descriptor walk; k_walk_ndt (input ray order) exits
        // unless the batch's box is too large for it (walk_det_ok)
        DevMap d2 = dm;
        d2.walk_det_launched = 1;
        d2.ray_order = 0;
        const dim3 ngrid((unsigned)std::max<long long>(
            1, std::min<long long>((long long)WN_BLOCKS * m->num_sms, (n * 3 + BLOCK - 1) / BLOCK)));
        cudaError_t ae = launch_wn(ngrid, s, d2, src);
        if (ae != cudaSuccess)
            return fail(VM_ERR_CUDA, std::string("walk shared-memory opt-in: ") + cudaGetErrorString(ae));
        if (mode == M_NDT_TM) k_walk_ndt<true, true, false><<<grid, block, 0, s>>>(d2, src, n);
        else k_walk_ndt<false, true, false><<<grid, block, 0, s>>>(d2, src, n);
        m->launches += 2;
        return check_launch("walk");
    }
    const size_t smem = sizeof(WalkSmem);
    cudaError_t ae = cudaSuccess;
    switch (mode) {
    case M_OCC:
        if (det) {
            // the lean deterministic walk; the generic one below exits unless
            // the batch's box is too large for it (walk_det_ok)
            DevMap d2 = dm;
            d2.walk_det_launched = 1;
            ae = rec_only ? launch_wd<true>(pgrid, s, d2, src) : launch_wd<false>(pgrid, s, d2, src);
            if (ae == cudaSuccess)
                ae = rec_only ? launch_w3<M_OCC, true, true>(pgrid, smem, s, d2, src)
                              : launch_w3<M_OCC, true, false>(pgrid, smem, s, d2, src);
            m->launches += 1;
        } else {
            ae = launch_w3<M_OCC, false, false>(pgrid, smem, s, dm, src);
        }
        break;
    case M_DECAY:
        if (det && rec_only) ae = launch_w3<M_DECAY, true, true>(pgrid, smem, s, dm, src);
        else if (det) ae = launch_w3<M_DECAY, true, false>(pgrid, smem, s, dm, src);
        else ae = launch_w3<M_DECAY, false, false>(pgrid, smem, s, dm, src);
        break;
    case M_NDT_OM:
        if (det && rec_only) k_walk_ndt<false, true, true><<<grid, block, 0, s>>>(dm, src, n);
        else if (det) k_walk_ndt<false, true, false><<<grid, block, 0, s>>>(dm, src, n);
        else k_walk_ndt<false, false, false><<<grid, block, 0, s>>>(dm, src, n);
        break;
    case M_NDT_TM:
        if (det && rec_only) k_walk_ndt<true, true, true><<<grid, block, 0, s>>>(dm, src, n);
        else if (det) k_walk_ndt<true, true, false><<<grid, block, 0, s>>>(dm, src, n);
        else k_walk_ndt<true, false, false><<<grid, block, 0, s>>>(dm, src, n);
        break;
    case M_TSDF:
        if (det) k_walk_tsdf<true><<<grid, block, 0, s>>>(dm, src, n);
        else k_walk_tsdf<false><<<grid, block, 0, s>>>(dm, src, n);
        break;
    }
    m->launches += 1;
    if (ae != cudaSuccess)
        return fail(VM_ERR_CUDA, std::string("walk shared-memory opt-in: ") + cudaGetErrorString(ae));
    return check_launch("walk");
}

template <class Src>
int launch_fold(vm_map *m, const DevMap &dm, const Src &src, const unsigned long long *keys,
                const unsigned *vals, long long R, int mode) {
    cudaStream_t s = m->stream;
    const unsigned grid_cap = 148 * 16;
    if (mode == M_OCC || mode == M_DECAY) {
        if (R > 0) {
            int rc = ensure_buf(&m->d_big, &m->big_cap, (size_t)R / FOLD_SERIAL_MAX + 2);
            if (rc) return rc;
            cudaMemsetAsync(m->d_nbig, 0, sizeof(unsigned long long), s);
            unsigned g = (unsigned)std::min<long long>((R + BLOCK - 1) / BLOCK, grid_cap);
            k_fold_occ<<<g, BLOCK, 0, s>>>(dm, src, keys, R, m->d_big, m->d_nbig);
            k_fold_occ_big<<<m->num_sms * 2, BLOCK, 0, s>>>(dm, src, keys, R, m->d_big, m->d_nbig);
            m->launches += 2;
        }
    } else {
        unsigned g = (unsigned)std::min<long long>((R + BLOCK - 1) / BLOCK, grid_cap);
        if (g) k_fold_tsdf<<<g, BLOCK, 0, s>>>(dm, src, keys, R);
        m->launches += g ? 1 : 0;
    }
    return check_launch("fold");
}

// Bucketed in-order fold (vm_bucket.cuh): no host sync, no global sort.
int ensure_buckets(vm_map *m, size_t nmarked_cap, size_t bwords) {
    if (nmarked_cap + 1 > m->bk_cap || !m->d_bk_cnt) {
        size_t nc = std::max(nmarked_cap + 1, m->bk_cap * 2);
        cudaFree(m->d_bk_cnt);
        cudaFree(m->d_bk_off);
        cudaFree(m->d_bk_big);
        cudaFree(m->d_bk_perm);
        cudaFree(m->d_bk_cnt2);
        cudaFree(m->d_bk_big2);
        m->d_bk_cnt = nullptr;
        m->d_bk_off = nullptr;
        m->d_bk_big = nullptr;
        m->d_bk_perm = nullptr;
        m->d_bk_cnt2 = nullptr;
        m->d_bk_big2 = nullptr;
        CK(cudaMalloc((void **)&m->d_bk_cnt2, nc * sizeof(unsigned)));
        CK(cudaMemset(m->d_bk_cnt2, 0, nc * sizeof(unsigned)));
        CK(cudaMalloc((void **)&m->d_bk_big2, nc * sizeof(int)));
        CK(cudaMalloc((void **)&m->d_bk_cnt, nc * sizeof(unsigned)));
        CK(cudaMemset(m->d_bk_cnt, 0, nc * sizeof(unsigned)));  // kept zero by the folds
        CK(cudaMalloc((void **)&m->d_bk_off, nc * sizeof(unsigned)));
        CK(cudaMalloc((void **)&m->d_bk_big, nc * sizeof(int)));
        CK(cudaMalloc((void **)&m->d_bk_perm, nc * sizeof(unsigned)));
        m->bk_cap = nc;
    }
    const size_t need = (size_t)m->num_sms * BK_BIG_BPS * 2 * bwords;
    if (need > m->bk_bits_cap || !m->d_bk_bits) {
        cudaFree(m->d_bk_bits);
        m->d_bk_bits = nullptr;
        CK(cudaMalloc((void **)&m->d_bk_bits, need * sizeof(unsigned)));
        m->bk_bits_cap = need;
    }
    return VM_OK;
}

template <class Src>
int launch_bucket_fold(vm_map *m, const DevMap &dm, const Src &src, long long n, int maxseg,
                       cudaEvent_t ev_mid) {
    cudaStream_t s = m->stream;
    const unsigned long long bwords = ((unsigned long long)n * maxseg + 31) / 32 + 1;
    int rc;
    if ((rc = ensure_buckets(m, m->smarked_cap, bwords))) return rc;
    if (!m->d_nbk_small) {
        CK(cudaMalloc((void **)&m->d_nbk_small, (2 * NBK_BINS + 4) * sizeof(unsigned)));
        CK(cudaMemset(m->d_nbk_small, 0, (2 * NBK_BINS + 4) * sizeof(unsigned)));
    }
    unsigned *cursor = m->d_nbk_small + 2 * NBK_BINS + 2;
    if (!m->d_nmid && (rc = dev_alloc(&m->d_nmid, 1))) return rc;
    BucketState b{m->d_bk_cnt, m->d_bk_off, cursor, reinterpret_cast<unsigned *>(m->d_rec2),
                  m->d_bk_big, m->d_nbig, m->d_bk_big2, m->d_nmid, m->d_bk_bits, bwords};
    CK(cudaMemsetAsync(m->d_nbig, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(m->d_nmid, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(cursor, 0, sizeof(unsigned), s));
    const unsigned g = (unsigned)m->num_sms * 8;
    const unsigned ga = (unsigned)std::max<long long>(
        1, std::min<long long>((long long)m->num_sms * 8, ((long long)m->smarked_cap + BLOCK - 1) / BLOCK));
    static const bool split = std::getenv("VOXMAP_B200_BK_SPLIT") != nullptr;  // A/B knob
    k_bk_count<<<g, BLOCK, 0, s>>>(dm, b);
    k_bk_alloc<<<ga, BLOCK, 0, s>>>(dm, b, !split);
    k_bk_scatter<<<g, BLOCK, 0, s>>>(dm, b);
    CK(cudaEventRecord(ev_mid, s));
    if (!split) {
        // one fold launch, block roles by bucket size (vm_bucket.cuh: k_bk_fold_all)
        const int nbig = m->num_sms * BK_BIG_BPS, nmid = m->num_sms * 4;
        k_bk_fold_all<<<(unsigned)(nbig + nmid + m->num_sms * 8), BLOCK, 0, s>>>(dm, src, b, nbig, nmid);
        m->launches += 4;
        return check_launch("bucket fold");
    }
    const unsigned gf = (unsigned)std::max<long long>(
        1, std::min<long long>((long long)m->num_sms * 8, ((long long)m->smarked_cap + BLOCK - 1) / BLOCK));
    k_bk_fold<<<gf, BLOCK, 0, s>>>(dm, src, b);
    k_bk_fold_mid<<<m->num_sms * 4, BLOCK, 0, s>>>(dm, src, b);
    k_bk_fold_big<<<m->num_sms * BK_BIG_BPS, BLOCK, 0, s>>>(dm, src, b);
    m->launches += 7;
    return check_launch("bucket fold");
}

// NDT records: bucketed by voxel index, sorted per bucket, folded in order
// (vm_ndt.cuh).  Every count is read on the device.  launch_ndt_prep runs the
// phase-1 weights and the bucket kernels on `s`; they touch the records and
// the Gaussians of voxels holding one (count >= 3), never a voxel k_resolve
// updates (those got only order-free misses), so the pipelined paths run
// them on a second stream next to k_resolve.  launch_ndt_fold_only folds.
template <class Src>
int launch_ndt_prep(vm_map *m, const DevMap &dm, const Src &src, long long n, int maxseg,
                    cudaStream_t s, NdtBuckets *out) {
    const unsigned long long span = (unsigned long long)n * maxseg;
    const unsigned long long bwords = (2 * span + 31) / 32 + 1;
    int rc;
    if ((rc = ensure_buckets(m, m->smarked_cap, bwords))) return rc;
    if (!m->d_nbk_small) {
        CK(cudaMalloc((void **)&m->d_nbk_small, (2 * NBK_BINS + 4) * sizeof(unsigned)));
        CK(cudaMemset(m->d_nbk_small, 0, (2 * NBK_BINS + 4) * sizeof(unsigned)));
    }
    if (!m->d_nbk_ctr) CK(cudaMalloc((void **)&m->d_nbk_ctr, 2 * sizeof(unsigned long long)));
    if ((rc = ensure_buf(&m->d_nbk_pos, &m->nbk_pos_cap, m->rec_cap))) return rc;
    NdtBuckets b{m->d_bk_cnt, m->d_bk_cnt2, m->d_bk_off, m->d_bk_perm, m->d_nbk_small,
                 m->d_nbk_small + NBK_BINS, m->d_rec2, m->d_rec, m->d_nbk_pos, m->d_bk_big,
                 m->d_bk_big2, m->d_nbk_ctr, m->d_nbk_ctr + 1, m->d_bk_bits, bwords, span};
    CK(cudaMemsetAsync(m->d_nbk_ctr, 0, 2 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(b.cursor + NBK_BINS, 0, 3 * sizeof(unsigned), s));
    const unsigned gr = (unsigned)m->num_sms * 8;
    const unsigned gm = (unsigned)std::max<long long>(
        1, std::min<long long>((long long)m->num_sms * 8, ((long long)m->smarked_cap + BLOCK - 1) / BLOCK));
    static const bool split = std::getenv("VOXMAP_B200_NBK_SPLIT") != nullptr;  // A/B knob
    if (!split) {
        // four launches (vm_ndt.cuh: fused bucket preparation)
        k_nbk_weigh_count<<<gr, BLOCK, 0, s>>>(dm, src, b);
        k_nbk_alloc_order<<<gm, BLOCK, 0, s>>>(dm, b);
        k_nbk_perm_scatter<<<gr, BLOCK, 0, s>>>(dm, b);
        k_nbk_sort_gather<<<gr, BLOCK, 0, s>>>(dm, src, b, m->num_sms, m->num_sms * 4);
        m->launches += 4;
        *out = b;
        return check_launch("ndt buckets");
    }
    k_ndt_weigh<<<gr, BLOCK, 0, s>>>(dm, src);
    k_nbk_count<<<gr, BLOCK, 0, s>>>(dm, b);
    k_nbk_alloc<<<gm, BLOCK, 0, s>>>(dm, b);
    if (std::getenv("VOXMAP_B200_NDT_DEBUG")) {
        unsigned h[NBK_BINS];
        unsigned long long st[NUM_STATS], nm = 0;
        CK(cudaMemcpyAsync(h, b.hist, sizeof(h), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(st, dm.stats, sizeof(st), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&nm, dm.nmarked, sizeof(nm), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[ndt] R=%llu M=%llu buckets by size:", st[S_RECORDS], nm);
        for (int i = 0; i < NBK_BINS; ++i)
            if (h[i]) std::fprintf(stderr, " %d:%u", i, h[i]);
        std::fprintf(stderr, "\n");
    }
    k_nbk_order<<<1, NBK_BINS, 0, s>>>(dm, b);
    k_nbk_perm<<<gm, BLOCK, 0, s>>>(dm, b);
    k_nbk_scatter<<<gr, BLOCK, 0, s>>>(dm, b);
    k_nbk_sort_small<<<gm, BLOCK, 0, s>>>(dm, b);
    k_nbk_sort_mid<<<m->num_sms * 4, BLOCK, 0, s>>>(dm, b);
    k_nbk_sort_big<<<m->num_sms, BLOCK, 0, s>>>(dm, b);
    k_nbk_gather<<<gr, BLOCK, 0, s>>>(dm, src, b);
    m->launches += 10;
    *out = b;
    return check_launch("ndt buckets");
}

int launch_ndt_fold_only(vm_map *m, const DevMap &dm, const NdtBuckets &b, bool tm) {
    cudaStream_t s = m->stream;
    const unsigned gm = (unsigned)std::max<long long>(
        1, std::min<long long>((long long)m->num_sms * 8, ((long long)m->smarked_cap + BLOCK - 1) / BLOCK));
#ifdef VM_FOLD_PROF
    {
        unsigned long long z[2] = {0, 0};
        cudaMemcpyToSymbolAsync(g_fold_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, s);
    }
#endif
    static const bool fold1 = std::getenv("VOXMAP_B200_FOLD1") != nullptr;  // A/B knob
    if (fold1) {
        if (tm) k_nbk_fold<true><<<gm, BLOCK, 0, s>>>(dm, b);
        else k_nbk_fold<false><<<gm, BLOCK, 0, s>>>(dm, b);
    } else {
        // three lanes per bucket, the rotations pipelined (vm_ndt.cuh: k_nbk_fold3)
        if (!m->d_ndt_roots) {
            CK(cudaMalloc((void **)&m->d_ndt_roots, NDT_ROOTS_N * sizeof(double4)));
            k_ndt_roots<<<NDT_ROOTS_N / BLOCK, BLOCK, 0, s>>>(m->d_ndt_roots, NDT_ROOTS_N);
            m->launches += 1;
        }
        NdtBuckets b3 = b;
        b3.roots = m->d_ndt_roots;
        b3.nroots = NDT_ROOTS_N;
        const unsigned g3 = (unsigned)std::max<long long>(
            1, std::min<long long>((long long)m->num_sms * 8,
                                   ((long long)m->smarked_cap + NBK3_PER_WARP * (BLOCK / 32) - 1) /
                                       (NBK3_PER_WARP * (BLOCK / 32))));
        if (tm) k_nbk_fold3<true><<<g3, BLOCK, 0, s>>>(dm, b3);
        else k_nbk_fold3<false><<<g3, BLOCK, 0, s>>>(dm, b3);
    }
#ifdef VM_FOLD_PROF
    {
        unsigned long long h[2];
        cudaMemcpyFromSymbolAsync(h, g_fold_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        std::fprintf(stderr, "[fold] slowest task %llu cycles (phase-1 max %llu, samples max %llu); all tasks %llu cycles\n",
                     h[0] >> 24, (h[0] >> 12) & 4095, h[0] & 4095, h[1]);
    }
#endif
    m->launches += 1;
    return check_launch("ndt fold");
}

// prep + fold on the map's stream (after k_resolve)
template <class Src>
int launch_ndt_fold(vm_map *m, const DevMap &dm, const Src &src, long long n, int maxseg, bool tm,
                    cudaEvent_t ev_mid) {
    NdtBuckets b;
    int rc = launch_ndt_prep(m, dm, src, n, maxseg, m->stream, &b);
    if (rc) return rc;
    CK(cudaEventRecord(ev_mid, m->stream));
    return launch_ndt_fold_only(m, dm, b, tm);
}

// The NDT batch tail with the bucket kernels next to k_resolve: the aux
// stream waits for `walked` (recorded after the walk on the map's stream),
// prepares the buckets; the map's stream resolves, waits for them (ev_mid,
// recorded on the aux stream), folds.
template <class Src>
int launch_ndt_tail(vm_map *m, const DevMap &dm, const Src &src, long long n, int maxseg, bool tm,
                    cudaEvent_t walked, cudaEvent_t resolved, cudaEvent_t ev_mid) {
    if (!m->aux_stream) CK(cudaStreamCreateWithFlags(&m->aux_stream, cudaStreamNonBlocking));
    cudaStream_t s = m->stream;
    CK(cudaStreamWaitEvent(m->aux_stream, walked, 0));
    NdtBuckets b;
    int rc = launch_ndt_prep(m, dm, src, n, maxseg, m->aux_stream, &b);
    if (rc) return rc;
    CK(cudaEventRecord(ev_mid, m->aux_stream));
    if (tm) k_resolve<true, true><<<m->num_sms * 8, BLOCK, 0, s>>>(dm);
    else k_resolve<true, false><<<m->num_sms * 8, BLOCK, 0, s>>>(dm);
    m->launches += 1;
    if ((rc = check_launch("resolve"))) return rc;
    CK(cudaEventRecord(resolved, s));
    CK(cudaStreamWaitEvent(s, ev_mid, 0));
    return launch_ndt_fold_only(m, dm, b, tm);
}

// Deterministic TSDF: the band visits bucketed by voxel (the NDT bucket
// kernels, every record a plain ray-order key) and merged per voxel in ray
// order (k_tsdf_fold).
template <class Src>
int launch_tsdf_fold(vm_map *m, const DevMap &dm, const Src &src, long long n, cudaEvent_t ev_mid) {
    cudaStream_t s = m->stream;
    const unsigned long long span = (unsigned long long)n;
    const unsigned long long bwords = (2 * span + 31) / 32 + 1;
    int rc;
    if ((rc = ensure_buckets(m, m->smarked_cap, bwords))) return rc;
    if (!m->d_nbk_small) {
        CK(cudaMalloc((void **)&m->d_nbk_small, (2 * NBK_BINS + 4) * sizeof(unsigned)));
        CK(cudaMemset(m->d_nbk_small, 0, (2 * NBK_BINS + 4) * sizeof(unsigned)));
    }
    if (!m->d_nbk_ctr) CK(cudaMalloc((void **)&m->d_nbk_ctr, 2 * sizeof(unsigned long long)));
    NdtBuckets b{m->d_bk_cnt, m->d_bk_cnt2, m->d_bk_off, m->d_bk_perm, m->d_nbk_small,
                 m->d_nbk_small + NBK_BINS, m->d_rec2, m->d_rec, nullptr, m->d_bk_big,
                 m->d_bk_big2, m->d_nbk_ctr, m->d_nbk_ctr + 1, m->d_bk_bits, bwords, span};
    CK(cudaMemsetAsync(m->d_nbk_ctr, 0, 2 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(b.cursor + NBK_BINS, 0, 2 * sizeof(unsigned), s));
    DevMap d2 = dm;
    d2.recval = nullptr;  // plain keys
    const unsigned gr = (unsigned)m->num_sms * 8;
    const unsigned gm = (unsigned)std::max<long long>(
        1, std::min<long long>((long long)m->num_sms * 8, ((long long)m->smarked_cap + BLOCK - 1) / BLOCK));
    k_nbk_count<<<gr, BLOCK, 0, s>>>(d2, b);
    k_nbk_alloc<<<gm, BLOCK, 0, s>>>(d2, b);
    k_nbk_order<<<1, NBK_BINS, 0, s>>>(d2, b);
    k_nbk_perm<<<gm, BLOCK, 0, s>>>(d2, b);
    k_nbk_scatter<<<gr, BLOCK, 0, s>>>(d2, b);
    k_nbk_sort_small<<<gm, BLOCK, 0, s>>>(d2, b);
    k_nbk_sort_mid<<<m->num_sms * 4, BLOCK, 0, s>>>(d2, b);
    k_nbk_sort_big<<<m->num_sms, BLOCK, 0, s>>>(d2, b);
    CK(cudaEventRecord(ev_mid, s));
    k_tsdf_fold<<<gm, BLOCK, 0, s>>>(d2, src, b);
    m->launches += 9;
    return check_launch("tsdf fold");
}

const uint32_t MODE_MASK[5] = {
    (1u << 1) | (1u << 2) | (1u << 3),
    (1u << 1) | (1u << 2) | (1u << 3) | (1u << 8) | (1u << 9),
    (1u << 1) | (1u << 2) | (1u << 3) | (1u << 4),
    (1u << 1) | (1u << 2) | (1u << 3) | (1u << 4) | (1u << 5) | (1u << 6) | (1u << 7),
    (1u << 10)};

// ---------------------------------------------------------------------------
// Eviction and spill (store.py:120-174): OHMS1 files, byte-compatible with
// the reference's _write_spill / _reload_region: b"OHMS1", <3q I> region key
// and layer count, u32 layer ids, zlib(level 6) of the layers' bytes in the
// host map's layer order.  A spilled region keeps its key in the device
// table with SLOT_SPILLED, so a batch that reaches it is refused by the guard
// and replayed after the reload (integrate_impl, integrate_pipelined).

std::string spill_path(const vm_map *m, long long key) {
    int r[3];
    unpack_region(key, r);
    return m->spill_dir + "/region_" + std::to_string(r[0]) + "_" + std::to_string(r[1]) + "_" +
           std::to_string(r[2]) + ".bin";
}

__global__ void k_revive(const __grid_constant__ DevMap m, long long key, int *slot_out) {
    // the table entry of a spilled key takes a fresh slot
    unsigned long long h = mix_key(key) & m.tmask;
    for (unsigned long long p = 0; p <= m.tmask; ++p) {
        const long long k = m.tkeys[h];
        if (k == key) {
            const int v = m.tvals[h];
            if (v == SLOT_SPILLED) {
                const int s = atomicAdd(m.cursor, 1);
                m.slot_keys[s] = key;
                m.tvals[h] = s;
                *slot_out = s;
            } else {
                *slot_out = v;
            }
            return;
        }
        if (k == -1) break;
        h = (h + 1) & m.tmask;
    }
    *slot_out = -1;
}

// Reload one spilled region from its file into a fresh slot (the file is
// consumed, store.py:145-170).  *slot_out = -1 if the key is not spilled.
int reload_region(vm_map *m, long long key, int *slot_out) {
    *slot_out = -1;
    if (!m->spilled.count(key)) return VM_OK;
    const std::string path = spill_path(m, key);
    FILE *f = std::fopen(path.c_str(), "rb");
    if (!f) return fail(VM_ERR_ARG, "spill file missing: " + path);
    std::vector<unsigned char> raw;
    {
        unsigned char buf[1 << 16];
        size_t k;
        while ((k = std::fread(buf, 1, sizeof(buf), f)) > 0) raw.insert(raw.end(), buf, buf + k);
        std::fclose(f);
    }
    const size_t nl = m->spill_ids.size();
    const size_t hdr = 5 + 28 + 4 * nl;
    if (raw.size() < hdr || std::memcmp(raw.data(), "OHMS1", 5) != 0)
        return fail(VM_ERR_ARG, "bad spill file " + path);
    long long k3[3];
    uint32_t nlayers;
    std::memcpy(k3, raw.data() + 5, 24);
    std::memcpy(&nlayers, raw.data() + 29, 4);
    int r[3];
    unpack_region(key, r);
    bool ok = k3[0] == r[0] && k3[1] == r[1] && k3[2] == r[2] && nlayers == nl;
    for (size_t i = 0; ok && i < nl; ++i) {
        uint32_t id;
        std::memcpy(&id, raw.data() + 33 + 4 * i, 4);
        ok = (int)id == m->spill_ids[i];
    }
    if (!ok) return fail(VM_ERR_ARG, "spill file " + path + " does not match map layout");
    size_t total = 0;
    for (int id : m->spill_ids) total += m->bpr[id];
    std::vector<unsigned char> payload(total);
    uLongf got = (uLongf)total;
    if (uncompress(payload.data(), &got, raw.data() + hdr, (uLong)(raw.size() - hdr)) != Z_OK ||
        got != total)
        return fail(VM_ERR_ARG, "corrupt spill file " + path);
    CK(cudaSetDevice(m->device));
    if (m->nreg + 1 > m->cap) {
        int rc = grow_pool(m, std::max<long long>(2 * m->cap, m->nreg + 64));
        if (rc) return rc;
    }
    int *d_slot = nullptr;
    CK(cudaMalloc(&d_slot, sizeof(int)));
    k_revive<<<1, 1, 0, m->stream>>>(make_dm(m), key, d_slot);
    int slot = -1;
    CK(cudaMemcpyAsync(&slot, d_slot, sizeof(int), cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    cudaFree(d_slot);
    if (slot < 0 || slot >= m->cap) return fail(VM_ERR_CUDA, "spilled region lost its table entry");
    size_t pos = 0;
    for (int id : m->spill_ids) {
        CK(cudaMemcpyAsync((char *)m->slab[id] + (size_t)slot * m->bpr[id], payload.data() + pos,
                           m->bpr[id], cudaMemcpyHostToDevice, m->stream));
        pos += m->bpr[id];
    }
    const unsigned last = m->batch_no;
    CK(cudaMemcpyAsync(m->d_slot_last + slot, &last, sizeof(unsigned), cudaMemcpyHostToDevice,
                       m->stream));
    CK(cudaMemsetAsync(m->d_gmask + slot, 0xFF, sizeof(unsigned), m->stream));  // conservative
    CK(cudaStreamSynchronize(m->stream));
    m->spilled.erase(key);
    std::remove(path.c_str());
    m->nreg = std::max<long long>(m->nreg, slot + 1);
    *slot_out = slot;
    return VM_OK;
}

// the spilled regions a refused attempt listed (stats already on the host)
int reload_listed(vm_map *m, unsigned long long listed) {
    const unsigned long long n = std::min<unsigned long long>(listed, RELOAD_CAP);
    std::vector<long long> keys(n);
    if (n) CK(cudaMemcpy(keys.data(), m->d_reload, n * sizeof(long long), cudaMemcpyDeviceToHost));
    std::set<long long> uniq(keys.begin(), keys.end());
    for (long long k : uniq) {
        int slot, rc = reload_region(m, k, &slot);
        if (rc) return rc;
    }
    return VM_OK;
}

template <class Src>
int integrate_impl(vm_map *m, const Src &src, long long n, int mode, int exec, vm_stats *out) {
    const bool ndt = mode == M_NDT_OM || mode == M_NDT_TM;
    const bool tsdf = mode == M_TSDF;
    const bool det = exec == VM_EXEC_DETERMINISTIC;
    const bool occ_det = det && (mode == M_OCC || mode == M_DECAY);
    const bool tsdf_det = tsdf && det;
    // occupancy on a sharded map: a sorted fold; NDT and TSDF: voxel buckets
    // (launch_ndt_fold / launch_tsdf_fold); occupancy on one GPU: sample-voxel
    // buckets (launch_bucket_fold)
    const bool sorted = occ_det;
    const bool vbuck = ndt || tsdf_det;  // records keyed by a claimed voxel index (L_NIDX)
    const bool resolve = occ_det || ndt;
    const int maxseg = (int)std::ceil(m->cfg.max_ray_range / m->cfg.segment_length) + 1;
    unsigned long long order_span = tsdf ? (unsigned long long)n
                                         : ((unsigned long long)n * maxseg) << 1;
    if (order_span >= (1ULL << 32))
        return fail(VM_ERR_ARG, "batch too large for 32-bit ray order keys; split it");
    const int order_bits = std::max(1, bitlen(order_span));
    // record keys: voxel id above the order bits, bit 63 free (walk candidates)
    if (order_bits + 1 + bitlen((unsigned long long)m->max_slots * (unsigned long long)m->vpr) > 63)
        return fail(VM_ERR_ARG, "batch too large for 64-bit record keys; split it");

    int rc;
    // deterministic NDT on one GPU walks segment descriptors (k_walk_ndt_det)
    const bool ndt_seg = ndt && det && m->shard_world == 1 && !m->ndt_generic;
    const bool emit = mode == M_OCC || mode == M_DECAY || ndt_seg;
    if (emit && (rc = ensure_buf(&m->d_segs, &m->seg_cap, (size_t)n * maxseg + 1))) return rc;
    if (emit && (rc = ensure_buf(&m->d_perm, &m->perm_cap, m->seg_cap))) return rc;
    if (emit && (rc = ensure_buf(&m->d_seg_bk, &m->seg_bk_cap, m->seg_cap))) return rc;
    // generic NDT walks take their rays longest first (k_discover buckets, k_seg_scatter orders)
    const bool ray_order = ndt && !ndt_seg && !m->no_ray_order;
    if (ray_order && (rc = ensure_buf(&m->d_perm, &m->perm_cap, (size_t)n + 1))) return rc;
    if (ray_order && (rc = ensure_buf(&m->d_seg_bk, &m->seg_bk_cap, (size_t)n + 1))) return rc;
    // occupancy / decay records key on the index in the batch's sample-voxel list
    const bool key_mi = occ_det && m->shard_world == 1;
    if (key_mi) {
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, (size_t)n + 1))) return rc;
        CK(cudaMemsetAsync(m->d_shard_cnt, 0, 2 * sizeof(unsigned long long), m->stream));
    }
    if (ndt) {
        // records keyed by the voxel index (vm_ndt.cuh): one list entry per record at most
        const size_t need = m->ndt_rec_override > 0 ? (size_t)m->ndt_rec_override
                                                     : (size_t)n * (det ? 8 : 1) + 1;
        if ((rc = ensure_records(m, std::max<size_t>(m->rec_cap, need)))) return rc;
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_rec_t, &m->rec_t_cap, m->rec_cap))) return rc;
        CK(cudaMemsetAsync(m->d_shard_cnt, 0, sizeof(unsigned long long), m->stream));
        CK(cudaMemsetAsync(m->d_nlost, 0, sizeof(unsigned long long), m->stream));
    }
    if (tsdf_det) {
        // at most one record per band visit: an upper bound, no overflow path
        const double band = 2.0 * m->cfg.tsdf_truncation / m->cfg.voxel_size;
        const size_t need = (size_t)n * (size_t)(3.0 * (std::ceil(band) + 2.0) + 4.0) + 1;
        if ((rc = ensure_records(m, std::max<size_t>(m->rec_cap, need)))) return rc;
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, m->rec_cap))) return rc;
        CK(cudaMemsetAsync(m->d_shard_cnt, 0, sizeof(unsigned long long), m->stream));
        CK(cudaMemsetAsync(m->d_nlost, 0, sizeof(unsigned long long), m->stream));
    }
    size_t rec_need = 0;
    if (occ_det) rec_need = std::max<size_t>(m->rec_cap, rec_floor(m, n));
    if (sorted && (rc = ensure_records(m, rec_need))) return rc;

    float ms_total = 0.f, ms_walk = 0.f, ms_disc = 0.f, ms_res = 0.f, ms_sort = 0.f, ms_fold = 0.f;
    const long long launches0 = m->launches;
    long long replays = 0;
    const long long nreg0 = m->nreg;
    for (;;) {
        long long headroom = std::max<long long>(512, 2 * m->max_growth);
        if (m->nreg + headroom > m->cap) {
            if ((rc = grow_pool(m, std::max(2 * m->cap, m->nreg + headroom)))) return rc;
        }
        m->epoch += 1;
        DevMap dm = make_dm(m);
        dm.order_bits = order_bits;
        dm.ray_order = ray_order ? 1 : 0;
        dm.ndt_segs = ndt_seg ? 1 : 0;
        if (key_mi || vbuck) {
            dm.key_mi = key_mi ? 1 : 0;
            dm.nlost = vbuck && m->shard_world == 1 ? m->d_nlost : nullptr;
            dm.marked = m->d_smarked;
            dm.nmarked = m->d_shard_cnt;
            dm.marked_cap = m->smarked_cap;
        }
        CK(cudaMemsetAsync(m->d_stats, 0, NUM_STATS * sizeof(unsigned long long), m->stream));
        {
            static const int box_init[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
            CK(cudaMemcpyAsync(m->d_rbox, box_init, sizeof(box_init), cudaMemcpyHostToDevice,
                               m->stream));
        }
        CK(cudaEventRecord(m->ev_start, m->stream));
        if (m->up.pending) {
            // host rays: chunk c is copied on copy_stream while chunk c-1 is discovered
            const int nc = n >= 65536 ? vm_map::UP_CHUNKS : 1;
            CK(cudaEventRecord(m->ev_up[0], m->stream));  // the previous batch is done with d_rays
            CK(cudaStreamWaitEvent(m->copy_stream, m->ev_up[0], 0));
            for (int c = 0; c < nc; ++c) {
                const long long lo = n * c / nc, hi = n * (c + 1) / nc;
                if (hi <= lo) continue;
                const auto &u = m->up;
                if (u.format == VM_RAYS_OHMB1) {
                    CK(cudaMemcpyAsync(m->d_rays + (size_t)lo * 40, u.rec + (size_t)lo * 40,
                                       (size_t)(hi - lo) * 40, cudaMemcpyHostToDevice, m->copy_stream));
                } else {
                    unsigned char *d = m->d_rays;
                    CK(cudaMemcpyAsync(d + lo * 24, (const unsigned char *)u.o + lo * 24, (hi - lo) * 24,
                                       cudaMemcpyHostToDevice, m->copy_stream));
                    CK(cudaMemcpyAsync(d + u.b_o + lo * 24, (const unsigned char *)u.e + lo * 24,
                                       (hi - lo) * 24, cudaMemcpyHostToDevice, m->copy_stream));
                    CK(cudaMemcpyAsync(d + 2 * u.b_o + lo, u.h + lo, hi - lo, cudaMemcpyHostToDevice,
                                       m->copy_stream));
                    if (u.it)
                        CK(cudaMemcpyAsync(d + 2 * u.b_o + u.b_h + lo * 4, (const unsigned char *)u.it + lo * 4,
                                           (hi - lo) * 4, cudaMemcpyHostToDevice, m->copy_stream));
                }
                CK(cudaEventRecord(m->ev_up[c], m->copy_stream));
                CK(cudaStreamWaitEvent(m->stream, m->ev_up[c], 0));
                DevMap dc = dm;
                dc.ray_lo = lo;
                if ((rc = launch_discover(m, dc, src, hi - lo, mode, det ? 1 : 0, emit ? 1 : 0, 1,
                                          m->stream)))
                    return rc;
            }
            m->up.pending = 0;
            m->launches += 1;  // guard
        } else {
            if ((rc = launch_discover(m, dm, src, n, mode, det ? 1 : 0, emit ? 1 : 0, 1, m->stream)))
                return rc;
            m->launches += 1;  // guard
        }
        if ((rc = check_launch("discover"))) return rc;
        int margin = 64 + (int)std::min<long long>(1 << 20, headroom / 4);
        k_guard<<<1, 1, 0, m->stream>>>(dm, margin);
        if (emit) {
            if (key_mi) {
                k_stamp<<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
                m->launches += 1;
            }
            k_rgrid<<<16, BLOCK, 0, m->stream>>>(dm);
            k_seg_scan<<<1, SEG_BUCKETS, 0, m->stream>>>(dm);
            k_seg_scatter<<<(unsigned)((n * maxseg + BLOCK - 1) / BLOCK), BLOCK, 0, m->stream>>>(dm);
            m->launches += 3;
        } else if (ray_order) {
            k_seg_scan<<<1, SEG_BUCKETS, 0, m->stream>>>(dm);
            k_seg_scatter<<<(unsigned)((n + BLOCK - 1) / BLOCK), BLOCK, 0, m->stream>>>(dm, n);
            m->launches += 2;
        }
        CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaMemcpyAsync(m->h_stats + NUM_STATS, m->d_cursor, sizeof(int),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaMemcpyAsync((int *)(m->h_stats + NUM_STATS) + 1, m->d_go, sizeof(int),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaEventRecord(m->ev_k1, m->stream));
        CK(cudaEventRecord(m->ev_w0, m->stream));
        if ((rc = launch_walk(m, dm, src, n, mode, det, false))) return rc;
        CK(cudaEventRecord(m->ev_w1, m->stream));
        if (sorted) {
            CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 1, m->d_stats + S_RECORDS,
                               sizeof(unsigned long long), cudaMemcpyDeviceToHost, m->stream));
            CK(cudaEventRecord(m->ev_k2, m->stream));
        }
        // deterministic NDT on one GPU: k_resolve runs inside launch_ndt_tail
        const bool ndt_tail = ndt && det && m->shard_world == 1;
        if (resolve && !ndt_tail) {
            if (ndt && mode == M_NDT_TM) k_resolve<true, true><<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
            else if (ndt) k_resolve<true, false><<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
            else k_resolve<false, false><<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
            m->launches += 1;
            if ((rc = check_launch("resolve"))) return rc;
        }
        if (!ndt_tail) CK(cudaEventRecord(m->ev_res, m->stream));
        if (key_mi || vbuck) {
            // the whole batch is enqueued; one sync at its end
            if (ndt_tail)
                rc = launch_ndt_tail(m, dm, src, n, maxseg, mode == M_NDT_TM, m->ev_w1, m->ev_res,
                                     m->ev_sort);
            else if (ndt) rc = launch_ndt_fold(m, dm, src, n, maxseg, mode == M_NDT_TM, m->ev_sort);
            else if (tsdf_det) rc = launch_tsdf_fold(m, dm, src, n, m->ev_sort);
            else rc = launch_bucket_fold(m, dm, src, n, maxseg, m->ev_sort);
            if (rc) return rc;
            CK(cudaEventRecord(m->ev_end, m->stream));
            CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, m->stream));
            CK(cudaMemcpyAsync(m->h_stats + NUM_STATS, m->d_cursor, sizeof(int),
                               cudaMemcpyDeviceToHost, m->stream));
            CK(cudaMemcpyAsync((int *)(m->h_stats + NUM_STATS) + 1, m->d_go, sizeof(int),
                               cudaMemcpyDeviceToHost, m->stream));
            CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 1, m->d_shard_cnt,
                               2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, m->stream));
            CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 3, m->d_nlost, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, m->stream));
            CK(cudaStreamSynchronize(m->stream));
            if ((rc = check_launch("batch"))) return rc;
            if (!key_mi) m->h_stats[NUM_STATS + 2] = 0;
            if (!dm.nlost) m->h_stats[NUM_STATS + 3] = 0;
        } else {
            CK(cudaEventSynchronize(m->ev_k1));
        }
        const unsigned long long *hs = m->h_stats;
        int cursor = *(const int *)(hs + NUM_STATS);
        int go = *((const int *)(hs + NUM_STATS) + 1);
        if (hs[S_RANGE_ERR]) {
            CK(cudaStreamSynchronize(m->stream));
            if (occ_det && hs[S_MARKED]) {
                const long long words = std::min<long long>(cursor, m->cap) * (long long)m->vpr;
                k_clear_marks<<<m->num_sms * 4, BLOCK, 0, m->stream>>>(dm, words);
            }
            if (vbuck || key_mi) {
                const long long words = std::min<long long>(cursor, m->cap) * (long long)m->vpr;
                k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, m->stream>>>(dm, words);
            }
            CK(cudaStreamSynchronize(m->stream));
            m->nreg = cursor;
            return fail(VM_ERR_RANGE, "ray coordinates outside the packable region range "
                                      "(|region| < 2**20, keys.py:76-86)");
        }
        if (!go && hs[S_SPILLED]) {
            // the batch reaches regions spilled to disk: reload them, replay
            CK(cudaStreamSynchronize(m->stream));
            m->nreg = cursor;
            if ((rc = reload_listed(m, hs[S_SPILLED]))) return rc;
            ++replays;
            continue;
        }
        if (!go) {
            // pool overflow: nothing was applied (the sample-voxel stamps are
            // idempotent and re-made by the replay); grow and replay
            CK(cudaStreamSynchronize(m->stream));
            m->max_growth = std::max<long long>(m->max_growth, cursor - m->nreg);
            if ((rc = grow_pool(m, std::max<long long>(2 * m->cap,
                                                       cursor + 2 * margin + headroom))))
                return rc;
            if (cursor + margin > m->cap)
                return fail(VM_ERR_OOM, "region pool exhausted (max regions reached)");
            m->nreg = cursor;
            ++replays;
            continue;
        }
        if (tsdf_det) {
            if (m->h_stats[S_RECORDS] > m->rec_cap || m->h_stats[NUM_STATS + 1] > m->smarked_cap) {
                m->nreg = cursor;  // the regions the discover created stay (like the reference's prefetch)
                return fail(VM_ERR_CUDA, "TSDF record bound exceeded");
            }
            CK(cudaEventElapsedTime(&ms_total, m->ev_start, m->ev_end));
            CK(cudaEventElapsedTime(&ms_walk, m->ev_w0, m->ev_w1));
            CK(cudaEventElapsedTime(&ms_disc, m->ev_start, m->ev_w0));
            CK(cudaEventElapsedTime(&ms_res, m->ev_w1, m->ev_res));
            CK(cudaEventElapsedTime(&ms_sort, m->ev_res, m->ev_sort));
            CK(cudaEventElapsedTime(&ms_fold, m->ev_sort, m->ev_end));
            break;
        }
        if (ndt) {
            unsigned long long R = m->h_stats[S_RECORDS], M = m->h_stats[NUM_STATS + 1];
            if (R > m->rec_cap || M > m->smarked_cap) {
                // records or voxel indices overflowed: every bucket kernel was a
                // no-op.  Drop the index stamps, make room, re-emit the records
                // only (discover without descriptors, histograms or statistics;
                // the walk without counts) and fold them.
                const long long words = std::min<long long>(cursor, m->cap) * (long long)m->vpr;
                k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, m->stream>>>(dm, words);
                if ((rc = ensure_records(m, std::max<size_t>((size_t)R + (R >> 2), m->rec_cap)))) return rc;
                if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, m->rec_cap))) return rc;
                if ((rc = ensure_buf(&m->d_rec_t, &m->rec_t_cap, m->rec_cap))) return rc;
                dm.rec = m->d_rec;
                dm.recval = m->d_val;
                dm.rec_t = m->d_rec_t;
                dm.rec_cap = m->rec_cap;
                dm.marked = m->d_smarked;
                dm.marked_cap = m->smarked_cap;
                dm.ray_order = 0;
                CK(cudaMemsetAsync(m->d_stats + S_RECORDS, 0, sizeof(unsigned long long), m->stream));
                CK(cudaMemsetAsync(m->d_shard_cnt, 0, sizeof(unsigned long long), m->stream));
                CK(cudaMemsetAsync(m->d_nlost, 0, sizeof(unsigned long long), m->stream));
                if ((rc = launch_discover(m, dm, src, n, mode, 1, 0, 0, m->stream))) return rc;
                if (det && (rc = launch_walk(m, dm, src, n, mode, det, true))) return rc;
                CK(cudaEventRecord(m->ev_res, m->stream));
                if ((rc = launch_ndt_fold(m, dm, src, n, maxseg, mode == M_NDT_TM, m->ev_sort))) return rc;
                CK(cudaEventRecord(m->ev_end, m->stream));
                CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, m->stream));
                CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 1, m->d_shard_cnt,
                                   sizeof(unsigned long long), cudaMemcpyDeviceToHost, m->stream));
                CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 3, m->d_nlost, sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, m->stream));
                CK(cudaStreamSynchronize(m->stream));
                if ((rc = check_launch("batch"))) return rc;
                if (m->h_stats[S_RECORDS] > m->rec_cap || m->h_stats[NUM_STATS + 1] > m->smarked_cap) {
                    m->nreg = cursor;
                    return fail(VM_ERR_CUDA, "NDT record re-emission overflowed");
                }
            }
            CK(cudaEventElapsedTime(&ms_total, m->ev_start, m->ev_end));
            CK(cudaEventElapsedTime(&ms_walk, m->ev_w0, m->ev_w1));
            CK(cudaEventElapsedTime(&ms_disc, m->ev_start, m->ev_w0));
            CK(cudaEventElapsedTime(&ms_res, m->ev_w1, m->ev_res));
            CK(cudaEventElapsedTime(&ms_sort, m->ev_res, m->ev_sort));
            CK(cudaEventElapsedTime(&ms_fold, m->ev_sort, m->ev_end));
            if (ms_sort < 0.f) {  // the buckets were ready before k_resolve ended
                ms_fold += ms_sort;
                ms_sort = 0.f;
            }
            break;
        }
        if (key_mi) {
            unsigned long long R = m->h_stats[S_RECORDS];
            if (R > m->rec_cap) {
                // records overflowed: every fold kernel was a no-op; re-emit
                // the records (nothing re-applied) and fold them
                if ((rc = ensure_records(m, (size_t)R + (R >> 2)))) return rc;
                dm.rec = m->d_rec;
                dm.recval = m->d_val;
                dm.rec_cap = m->rec_cap;
                CK(cudaMemsetAsync(m->d_stats + S_RECORDS, 0, sizeof(unsigned long long),
                                   m->stream));
                if ((rc = launch_walk(m, dm, src, n, mode, det, true))) return rc;
                CK(cudaEventRecord(m->ev_res, m->stream));
                if ((rc = launch_bucket_fold(m, dm, src, n, maxseg, m->ev_sort))) return rc;
                CK(cudaEventRecord(m->ev_end, m->stream));
                CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, m->stream));
                CK(cudaStreamSynchronize(m->stream));
                if ((rc = check_launch("batch"))) return rc;
            }
            CK(cudaEventElapsedTime(&ms_total, m->ev_start, m->ev_end));
            CK(cudaEventElapsedTime(&ms_walk, m->ev_w0, m->ev_w1));
            CK(cudaEventElapsedTime(&ms_disc, m->ev_start, m->ev_w0));
            CK(cudaEventElapsedTime(&ms_res, m->ev_w1, m->ev_res));
            CK(cudaEventElapsedTime(&ms_sort, m->ev_res, m->ev_sort));
            CK(cudaEventElapsedTime(&ms_fold, m->ev_sort, m->ev_end));
            break;
        }
        if (sorted) {
            CK(cudaEventSynchronize(m->ev_k2));
            unsigned long long R = m->h_stats[NUM_STATS + 1];
            if (R > m->rec_cap) {
                // records overflowed: re-emit them (records only, nothing re-applied)
                if (!occ_det) return fail(VM_ERR_CUDA, "record buffer overflow");
                CK(cudaStreamSynchronize(m->stream));
                if ((rc = ensure_records(m, (size_t)R + (R >> 2)))) return rc;
                dm.rec = m->d_rec;
                dm.recval = m->d_val;
                dm.rec_cap = m->rec_cap;
                CK(cudaMemsetAsync(m->d_stats + S_RECORDS, 0, sizeof(unsigned long long),
                                   m->stream));
                if ((rc = launch_walk(m, dm, src, n, mode, det, true))) return rc;
                CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 1, m->d_stats + S_RECORDS,
                                   sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   m->stream));
                CK(cudaStreamSynchronize(m->stream));
                R = m->h_stats[NUM_STATS + 1];
            }
            int end_bit = order_bits +
                          std::max(1, bitlen((unsigned long long)(cursor + 1) * m->vpr));
            if (key_mi) {
                unsigned long long M = 0;
                CK(cudaMemcpy(&M, m->d_shard_cnt, sizeof(M), cudaMemcpyDeviceToHost));
                end_bit = order_bits + std::max(1, bitlen(std::min<unsigned long long>(M, m->smarked_cap)));
            }
            end_bit = std::min(end_bit, 64);
            cub::DoubleBuffer<unsigned long long> db(m->d_rec, m->d_rec2);
            cub::DoubleBuffer<unsigned> dv(m->d_val, m->d_val2);
            if (R > 1) {
                if ((rc = ensure_sort_tmp(m))) return rc;
                size_t bytes = m->sort_tmp_bytes;
                CK(cub::DeviceRadixSort::SortKeys(m->d_sort_tmp, bytes, db, (int)R, 0, end_bit,
                                                  m->stream));
            }
            CK(cudaEventRecord(m->ev_sort, m->stream));
            if ((rc = launch_fold(m, dm, src, db.Current(), dv.Current(), (long long)R, mode)))
                return rc;
        }
        CK(cudaEventRecord(m->ev_end, m->stream));
        CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaMemcpyAsync(m->h_stats + NUM_STATS, m->d_cursor, sizeof(int),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaStreamSynchronize(m->stream));
        if ((rc = check_launch("batch"))) return rc;
        CK(cudaEventElapsedTime(&ms_total, m->ev_start, m->ev_end));
        CK(cudaEventElapsedTime(&ms_walk, m->ev_w0, m->ev_w1));
        CK(cudaEventElapsedTime(&ms_disc, m->ev_start, m->ev_w0));
        CK(cudaEventElapsedTime(&ms_res, m->ev_w1, m->ev_res));
        if (sorted) {
            CK(cudaEventElapsedTime(&ms_sort, m->ev_res, m->ev_sort));
            CK(cudaEventElapsedTime(&ms_fold, m->ev_sort, m->ev_end));
        }
        break;
    }
    const unsigned long long *hs = m->h_stats;
    int cursor = *(const int *)(hs + NUM_STATS);
    std::memset(out, 0, sizeof(*out));
    out->rays_in = n;
    out->rays_processed = (int64_t)hs[S_PROCESSED];
    out->segments = (int64_t)hs[S_SEGMENTS];
    out->voxel_visits = (int64_t)hs[S_VISITS];
    out->cas_retries = (int64_t)hs[S_RETRIES];
    out->cas_failures = 0;
    out->region_misses = (int64_t)hs[S_RMISS];
    out->regions_touched = (int64_t)hs[S_PREF_TOUCHED];
    out->records = (int64_t)hs[S_RECORDS];
    out->marked_voxels = key_mi   ? (int64_t)(hs[NUM_STATS + 1] - hs[NUM_STATS + 2])
                         : vbuck ? (int64_t)(hs[NUM_STATS + 1] - hs[NUM_STATS + 3])
                                 : (int64_t)hs[S_MARKED];
    out->regions_total = cursor;
    out->new_regions = cursor - nreg0;
    out->replays = replays;
    out->touched_regions_walk = (int64_t)hs[S_WALK_TOUCHED];
    out->launches = m->launches - launches0;
    out->gpu_ms = ms_total;
    out->walk_ms = ms_walk;
    out->discover_ms = ms_disc;
    out->resolve_ms = ms_res;
    out->sort_ms = ms_sort;
    out->fold_ms = ms_fold;
    m->max_growth = std::max<long long>(m->max_growth, cursor - m->nreg);
    m->nreg = cursor;
    return VM_OK;
}

// ---------------------------------------------------------------------------
// Pipelined sequences of deterministic occupancy batches (vm_integrate_many).
//
// Every batch is enqueued behind the previous one with no host round trip
// (the bucketed fold reads all its counts on the device); host records are
// uploaded on copy_stream into a ring of device buffers while earlier batches
// compute.  One sync at the end of the sequence.  The first batch the guard
// refuses (region pool growth, invalid coordinates) or whose records
// overflow sets the chain flag: every later batch is a no-op, the host
// recovers that batch exactly as integrate_impl would and re-enqueues the rest.
constexpr int MSTRIDE = NUM_STATS + 2;  // per-batch slot: stats, cursor after, fin flags

void fill_stats(const unsigned long long *slot, long long n, long long regions_before,
                vm_stats *o) {
    std::memset(o, 0, sizeof(*o));
    o->rays_in = n;
    o->rays_processed = (int64_t)slot[S_PROCESSED];
    o->segments = (int64_t)slot[S_SEGMENTS];
    o->voxel_visits = (int64_t)slot[S_VISITS];
    o->cas_retries = (int64_t)slot[S_RETRIES];
    o->region_misses = (int64_t)slot[S_RMISS];
    o->regions_touched = (int64_t)slot[S_PREF_TOUCHED];
    o->records = (int64_t)slot[S_RECORDS];
    o->marked_voxels = (int64_t)slot[S_MARKED];
    o->regions_total = (int64_t)slot[NUM_STATS];
    o->new_regions = o->regions_total - regions_before;
    o->touched_regions_walk = (int64_t)slot[S_WALK_TOUCHED];
}

// per-batch stats slots, 8 events per batch, the host-upload ring
int sequence_buffers(vm_map *m, int nb, long long nmax, bool any_host) {
    if ((size_t)nb > m->mstats_cap) {
        cudaFree(m->d_mstats);
        if (m->h_mstats) cudaFreeHost(m->h_mstats);
        m->d_mstats = nullptr;
        m->h_mstats = nullptr;
        CK(cudaMalloc((void **)&m->d_mstats, (size_t)nb * MSTRIDE * sizeof(unsigned long long)));
        CK(cudaMallocHost((void **)&m->h_mstats, (size_t)nb * MSTRIDE * sizeof(unsigned long long)));
        m->mstats_cap = nb;
    }
    while (m->mev.size() < (size_t)nb * 8) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        m->mev.push_back(e);
    }
    if (any_host && (size_t)nmax * 40 > m->ring_bytes) {
        for (int r = 0; r < vm_map::RING; ++r) {
            cudaFree(m->d_ring[r]);
            m->d_ring[r] = nullptr;
            CK(cudaMalloc((void **)&m->d_ring[r], (size_t)nmax * 40));
            if (!m->ev_ring[r]) CK(cudaEventCreateWithFlags(&m->ev_ring[r], cudaEventDisableTiming));
            if (!m->ev_ring_up[r])
                CK(cudaEventCreateWithFlags(&m->ev_ring_up[r], cudaEventDisableTiming));
        }
        m->ring_bytes = (size_t)nmax * 40;
    }
    return VM_OK;
}

// stage times of a finished sequence (events 0..6 of each batch)
int sequence_times(vm_map *m, const vm_rays *rays, int nb, const std::vector<long long> &reps,
                   const std::vector<long long> &launches, vm_stats *out) {
    for (int b = 0; b < nb; ++b) {
        if (rays[b].count <= 0) continue;
        cudaEvent_t *ev = &m->mev[(size_t)8 * b];
        float t[5] = {0, 0, 0, 0, 0}, tot = 0;
        CK(cudaEventElapsedTime(&tot, ev[0], ev[5]));
        for (int k = 0; k < 5; ++k) CK(cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]));
        CK(cudaEventElapsedTime(&t[1], ev[6], ev[2]));  // the walk itself (not the wait for b-1)
        if (t[3] < 0.f) {  // NDT: the buckets were ready before k_resolve ended
            t[4] += t[3];
            t[3] = 0.f;
        }
        out[b].gpu_ms = tot;
        out[b].discover_ms = t[0];
        out[b].walk_ms = t[1];
        out[b].resolve_ms = t[2];
        out[b].sort_ms = t[3];
        out[b].fold_ms = t[4];
        out[b].replays = reps[b];
        out[b].launches = launches[b];
    }
    return VM_OK;
}

// the discover stream and the batch-scoped buffers of parity 1
int ensure_disc_stream(vm_map *m) {
    int rc;
    if (!m->disc_stream) {
        CK(cudaStreamCreateWithFlags(&m->disc_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&m->ev_seq0, cudaEventDisableTiming));
        if ((rc = dev_alloc(&m->d_touched2, m->max_slots)) || (rc = dev_alloc(&m->d_rgrid2, RG_MAX)) ||
            (rc = dev_alloc(&m->d_rbox2, 6)) || (rc = dev_alloc(&m->d_go2, 1)) ||
            (rc = dev_alloc(&m->d_mk2, 2)) || (rc = dev_alloc(&m->d_nlost2, 1)))
            return rc;
    }
    return VM_OK;
}

// Pipelined sequences of deterministic NDT-OM / NDT-TM batches: every batch is
// integrate_impl's NDT path enqueued behind the previous one (its counts are
// all read on the device), host records uploaded on copy_stream into the
// ring.  One sync per sequence.  Batch b+1's discover runs on disc_stream
// while batch b folds (the fold's long serial tail leaves most SMs idle): it
// starts once b's k_resolve and bucket kernels are done, claims its voxel
// indices in the other index layer (L_NIDX2 for odd batches) with its own
// index list, counters and guard flag; b+1's walk follows b's fold on the
// map's stream.  A guard refusal or a record / voxel-index overflow stops
// the chain at that batch (later batches are no-ops); the host recovers it
// exactly as integrate_impl does and re-enqueues the rest.
int integrate_pipelined_ndt(vm_map *m, const vm_rays *rays, int nb, int mode, vm_stats *out,
                            int maxseg, long long nmax, bool any_host, bool ray_order) {
    cudaStream_t s = m->stream;
    const bool tm = mode == M_NDT_TM;
    int rc;
    if ((rc = sequence_buffers(m, nb, nmax, any_host))) return rc;
    if ((rc = ensure_disc_stream(m))) return rc;
    if ((rc = ensure_buf(&m->d_smarked2, &m->smarked2_cap, m->smarked_cap))) return rc;
    cudaStream_t ds = m->disc_stream;
    // batch-scoped state of odd batches; parity = position among the
    // non-empty batches (consecutive batches alternate, an empty one between or not)
    std::vector<int> par(nb, 0);
    for (int b = 0, k = 0; b < nb; ++b)
        if (rays[b].count > 0) par[b] = (k++) & 1;
    auto parity = [&](DevMap &dm, int b) {
        if (!par[b]) return;
        dm.nidx = L_NIDX2;
        dm.go = m->d_go2;
        dm.marked = m->d_smarked2;
        dm.nmarked = m->d_mk2;
        dm.marked_cap = m->smarked2_cap;
        dm.nlost = m->d_nlost2;
    };
    std::vector<DevMap> dms(nb);
    std::vector<const unsigned char *> srcp(nb, nullptr);
    std::vector<long long> reps(nb, 0), launches(nb, 0), before(nb, 0), first_before(nb, -1);
    bool keep_claims = false;  // a replayed batch keeps its voxel-index claims (integrate_impl)
    int b0 = 0;
    while (b0 < nb) {
        const long long headroom = std::max<long long>(512, 2 * m->max_growth);
        if (m->nreg + headroom > m->cap &&
            (rc = grow_pool(m, std::max(2 * m->cap, m->nreg + headroom))))
            return rc;
        const int margin = 64 + (int)std::min<long long>(1 << 20, headroom / 4);
        CK(cudaMemsetAsync(m->d_chain, 0, sizeof(int), s));
        CK(cudaEventRecord(m->ev_seq0, s));  // the discover stream starts after the map's prior work
        CK(cudaStreamWaitEvent(ds, m->ev_seq0, 0));
        for (int b = b0; b < nb; ++b) {
            const long long n = rays[b].count;
            cudaEvent_t *ev = &m->mev[(size_t)8 * b];
            if (n <= 0) continue;
            m->epoch += 1;
            DevMap dm = make_dm(m);
            dm.batch_no = m->batch_no + (unsigned)b;
            dm.order_bits = std::max(1, bitlen(((unsigned long long)n * maxseg) << 1));
            dm.ray_order = ray_order ? 1 : 0;
            dm.ndt_segs = m->ndt_generic ? 0 : 1;
            dm.key_mi = 0;
            dm.nlost = m->d_nlost;
            dm.marked = m->d_smarked;
            dm.nmarked = m->d_shard_cnt;
            dm.marked_cap = m->smarked_cap;
            dm.stats = m->d_mstats + (size_t)b * MSTRIDE;
            dm.chain = m->d_chain;
            dm.batch_idx = b;
            parity(dm, b);
            if (rays[b].on_device) {
                srcp[b] = (const unsigned char *)rays[b].records;
            } else {
                const int r = b % vm_map::RING;
                CK(cudaStreamWaitEvent(m->copy_stream, m->ev_ring[r], 0));  // the slot's last batch is done
                CK(cudaMemcpyAsync(m->d_ring[r], rays[b].records, (size_t)n * 40,
                                   cudaMemcpyHostToDevice, m->copy_stream));
                CK(cudaEventRecord(m->ev_ring_up[r], m->copy_stream));
                CK(cudaStreamWaitEvent(ds, m->ev_ring_up[r], 0));
                srcp[b] = m->d_ring[r];
            }
            const SrcOHMB1 src{srcp[b]};
            const long long l0 = m->launches;
            // discover stream (after the previous batch's resolve + buckets, queued
            // below): the batch's preprocessing, next to the previous fold
            k_batch_init<<<1, 32, 0, ds>>>(dm, (b == b0 && keep_claims) ? 0 : 1);
            CK(cudaEventRecord(ev[0], ds));
            if ((rc = launch_discover(m, dm, src, n, mode, 1, dm.ndt_segs, 1, ds))) return rc;
            k_guard<<<1, 1, 0, ds>>>(dm, margin);
            m->launches += 2;
            if (dm.ndt_segs) {
                k_rgrid<<<16, BLOCK, 0, ds>>>(dm);
                k_seg_scan<<<1, SEG_BUCKETS, 0, ds>>>(dm);
                k_seg_scatter<<<(unsigned)((n * maxseg + BLOCK - 1) / BLOCK), BLOCK, 0, ds>>>(dm);
                m->launches += 3;
            } else if (ray_order) {
                k_seg_scan<<<1, SEG_BUCKETS, 0, ds>>>(dm);
                k_seg_scatter<<<(unsigned)((n + BLOCK - 1) / BLOCK), BLOCK, 0, ds>>>(dm, n);
                m->launches += 2;
            }
            if ((rc = check_launch("discover"))) return rc;
            CK(cudaEventRecord(ev[1], ds));
            // the map's stream: walk (after the previous fold), resolve, fold
            CK(cudaStreamWaitEvent(s, ev[1], 0));
            CK(cudaEventRecord(ev[6], s));
            if ((rc = launch_walk(m, dm, src, n, mode, true, false))) return rc;
            k_batch_regions<<<1, 1, 0, s>>>(dm);
            CK(cudaEventRecord(ev[2], s));
            m->launches += 1;
            if ((rc = launch_ndt_tail(m, dm, src, n, maxseg, tm, ev[2], ev[3], ev[4]))) return rc;
            // batch b+1's discover may start: b's k_resolve (ev[3]) and bucket
            // kernels (ev[4]) are done with the region box, grid, touched list
            // and record buffer
            CK(cudaStreamWaitEvent(ds, ev[3], 0));
            CK(cudaStreamWaitEvent(ds, ev[4], 0));
            k_batch_fin<<<1, 1, 0, s>>>(dm);
            m->launches += 1;
            CK(cudaEventRecord(ev[5], s));
            if (!rays[b].on_device) CK(cudaEventRecord(m->ev_ring[b % vm_map::RING], s));
            if ((rc = check_launch("batch"))) return rc;
            dms[b] = dm;
            launches[b] = m->launches - l0;
        }
        CK(cudaMemcpyAsync(m->h_mstats + (size_t)b0 * MSTRIDE, m->d_mstats + (size_t)b0 * MSTRIDE,
                           (size_t)(nb - b0) * MSTRIDE * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if ((rc = check_launch("sequence"))) return rc;
        keep_claims = false;
        int f = nb;
        long long regions = m->nreg;
        for (int b = b0; b < nb; ++b) {
            if (rays[b].count <= 0) {
                out[b].regions_total = regions;
                continue;
            }
            const unsigned long long *slot = m->h_mstats + (size_t)b * MSTRIDE;
            if (slot[NUM_STATS + 1] != 3ULL) {
                f = b;
                break;
            }
            before[b] = first_before[b] >= 0 ? first_before[b] : regions;
            regions = (long long)slot[NUM_STATS];
        }
        for (int b = b0; b < f; ++b) {
            if (rays[b].count <= 0) continue;
            fill_stats(m->h_mstats + (size_t)b * MSTRIDE, rays[b].count, before[b], out + b);
            m->max_growth = std::max<long long>(m->max_growth, out[b].new_regions);
        }
        m->nreg = regions;
        if (f == nb) break;
        // ---- recover batch f (integrate_impl's NDT branches) ----
        unsigned long long *slot = m->h_mstats + (size_t)f * MSTRIDE;
        const int cursor = (int)slot[NUM_STATS];
        DevMap dm = dms[f];
        const long long words = std::min<long long>(cursor, m->cap) * (long long)m->vpr;
        if (slot[S_RANGE_ERR]) {
            k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, s>>>(dm, words);
            CK(cudaStreamSynchronize(s));
            m->nreg = cursor;
            return fail(VM_ERR_RANGE, "ray coordinates outside the packable region range "
                                      "(|region| < 2**20, keys.py:76-86)");
        }
        if (!(slot[NUM_STATS + 1] & 1ULL)) {
            // refused: spilled regions reached (reload) or the pool is short
            // (grow); nothing was applied, the claims stay for the replay
            m->nreg = cursor;
            if (slot[S_SPILLED]) {
                if ((rc = reload_listed(m, slot[S_SPILLED]))) return rc;
            } else {
                m->max_growth = std::max<long long>(m->max_growth, cursor - regions);
                if ((rc = grow_pool(m, std::max<long long>(2 * m->cap,
                                                           cursor + 2 * margin + headroom))))
                    return rc;
                if (cursor + margin > m->cap)
                    return fail(VM_ERR_OOM, "region pool exhausted (max regions reached)");
            }
            if (first_before[f] < 0) first_before[f] = regions;
            reps[f] += 1;
            b0 = f;
            keep_claims = true;
            continue;
        }
        // records or voxel indices overflowed: walk + resolve were applied,
        // no bucket kernel ran.  Drop the claims, make room, re-emit the
        // records only and fold them.
        unsigned long long R = slot[S_RECORDS], M = 0;
        int cur = 0;
        CK(cudaMemcpyAsync(&M, dm.nmarked, sizeof(M), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&cur, m->d_cursor, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, s>>>(dm, words);
        {
            // batch f+1's discover may have run next to f's (aborted) fold:
            // drop its claims in the other index layer; f+1 restarts clean
            DevMap d2 = dm;
            d2.nidx = dm.nidx == L_NIDX ? L_NIDX2 : L_NIDX;
            const long long w2 = std::min<long long>(cur, m->cap) * (long long)m->vpr;
            k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, s>>>(d2, w2);
        }
        const size_t grow = std::max<size_t>(std::max<size_t>(R, M) + (std::max(R, M) >> 2), m->rec_cap);
        if ((rc = ensure_records(m, grow))) return rc;
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_smarked2, &m->smarked2_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_rec_t, &m->rec_t_cap, m->rec_cap))) return rc;
        dm.rec = m->d_rec;
        dm.recval = m->d_val;
        dm.rec_t = m->d_rec_t;
        dm.rec_cap = m->rec_cap;
        dm.marked = par[f] ? m->d_smarked2 : m->d_smarked;
        dm.marked_cap = par[f] ? m->smarked2_cap : m->smarked_cap;
        dm.ray_order = 0;
        static const int one = 1;
        CK(cudaMemsetAsync(m->d_chain, 0, sizeof(int), s));
        CK(cudaMemcpyAsync(dm.go, &one, sizeof(int), cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(dm.stats + S_RECORDS, 0, sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(dm.nmarked, 0, sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(dm.nlost, 0, sizeof(unsigned long long), s));
        if (!rays[f].on_device) {
            CK(cudaMemcpyAsync(m->d_ring[f % vm_map::RING], rays[f].records,
                               (size_t)rays[f].count * 40, cudaMemcpyHostToDevice, s));
            srcp[f] = m->d_ring[f % vm_map::RING];
        }
        const SrcOHMB1 src{srcp[f]};
        const long long n = rays[f].count;
        cudaEvent_t *ev = &m->mev[(size_t)8 * f];
        if ((rc = launch_discover(m, dm, src, n, mode, 1, 0, 0, s))) return rc;
        if ((rc = launch_walk(m, dm, src, n, mode, true, true))) return rc;
        CK(cudaEventRecord(ev[3], s));
        if ((rc = launch_ndt_fold(m, dm, src, n, maxseg, tm, ev[4]))) return rc;
        k_batch_fin<<<1, 1, 0, s>>>(dm);
        CK(cudaEventRecord(ev[5], s));
        CK(cudaMemcpyAsync(slot, dm.stats, MSTRIDE * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if ((rc = check_launch("record re-emit"))) return rc;
        if (slot[NUM_STATS + 1] != 3ULL) {
            m->nreg = cursor;
            return fail(VM_ERR_CUDA, "NDT record re-emission overflowed");
        }
        fill_stats(slot, n, first_before[f] >= 0 ? first_before[f] : m->nreg, out + f);
        m->max_growth = std::max<long long>(m->max_growth, out[f].new_regions);
        m->nreg = (long long)slot[NUM_STATS];
        b0 = f + 1;
    }
    return sequence_times(m, rays, nb, reps, launches, out);
}

int integrate_pipelined(vm_map *m, const vm_rays *rays, int nb, int mode, vm_stats *out) {
    cudaStream_t s = m->stream;
    const int maxseg = (int)std::ceil(m->cfg.max_ray_range / m->cfg.segment_length) + 1;
    long long nmax = 0;
    bool any_host = false;
    for (int b = 0; b < nb; ++b) {
        nmax = std::max<long long>(nmax, rays[b].count);
        if (rays[b].count > 0 && !rays[b].on_device) any_host = true;
    }
    for (int b = 0; b < nb; ++b) std::memset(out + b, 0, sizeof(vm_stats));
    if (nmax <= 0) {
        for (int b = 0; b < nb; ++b) out[b].regions_total = m->nreg;
        return VM_OK;
    }
    const unsigned long long span_max = ((unsigned long long)nmax * maxseg) << 1;
    if (span_max >= (1ULL << 32))
        return fail(VM_ERR_ARG, "batch too large for 32-bit ray order keys; split it");
    int rc;
    const bool ndt = mode == M_NDT_OM || mode == M_NDT_TM;
    const bool ray_order = ndt && m->ndt_generic && !m->no_ray_order;
    if (ndt) {
        // sized for the largest batch up front: nothing is reallocated while
        // the sequence is in flight (integrate_impl's NDT bounds)
        const size_t need = m->ndt_rec_override > 0 ? (size_t)m->ndt_rec_override
                                                     : (size_t)nmax * 8 + 1;
        const size_t nwork = m->ndt_generic ? (size_t)nmax + 1 : (size_t)nmax * maxseg + 1;
        if (!m->ndt_generic && (rc = ensure_buf(&m->d_segs, &m->seg_cap, nwork))) return rc;
        if ((rc = ensure_buf(&m->d_perm, &m->perm_cap, nwork))) return rc;
        if ((rc = ensure_buf(&m->d_seg_bk, &m->seg_bk_cap, nwork))) return rc;
        if ((rc = ensure_records(m, std::max<size_t>(m->rec_cap, need)))) return rc;
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_rec_t, &m->rec_t_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_nbk_pos, &m->nbk_pos_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buckets(m, m->smarked_cap,
                                 (2 * (unsigned long long)nmax * maxseg + 31) / 32 + 1)))
            return rc;
        if (!m->d_chain && (rc = dev_alloc(&m->d_chain, 1))) return rc;
        return integrate_pipelined_ndt(m, rays, nb, mode, out, maxseg, nmax, any_host, ray_order);
    }
    if ((rc = ensure_buf(&m->d_segs, &m->seg_cap, (size_t)nmax * maxseg + 1))) return rc;
    if ((rc = ensure_buf(&m->d_perm, &m->perm_cap, m->seg_cap))) return rc;
    if ((rc = ensure_buf(&m->d_seg_bk, &m->seg_bk_cap, m->seg_cap))) return rc;
    if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, (size_t)nmax + 1))) return rc;
    if ((rc = ensure_records(m, std::max<size_t>(m->rec_cap, rec_floor(m, nmax)))))
        return rc;
    if ((rc = ensure_buckets(m, m->smarked_cap, ((unsigned long long)nmax * maxseg + 31) / 32 + 1)))
        return rc;
    if (!m->d_chain && (rc = dev_alloc(&m->d_chain, 1))) return rc;
    if ((rc = ensure_disc_stream(m))) return rc;
    if ((rc = ensure_buf(&m->d_smarked2, &m->smarked2_cap, m->smarked_cap))) return rc;
    if ((rc = ensure_buf(&m->d_segs2, &m->segs2_cap, m->seg_cap))) return rc;
    if ((rc = ensure_buf(&m->d_perm2, &m->perm2_cap, m->seg_cap))) return rc;
    if ((rc = ensure_buf(&m->d_seg_bk2, &m->seg_bk2_cap, m->seg_cap))) return rc;
    cudaStream_t ds = m->disc_stream;
    if ((rc = sequence_buffers(m, nb, nmax, any_host))) return rc;
    std::vector<DevMap> dms(nb);
    std::vector<const unsigned char *> srcp(nb, nullptr);
    std::vector<long long> reps(nb, 0), launches(nb, 0), before(nb, 0), first_before(nb, -1);
    bool keep_marks = false;  // a replayed batch keeps its sample-voxel stamps
    int b0 = 0;
    auto upload = [&](int b, cudaStream_t st) -> int {
        const int r = b % vm_map::RING;
        CK(cudaStreamWaitEvent(st, m->ev_ring[r], 0));  // the slot's previous batch is done
        CK(cudaMemcpyAsync(m->d_ring[r], rays[b].records, (size_t)rays[b].count * 40,
                           cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(m->ev_ring_up[r], st));
        CK(cudaStreamWaitEvent(ds, m->ev_ring_up[r], 0));  // the batch's discover reads it
        srcp[b] = m->d_ring[r];
        return VM_OK;
    };
    // batch-scoped buffers of parity 1 (parity 0 uses the map's own); parity =
    // position among the non-empty batches, so consecutive batches of the
    // pipeline alternate with an empty batch in between too
    std::vector<int> par(nb, 0);
    for (int b = 0, k = 0; b < nb; ++b)
        if (rays[b].count > 0) par[b] = (k++) & 1;
    auto parity = [&](DevMap &dm, int b) {
        if (!par[b]) return;
        dm.touched = m->d_touched2;
        dm.rgrid = m->d_rgrid2;
        dm.rbox = m->d_rbox2;
        dm.go = m->d_go2;
        dm.marked = m->d_smarked2;
        dm.nmarked = m->d_mk2;
        dm.segs = m->d_segs2;
        dm.perm = m->d_perm2;
        dm.seg_bk = m->d_seg_bk2;
        dm.seg_cap = std::min(m->segs2_cap, std::min(m->perm2_cap, m->seg_bk2_cap));
    };
    while (b0 < nb) {
        const long long headroom = std::max<long long>(512, 2 * m->max_growth);
        if (m->nreg + headroom > m->cap &&
            (rc = grow_pool(m, std::max(2 * m->cap, m->nreg + headroom))))
            return rc;
        const int margin = 64 + (int)std::min<long long>(1 << 20, headroom / 4);
        CK(cudaMemsetAsync(m->d_chain, 0, sizeof(int), s));
        CK(cudaEventRecord(m->ev_seq0, s));  // the discover stream starts after the map's prior work
        CK(cudaStreamWaitEvent(ds, m->ev_seq0, 0));
        for (int b = b0; b < nb; ++b) {
            const long long n = rays[b].count;
            cudaEvent_t *ev = &m->mev[(size_t)8 * b];
            if (n <= 0) continue;
            m->epoch += 1;
            DevMap dm = make_dm(m);
            dm.batch_no = m->batch_no + (unsigned)b;  // the sequence's batches count on
            dm.order_bits = std::max(1, bitlen(((unsigned long long)n * maxseg) << 1));
            dm.key_mi = 1;
            dm.marked = m->d_smarked;
            dm.nmarked = m->d_shard_cnt;
            dm.marked_cap = m->smarked_cap;
            dm.stats = m->d_mstats + (size_t)b * MSTRIDE;
            dm.chain = m->d_chain;
            dm.batch_idx = b;
            parity(dm, b);
            if (rays[b].on_device) srcp[b] = (const unsigned char *)rays[b].records;
            else if ((rc = upload(b, m->copy_stream))) return rc;
            const SrcOHMB1 src{srcp[b]};
            const long long l0 = m->launches;
            // discover stream: batch b's preprocessing, concurrent with batch
            // b-1's resolve and fold (it waited for b-1's walk)
            k_batch_init<<<1, 32, 0, ds>>>(dm, (b == b0 && keep_marks) ? 0 : 1);
            CK(cudaEventRecord(ev[0], ds));
            if ((rc = launch_discover(m, dm, src, n, mode, 1, 1, 1, ds))) return rc;
            k_guard<<<1, 1, 0, ds>>>(dm, margin);
            k_rgrid<<<16, BLOCK, 0, ds>>>(dm);
            k_seg_scan<<<1, SEG_BUCKETS, 0, ds>>>(dm);
            k_seg_scatter<<<(unsigned)((n * maxseg + BLOCK - 1) / BLOCK), BLOCK, 0, ds>>>(dm);
            m->launches += 5;
            if ((rc = check_launch("discover"))) return rc;
            CK(cudaEventRecord(ev[1], ds));
            // the map's stream: stamps (after b-1's fold), walk, resolve, fold
            CK(cudaStreamWaitEvent(s, ev[1], 0));
            k_stamp<<<m->num_sms * 8, BLOCK, 0, s>>>(dm);
            CK(cudaEventRecord(ev[6], s));
            if ((rc = launch_walk(m, dm, src, n, mode, true, false))) return rc;
            k_batch_regions<<<1, 1, 0, s>>>(dm);
            CK(cudaEventRecord(ev[2], s));
            CK(cudaStreamWaitEvent(ds, ev[2], 0));  // batch b+1's discover may start
            k_resolve<false, false><<<m->num_sms * 8, BLOCK, 0, s>>>(dm);
            m->launches += 3;
            CK(cudaEventRecord(ev[3], s));
            if ((rc = launch_bucket_fold(m, dm, src, n, maxseg, ev[4]))) return rc;
            k_batch_fin<<<1, 1, 0, s>>>(dm);
            m->launches += 1;
            CK(cudaEventRecord(ev[5], s));
            if (!rays[b].on_device) CK(cudaEventRecord(m->ev_ring[b % vm_map::RING], s));
            if ((rc = check_launch("batch"))) return rc;
            dms[b] = dm;
            launches[b] = m->launches - l0;
        }
        CK(cudaMemcpyAsync(m->h_mstats + (size_t)b0 * MSTRIDE, m->d_mstats + (size_t)b0 * MSTRIDE,
                           (size_t)(nb - b0) * MSTRIDE * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if ((rc = check_launch("sequence"))) return rc;
        keep_marks = false;
        int f = nb;
        long long regions = m->nreg;
        for (int b = b0; b < nb; ++b) {
            if (rays[b].count <= 0) {
                out[b].regions_total = regions;
                continue;
            }
            const unsigned long long *slot = m->h_mstats + (size_t)b * MSTRIDE;
            if (slot[NUM_STATS + 1] != 3ULL) {
                f = b;
                break;
            }
            before[b] = first_before[b] >= 0 ? first_before[b] : regions;
            regions = (long long)slot[NUM_STATS];
        }
        for (int b = b0; b < f; ++b) {
            if (rays[b].count <= 0) continue;
            const unsigned long long *slot = m->h_mstats + (size_t)b * MSTRIDE;
            fill_stats(slot, rays[b].count, before[b], out + b);
            m->max_growth = std::max<long long>(m->max_growth, out[b].new_regions);
        }
        m->nreg = regions;
        if (f == nb) break;
        // ---- recover batch f ----
        const unsigned long long *slot = m->h_mstats + (size_t)f * MSTRIDE;
        const int cursor = (int)slot[NUM_STATS];
        DevMap dm = dms[f];
        if (slot[S_RANGE_ERR]) {
            const long long words = std::min<long long>(cursor, m->cap) * (long long)m->vpr;
            k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, s>>>(dm, words);  // the claims (never stamped)
            CK(cudaStreamSynchronize(s));
            m->nreg = cursor;
            return fail(VM_ERR_RANGE, "ray coordinates outside the packable region range "
                                      "(|region| < 2**20, keys.py:76-86)");
        }
        if (!(slot[NUM_STATS + 1] & 1ULL) && slot[S_SPILLED]) {
            // spilled regions reached: reload them and replay from f
            m->nreg = cursor;
            if ((rc = reload_listed(m, slot[S_SPILLED]))) return rc;
            if (first_before[f] < 0) first_before[f] = regions;
            reps[f] += 1;
            b0 = f;
            keep_marks = true;
            continue;
        }
        if (!(slot[NUM_STATS + 1] & 1ULL)) {
            // region pool: grow and replay from f (its stamps stay valid)
            m->max_growth = std::max<long long>(m->max_growth, cursor - m->nreg);
            if ((rc = grow_pool(m, std::max<long long>(2 * m->cap, cursor + 2 * margin + headroom))))
                return rc;
            if (cursor + margin > m->cap)
                return fail(VM_ERR_OOM, "region pool exhausted (max regions reached)");
            if (first_before[f] < 0) first_before[f] = regions;  // new_regions spans the replays
            m->nreg = cursor;
            reps[f] += 1;
            b0 = f;
            keep_marks = true;
            continue;
        }
        // records overflowed: walk + resolve were applied, the fold was not;
        // re-emit the records (nothing re-applied) and fold them
        const unsigned long long R = slot[S_RECORDS];
        if ((rc = ensure_records(m, (size_t)R + (R >> 2)))) return rc;
        dm.rec = m->d_rec;
        dm.recval = m->d_val;
        dm.rec_cap = m->rec_cap;
        static const int one = 1;
        CK(cudaMemsetAsync(m->d_chain, 0, sizeof(int), s));
        CK(cudaMemcpyAsync(dm.go, &one, sizeof(int), cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(dm.stats + S_RECORDS, 0, sizeof(unsigned long long), s));
        if (!rays[f].on_device) {
            CK(cudaMemcpyAsync(m->d_ring[f % vm_map::RING], rays[f].records,
                               (size_t)rays[f].count * 40, cudaMemcpyHostToDevice, s));
            srcp[f] = m->d_ring[f % vm_map::RING];
        }
        const SrcOHMB1 src{srcp[f]};
        const long long n = rays[f].count;
        if ((rc = launch_walk(m, dm, src, n, mode, true, true))) return rc;
        cudaEvent_t *ev = &m->mev[(size_t)8 * f];
        CK(cudaEventRecord(ev[3], s));
        if ((rc = launch_bucket_fold(m, dm, src, n, maxseg, ev[4]))) return rc;
        k_batch_fin<<<1, 1, 0, s>>>(dm);
        CK(cudaEventRecord(ev[5], s));
        // batch f+1's discover may have run concurrently with f's (aborted)
        // fold: drop its index claims; f+1 restarts from a clean list
        {
            int cur = 0;
            CK(cudaMemcpyAsync(&cur, m->d_cursor, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const long long words = std::min<long long>(cur, m->cap) * (long long)m->vpr;
            k_nbk_clear<<<m->num_sms * 4, BLOCK, 0, s>>>(dm, words);
            CK(cudaMemsetAsync(m->d_shard_cnt, 0, 2 * sizeof(unsigned long long), s));
            CK(cudaMemsetAsync(m->d_mk2, 0, 2 * sizeof(unsigned long long), s));
        }
        CK(cudaMemcpyAsync(m->h_mstats + (size_t)f * MSTRIDE, dm.stats,
                           MSTRIDE * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if ((rc = check_launch("record re-emit"))) return rc;
        if (slot[NUM_STATS + 1] != 3ULL) return fail(VM_ERR_CUDA, "record re-emit failed");
        fill_stats(slot, n, first_before[f] >= 0 ? first_before[f] : m->nreg, out + f);
        m->nreg = (long long)slot[NUM_STATS];
        b0 = f + 1;
    }
    return sequence_times(m, rays, nb, reps, launches, out);
}

std::mutex g_walk_mu;

}  // namespace

// =================================================================== C ABI

extern "C" {

const char *vm_last_error(void) { return g_err.c_str(); }

const char *vm_build_info(void) {
    return "voxmap_b200: sm_100a, -fmad=false, fp64 DDA, CUB radix sort";
}

int vm_device_count(int32_t *out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *out = n;
    return VM_OK;
}

uint64_t vm_hash_mix(int64_t key) { return mix_key(key); }

int vm_map_create(const vm_config *cfg, uint32_t layer_mask, int32_t device,
                  int64_t initial_regions, vm_map **out) {
    if (!cfg || !out) return fail(VM_ERR_ARG, "null argument");
    *out = nullptr;
    if (!(cfg->voxel_size > 0) || !std::isfinite(cfg->voxel_size))
        return fail(VM_ERR_ARG, "voxel_size must be positive");
    if (cfg->region_dim < 1 || cfg->region_dim > 1024)
        return fail(VM_ERR_ARG, "region_dim must be in [1, 1024]");
    if (!(cfg->segment_length > 0) || !(cfg->max_ray_range > 0))
        return fail(VM_ERR_ARG, "segment_length and max_ray_range must be positive");
    if ((layer_mask & ~0x7FEu) != 0) return fail(VM_ERR_ARG, "unknown layer id in mask");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(VM_ERR_NODEV, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(VM_ERR_ARG, "bad device index");
    CK(cudaSetDevice(device));
    vm_map *m = new vm_map();
    m->cfg = *cfg;
    m->mask = layer_mask;
    m->device = device;
    m->dim = cfg->region_dim;
    m->vpr = cfg->region_dim * cfg->region_dim * cfg->region_dim;
    m->max_slots = std::min<long long>(1LL << 20, (long long)(0xFFFFFFFFull / (unsigned long long)m->vpr));
    unsigned long long ts = 1;
    while (ts < 2ULL * (unsigned long long)m->max_slots) ts <<= 1;
    m->tsize = ts;
    for (int l = 0; l < NUM_LAYERS; ++l) {
        bool on = l == L_SCRATCH ? true
                  : l == L_NIDX  ? true  // voxel index claims (every deterministic path)
                  : l == L_NIDX2 ? ((layer_mask >> L_COV) & 1u) != 0  // NDT: odd batches' claims
                                 : ((layer_mask >> l) & 1u) != 0;
        m->bpr[l] = on ? (size_t)m->vpr * LAYER_COMP[l] * LAYER_ELEM[l] : 0;
    }
    int rc;
    auto cleanup = [&](int code) {
        vm_map_destroy(m);
        return code;
    };
    if (cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(fail(VM_ERR_CUDA, "stream create failed"));
    for (auto &e : m->ev_up)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
            return cleanup(fail(VM_ERR_CUDA, "event create"));
    m->own_stream = true;
    if ((rc = dev_alloc(&m->d_tkeys, ts, 0xFF)) || (rc = dev_alloc(&m->d_tvals, ts, 0xFF)) ||
        (rc = dev_alloc(&m->d_cursor, 1)) || (rc = dev_alloc(&m->d_slot_keys, m->max_slots)) ||
        (rc = dev_alloc(&m->d_slot_touch, m->max_slots)) ||
        (rc = dev_alloc(&m->d_slot_pref, m->max_slots)) || (rc = dev_alloc(&m->d_stats, NUM_STATS)) ||
        (rc = dev_alloc(&m->d_go, 1)) || (rc = dev_alloc(&m->d_touched, m->max_slots)) ||
        (rc = dev_alloc(&m->d_work, 1)) ||
        (rc = dev_alloc(&m->d_rgrid, RG_MAX)) || (rc = dev_alloc(&m->d_rbox, 6)) ||
        (rc = dev_alloc(&m->d_bmask, m->max_slots)) || (rc = dev_alloc(&m->d_gmask, m->max_slots)) ||
        (rc = dev_alloc(&m->d_seg_hist, SEG_BUCKETS)) ||
        (rc = dev_alloc(&m->d_shard_cnt, 3)) || (rc = dev_alloc(&m->d_nlost, 1)) ||
        (rc = dev_alloc(&m->d_seg_cursor, SEG_BUCKETS)) ||
        (rc = dev_alloc(&m->d_nbig, 1)) || (rc = dev_alloc(&m->d_reload, RELOAD_CAP)) ||
        (rc = dev_alloc(&m->d_slot_last, m->max_slots)))
        return cleanup(rc);
    for (int l = 0; l < NUM_LAYERS; ++l)
        if (m->bpr[l] && (rc = dev_alloc(&m->d_lptr[l], m->max_slots))) return cleanup(rc);
    if (cudaMallocHost((void **)&m->h_stats, (NUM_STATS + 4) * sizeof(unsigned long long)) !=
        cudaSuccess)
        return cleanup(fail(VM_ERR_OOM, "pinned alloc failed"));
    cudaEvent_t *evs[] = {&m->ev_start, &m->ev_end, &m->ev_w0, &m->ev_w1,
                          &m->ev_k1,    &m->ev_k2,  &m->ev_res, &m->ev_sort};
    for (auto *e : evs)
        if (cudaEventCreate(e) != cudaSuccess) return cleanup(fail(VM_ERR_CUDA, "event create"));
    {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) m->num_sms = prop.multiProcessorCount;
    }
    if (const char *rc_env = std::getenv("VOXMAP_B200_TEST_REC_CAP")) m->rec_floor_override = std::atoll(rc_env);
    if (const char *rc_env = std::getenv("VOXMAP_B200_TEST_NDT_REC_CAP"))
        m->ndt_rec_override = std::atoll(rc_env);
    if (std::getenv("VOXMAP_B200_NO_RAY_ORDER")) m->no_ray_order = 1;
    if (std::getenv("VOXMAP_B200_NO_PIPELINE")) m->no_pipeline = 1;
    if (std::getenv("VOXMAP_B200_NDT_GENERIC")) m->ndt_generic = 1;
    if ((rc = grow_pool(m, std::max<long long>(64, initial_regions)))) return cleanup(rc);
    *out = m;
    return VM_OK;
}

int vm_map_destroy(vm_map *m) {
    if (!m) return VM_OK;
    cudaSetDevice(m->device);
    if (m->stream) cudaStreamSynchronize(m->stream);
    for (int l = 0; l < NUM_LAYERS; ++l) {
        cudaFree(m->slab[l]);
        cudaFree(m->d_lptr[l]);
    }
    cudaFree(m->d_tkeys);
    cudaFree(m->d_tvals);
    cudaFree(m->d_cursor);
    cudaFree(m->d_slot_keys);
    cudaFree(m->d_slot_touch);
    cudaFree(m->d_slot_pref);
    cudaFree(m->d_segs);
    cudaFree(m->d_perm);
    cudaFree(m->d_seg_bk);
    cudaFree(m->d_seg_hist);
    cudaFree(m->d_seg_cursor);
    cudaFree(m->d_work);
    cudaFree(m->d_rgrid);
    cudaFree(m->d_smarked);
    cudaFree(m->d_shard_cnt);
    cudaFree(m->d_nlost);
    cudaFree(m->d_nlost2);
    cudaFree(m->d_gx);
    cudaFree(m->d_ngx);
    cudaFree(m->d_touched2);
    cudaFree(m->d_rgrid2);
    cudaFree(m->d_rbox2);
    cudaFree(m->d_go2);
    cudaFree(m->d_smarked2);
    cudaFree(m->d_mk2);
    cudaFree(m->d_segs2);
    cudaFree(m->d_perm2);
    cudaFree(m->d_seg_bk2);
    if (m->disc_stream) cudaStreamDestroy(m->disc_stream);
    if (m->aux_stream) cudaStreamDestroy(m->aux_stream);
    if (m->ev_seq0) cudaEventDestroy(m->ev_seq0);
    cudaFree(m->d_reload);
    cudaFree(m->d_slot_last);
    cudaFree(m->d_bmask);
    cudaFree(m->d_gmask);
    cudaFree(m->d_big);
    cudaFree(m->d_nbig);
    cudaFree(m->d_nmid);
    cudaFree(m->d_bk_cnt);
    cudaFree(m->d_bk_off);
    cudaFree(m->d_bk_big);
    cudaFree(m->d_bk_perm);
    cudaFree(m->d_bk_cnt2);
    cudaFree(m->d_bk_big2);
    cudaFree(m->d_nbk_ctr);
    cudaFree(m->d_nbk_pos);
    cudaFree(m->d_rec_t);
    cudaFree(m->d_nbk_small);
    cudaFree(m->d_ndt_roots);
    cudaFree(m->d_bk_bits);
    cudaFree(m->d_chain);
    cudaFree(m->d_mstats);
    if (m->h_mstats) cudaFreeHost(m->h_mstats);
    for (cudaEvent_t e : m->mev) cudaEventDestroy(e);
    for (int r = 0; r < vm_map::RING; ++r) {
        cudaFree(m->d_ring[r]);
        if (m->ev_ring[r]) cudaEventDestroy(m->ev_ring[r]);
        if (m->ev_ring_up[r]) cudaEventDestroy(m->ev_ring_up[r]);
    }
    cudaFree(m->d_rbox);
    cudaFree(m->d_stats);
    cudaFree(m->d_go);
    cudaFree(m->d_rec);
    cudaFree(m->d_rec2);
    cudaFree(m->d_val);
    cudaFree(m->d_val2);
    cudaFree(m->d_touched);
    cudaFree(m->d_sort_tmp);
    cudaFree(m->d_rays);
    if (m->h_stats) cudaFreeHost(m->h_stats);
    cudaEvent_t evs[] = {m->ev_start, m->ev_end, m->ev_w0,  m->ev_w1,
                         m->ev_k1,    m->ev_k2,  m->ev_res, m->ev_sort};
    for (auto e : evs)
        if (e) cudaEventDestroy(e);
    if (m->own_stream && m->stream) cudaStreamDestroy(m->stream);
    for (auto e : m->ev_up)
        if (e) cudaEventDestroy(e);
    if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
    delete m;
    (void)cudaGetLastError();  // nothing of this map may leak into later calls
    return VM_OK;
}

int vm_map_reset(vm_map *m) {
    if (!m) return fail(VM_ERR_ARG, "null map");
    CK(cudaSetDevice(m->device));
    for (int l = 0; l < NUM_LAYERS; ++l)
        if (m->bpr[l] && m->nreg)
            CK(cudaMemsetAsync(m->slab[l], 0, (size_t)m->nreg * m->bpr[l], m->stream));
    CK(cudaMemsetAsync(m->d_tkeys, 0xFF, m->tsize * sizeof(long long), m->stream));
    CK(cudaMemsetAsync(m->d_tvals, 0xFF, m->tsize * sizeof(int), m->stream));
    CK(cudaMemsetAsync(m->d_cursor, 0, sizeof(int), m->stream));
    CK(cudaMemsetAsync(m->d_bmask, 0, m->max_slots * sizeof(unsigned), m->stream));
    CK(cudaMemsetAsync(m->d_gmask, 0, m->max_slots * sizeof(unsigned), m->stream));
    CK(cudaMemsetAsync(m->d_slot_last, 0, m->max_slots * sizeof(unsigned), m->stream));
    CK(cudaStreamSynchronize(m->stream));
    m->nreg = 0;
    m->spilled.clear();  // the files stay on disk
    return VM_OK;
}

int vm_map_set_batch_counter(vm_map *m, uint32_t counter) {
    if (!m) return fail(VM_ERR_ARG, "null map");
    m->batch_no = counter;
    return VM_OK;
}

int vm_map_region_last_access(vm_map *m, int64_t first, int64_t count, uint32_t *out) {
    if (!m || !out || first < 0 || count < 0 || first + count > m->nreg)
        return fail(VM_ERR_ARG, "bad region range");
    if (!count) return VM_OK;
    CK(cudaSetDevice(m->device));
    CK(cudaMemcpyAsync(out, m->d_slot_last + first, count * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                       m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return VM_OK;
}

int vm_map_set_spill(vm_map *m, const char *dir, const int32_t *layer_ids, int32_t n) {
    if (!m || !dir || (n && !layer_ids)) return fail(VM_ERR_ARG, "null argument");
    std::vector<int> ids(layer_ids, layer_ids + n);
    for (int id : ids)
        if (id < 1 || id > L_TSDF || !m->bpr[id]) return fail(VM_ERR_ARG, "spill layer not in map");
    m->spill_dir = dir;
    m->spill_ids = ids;
    return VM_OK;
}

int vm_map_evict_regions(vm_map *m, const int64_t *keys, int64_t n, int64_t *evicted_out) {
    if (!m || !evicted_out || (n && !keys)) return fail(VM_ERR_ARG, "null argument");
    *evicted_out = 0;
    if (m->spill_dir.empty()) return fail(VM_ERR_ARG, "map was created without a spill directory");
    if (!n) return VM_OK;
    CK(cudaSetDevice(m->device));
    CK(cudaStreamSynchronize(m->stream));
    const long long nreg = m->nreg;
    std::vector<long long> skeys((size_t)nreg);
    std::vector<unsigned> last((size_t)nreg);
    if (nreg) {
        CK(cudaMemcpy(skeys.data(), m->d_slot_keys, nreg * sizeof(long long), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(last.data(), m->d_slot_last, nreg * sizeof(unsigned), cudaMemcpyDeviceToHost));
    }
    std::set<long long> want(keys, keys + n);
    std::vector<char> gone((size_t)nreg, 0);
    size_t total = 0;
    for (int id : m->spill_ids) total += m->bpr[id];
    std::vector<unsigned char> payload(total);
    std::vector<unsigned char> blob(compressBound((uLong)total));
    long long evicted = 0;
    for (long long s = 0; s < nreg; ++s) {
        if (!want.count(skeys[s])) continue;
        size_t pos = 0;
        for (int id : m->spill_ids) {
            CK(cudaMemcpy(payload.data() + pos, (char *)m->slab[id] + (size_t)s * m->bpr[id], m->bpr[id],
                          cudaMemcpyDeviceToHost));
            pos += m->bpr[id];
        }
        uLongf bl = (uLongf)blob.size();
        if (compress2(blob.data(), &bl, payload.data(), (uLong)total, 6) != Z_OK)
            return fail(VM_ERR_OOM, "zlib compression failed");
        int r[3];
        unpack_region(skeys[s], r);
        const long long k3[3] = {r[0], r[1], r[2]};
        const uint32_t nl = (uint32_t)m->spill_ids.size();
        const std::string path = spill_path(m, skeys[s]);
        FILE *f = std::fopen(path.c_str(), "wb");
        bool ok = f != nullptr;
        if (ok) {
            ok = std::fwrite("OHMS1", 1, 5, f) == 5 && std::fwrite(k3, 8, 3, f) == 3 &&
                 std::fwrite(&nl, 4, 1, f) == 1;
            for (int id : m->spill_ids) {
                const uint32_t u = (uint32_t)id;
                ok = ok && std::fwrite(&u, 4, 1, f) == 1;
            }
            ok = ok && std::fwrite(blob.data(), 1, bl, f) == bl;
            ok = (std::fclose(f) == 0) && ok;
        }
        if (!ok) {
            // store.py:127-131: a failed spill keeps the region in memory
            std::fprintf(stderr, "voxmap_b200: spill of region (%d, %d, %d) failed, keeping it\n",
                         r[0], r[1], r[2]);
            std::remove(path.c_str());
            continue;
        }
        gone[(size_t)s] = 1;
        m->spilled.insert(skeys[s]);
        ++evicted;
    }
    if (!evicted) return VM_OK;
    // compact the pool: survivors move down in slot (= creation) order
    std::vector<long long> keep;
    std::vector<unsigned> keep_last;
    for (long long s = 0; s < nreg; ++s) {
        if (gone[(size_t)s]) continue;
        const long long t = (long long)keep.size();
        if (t != s)
            for (int l = 0; l < NUM_LAYERS; ++l)
                if (m->bpr[l])
                    CK(cudaMemcpyAsync((char *)m->slab[l] + (size_t)t * m->bpr[l],
                                       (char *)m->slab[l] + (size_t)s * m->bpr[l], m->bpr[l],
                                       cudaMemcpyDeviceToDevice, m->stream));
        keep.push_back(skeys[(size_t)s]);
        keep_last.push_back(last[(size_t)s]);
    }
    const long long nk = (long long)keep.size();
    for (int l = 0; l < NUM_LAYERS; ++l)
        if (m->bpr[l] && nreg > nk)
            CK(cudaMemsetAsync((char *)m->slab[l] + (size_t)nk * m->bpr[l], 0,
                               (size_t)(nreg - nk) * m->bpr[l], m->stream));
    // the region table: survivors at their new slots, spilled keys marked
    std::vector<long long> tk(m->tsize, -1);
    std::vector<int> tv(m->tsize, -1);
    auto put = [&](long long key, int v) {
        unsigned long long h = mix_key(key) & (m->tsize - 1);
        while (tk[h] != -1) h = (h + 1) & (m->tsize - 1);
        tk[h] = key;
        tv[h] = v;
    };
    for (long long t = 0; t < nk; ++t) put(keep[(size_t)t], (int)t);
    for (long long k : m->spilled) put(k, SLOT_SPILLED);
    CK(cudaMemcpyAsync(m->d_tkeys, tk.data(), m->tsize * sizeof(long long), cudaMemcpyHostToDevice, m->stream));
    CK(cudaMemcpyAsync(m->d_tvals, tv.data(), m->tsize * sizeof(int), cudaMemcpyHostToDevice, m->stream));
    if (nk) {
        CK(cudaMemcpyAsync(m->d_slot_keys, keep.data(), nk * sizeof(long long), cudaMemcpyHostToDevice, m->stream));
        CK(cudaMemcpyAsync(m->d_slot_last, keep_last.data(), nk * sizeof(unsigned), cudaMemcpyHostToDevice,
                           m->stream));
    }
    const int cur = (int)nk;
    CK(cudaMemcpyAsync(m->d_cursor, &cur, sizeof(int), cudaMemcpyHostToDevice, m->stream));
    CK(cudaMemsetAsync(m->d_bmask, 0, (size_t)nreg * sizeof(unsigned), m->stream));
    CK(cudaMemsetAsync(m->d_gmask, 0xFF, (size_t)nreg * sizeof(unsigned), m->stream));  // conservative
    CK(cudaMemsetAsync(m->d_slot_touch, 0, (size_t)nreg * sizeof(unsigned), m->stream));
    CK(cudaMemsetAsync(m->d_slot_pref, 0, (size_t)nreg * sizeof(unsigned), m->stream));
    CK(cudaStreamSynchronize(m->stream));
    m->nreg = nk;
    *evicted_out = evicted;
    return VM_OK;
}

int vm_map_reload_region(vm_map *m, int64_t key, int32_t *slot_out) {
    if (!m || !slot_out) return fail(VM_ERR_ARG, "null argument");
    CK(cudaSetDevice(m->device));
    int slot = -1;
    const int rc = reload_region(m, key, &slot);
    *slot_out = slot;
    return rc;
}

int vm_map_spilled_keys(vm_map *m, int64_t *out, int64_t cap, int64_t *n_out) {
    if (!m || !n_out || (cap && !out)) return fail(VM_ERR_ARG, "null argument");
    int64_t i = 0;
    for (long long k : m->spilled) {
        if (i < cap) out[i] = k;
        ++i;
    }
    *n_out = i;
    return VM_OK;
}

int vm_map_set_stream(vm_map *m, void *stream) {
    if (!m) return fail(VM_ERR_ARG, "null map");
    CK(cudaSetDevice(m->device));
    CK(cudaStreamSynchronize(m->stream));
    if (m->own_stream) cudaStreamDestroy(m->stream);
    if (stream) {
        m->stream = (cudaStream_t)stream;
        m->own_stream = false;
    } else {
        CK(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
        m->own_stream = true;
    }
    return VM_OK;
}

int vm_map_region_count(const vm_map *m, int64_t *out) {
    if (!m || !out) return fail(VM_ERR_ARG, "null argument");
    *out = m->nreg;
    return VM_OK;
}

int vm_map_region_keys(const vm_map *m, int64_t first, int64_t count, int64_t *keys_out) {
    if (!m || !keys_out || first < 0 || count < 0 || first + count > m->nreg)
        return fail(VM_ERR_ARG, "bad region key range");
    if (!count) return VM_OK;
    CK(cudaSetDevice(m->device));
    CK(cudaMemcpyAsync(keys_out, m->d_slot_keys + first, count * sizeof(int64_t),
                       cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return VM_OK;
}

}  // extern "C"

namespace {
__global__ void k_ensure(const __grid_constant__ DevMap m, const long long *keys, long long n, int *slots, int insert) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    slots[i] = region_slot(m, keys[i]);
}

int ensure_or_find(vm_map *m, const int64_t *keys, int64_t n, int32_t *slots_out, int insert) {
    if (!m || (n && (!keys || !slots_out))) return fail(VM_ERR_ARG, "null argument");
    if (!n) return VM_OK;
    CK(cudaSetDevice(m->device));
    int rc;
    for (int64_t i = 0; i < n && !m->spilled.empty(); ++i) {  // spilled: reload transparently
        int slot;
        if ((rc = reload_region(m, keys[i], &slot))) return rc;
    }
    if (insert && m->nreg + n > m->cap) {
        if ((rc = grow_pool(m, std::max<long long>(2 * m->cap, m->nreg + n + 64)))) return rc;
    }
    long long *dk = nullptr;
    int *ds = nullptr;
    CK(cudaMalloc(&dk, n * sizeof(long long)));
    CK(cudaMalloc(&ds, n * sizeof(int)));
    CK(cudaMemcpyAsync(dk, keys, n * sizeof(long long), cudaMemcpyHostToDevice, m->stream));
    DevMap dm = make_dm(m);
    dm.insert = insert;
    k_ensure<<<(unsigned)((n + 255) / 256), 256, 0, m->stream>>>(dm, dk, n, ds, insert);
    CK(cudaMemcpyAsync(slots_out, ds, n * sizeof(int), cudaMemcpyDeviceToHost, m->stream));
    int cursor = 0;
    CK(cudaMemcpyAsync(&cursor, m->d_cursor, sizeof(int), cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    cudaFree(dk);
    cudaFree(ds);
    if ((rc = check_launch("ensure"))) return rc;
    m->nreg = cursor;
    for (int64_t i = 0; i < n; ++i)
        if (insert && (slots_out[i] < 0 || slots_out[i] >= m->cap))
            return fail(VM_ERR_OOM, "region pool exhausted");
    return VM_OK;
}
}  // namespace

extern "C" {

int vm_map_ensure_regions(vm_map *m, const int64_t *keys, int64_t n, int32_t *slots_out) {
    return ensure_or_find(m, keys, n, slots_out, 1);
}

int vm_map_find_region(vm_map *m, int64_t key, int32_t *slot_out) {
    return ensure_or_find(m, &key, 1, slot_out, 0);
}

static int layer_io(vm_map *m, int32_t slot, int32_t layer, int64_t bytes, size_t *off) {
    if (!m || layer < 1 || layer > 10 || !m->bpr[layer])
        return fail(VM_ERR_ARG, "layer not present in map");
    if (slot < 0 || slot >= m->nreg) return fail(VM_ERR_ARG, "bad region slot");
    if ((size_t)bytes != m->bpr[layer]) return fail(VM_ERR_ARG, "byte count mismatch");
    *off = (size_t)slot * m->bpr[layer];
    return VM_OK;
}

int vm_map_read_layer(vm_map *m, int32_t slot, int32_t layer, void *dst, int64_t bytes) {
    size_t off;
    int rc = layer_io(m, slot, layer, bytes, &off);
    if (rc) return rc;
    CK(cudaSetDevice(m->device));
    CK(cudaMemcpyAsync(dst, (char *)m->slab[layer] + off, bytes, cudaMemcpyDeviceToHost,
                       m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return VM_OK;
}

int vm_map_write_layer(vm_map *m, int32_t slot, int32_t layer, const void *src, int64_t bytes) {
    size_t off;
    int rc = layer_io(m, slot, layer, bytes, &off);
    if (rc) return rc;
    CK(cudaSetDevice(m->device));
    if (layer == L_COUNT)  // the host may have made Gaussians anywhere in the region
        CK(cudaMemsetAsync(m->d_gmask + slot, 0xFF, sizeof(unsigned), m->stream));
    CK(cudaMemcpyAsync((char *)m->slab[layer] + off, src, bytes, cudaMemcpyHostToDevice,
                       m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return VM_OK;
}

int vm_map_layer_ptr(vm_map *m, int32_t slot, int32_t layer, void **out) {
    size_t off;
    if (!m || !out) return fail(VM_ERR_ARG, "null argument");
    int rc = layer_io(m, slot, layer, (int64_t)(layer >= 1 && layer <= 10 ? m->bpr[layer] : 0), &off);
    if (rc) return rc;
    *out = (char *)m->slab[layer] + off;
    return VM_OK;
}

int vm_integrate(vm_map *m, const vm_rays *rays, int32_t mode, int32_t exec, vm_stats *out) {
    if (!m || !rays || !out) return fail(VM_ERR_ARG, "null argument");
    if (mode < 0 || mode > 4) return fail(VM_ERR_ARG, "unknown mode");
    if (exec != VM_EXEC_CAS && exec != VM_EXEC_DETERMINISTIC) return fail(VM_ERR_ARG, "bad exec");
    if ((m->mask & MODE_MASK[mode]) != MODE_MASK[mode])
        return fail(VM_ERR_ARG, "map lacks layers required by mode");
    CK(cudaSetDevice(m->device));
    (void)cudaGetLastError();  // a stale non-sticky error of an unrelated call
    long long n = rays->count;
    std::memset(out, 0, sizeof(*out));
    if (n <= 0) {
        out->regions_total = m->nreg;
        return VM_OK;
    }
    m->up = vm_map::Upload{};
    if (rays->format == VM_RAYS_OHMB1) {
        if (!rays->records) return fail(VM_ERR_ARG, "null records");
        const unsigned char *p = (const unsigned char *)rays->records;
        if (!rays->on_device) {
            int rc = ensure_buf(&m->d_rays, &m->rays_bytes, (size_t)n * 40);
            if (rc) return rc;
            m->up.pending = 1;
            m->up.format = VM_RAYS_OHMB1;
            m->up.rec = p;
            p = m->d_rays;
        }
        SrcOHMB1 src{p};
        const int rc = integrate_impl(m, src, n, mode, exec, out);
        m->up.pending = 0;
        return rc;
    }
    if (rays->format == VM_RAYS_F64) {
        if (!rays->origins || !rays->ends || !rays->has_sample)
            return fail(VM_ERR_ARG, "null ray arrays");
        SrcF64 src{rays->origins, rays->ends, rays->has_sample, rays->intensity};
        if (!rays->on_device) {
            size_t b_o = (size_t)n * 24, b_h = ((size_t)n + 7) & ~(size_t)7, b_i = (size_t)n * 4;
            size_t total = 2 * b_o + b_h + (rays->intensity ? b_i : 0);
            int rc = ensure_buf(&m->d_rays, &m->rays_bytes, total);
            if (rc) return rc;
            unsigned char *d = m->d_rays;
            m->up.pending = 1;
            m->up.format = VM_RAYS_F64;
            m->up.o = rays->origins;
            m->up.e = rays->ends;
            m->up.h = rays->has_sample;
            m->up.it = rays->intensity;
            m->up.b_o = b_o;
            m->up.b_h = b_h;
            src = SrcF64{(const double *)d, (const double *)(d + b_o), d + 2 * b_o,
                         rays->intensity ? (const float *)(d + 2 * b_o + b_h) : nullptr};
        }
        const int rc = integrate_impl(m, src, n, mode, exec, out);
        m->up.pending = 0;
        return rc;
    }
    return fail(VM_ERR_ARG, "unknown ray format");
}

int vm_integrate_many(vm_map *m, const vm_rays *rays, int32_t nbatches, int32_t mode, int32_t exec,
                      vm_stats *out) {
    if (!m || (!rays && nbatches > 0) || (!out && nbatches > 0)) return fail(VM_ERR_ARG, "null argument");
    if (nbatches < 0) return fail(VM_ERR_ARG, "negative batch count");
    if (mode < 0 || mode > 4) return fail(VM_ERR_ARG, "unknown mode");
    if (exec != VM_EXEC_CAS && exec != VM_EXEC_DETERMINISTIC) return fail(VM_ERR_ARG, "bad exec");
    if ((m->mask & MODE_MASK[mode]) != MODE_MASK[mode])
        return fail(VM_ERR_ARG, "map lacks layers required by mode");
    bool pipelined = (mode == M_OCC || mode == M_NDT_OM || mode == M_NDT_TM) &&
                     exec == VM_EXEC_DETERMINISTIC && m->shard_world == 1 && !m->sb.open &&
                     !m->no_pipeline;
    for (int b = 0; b < nbatches && pipelined; ++b) {
        if (rays[b].count > 0 && (rays[b].format != VM_RAYS_OHMB1 || !rays[b].records))
            pipelined = false;
    }
    if (!pipelined) {
        // one vm_integrate per batch; host OHMB1 batches are prefetched: batch
        // b+1 is copied on copy_stream into a ring buffer while batch b computes
        bool prefetch = nbatches > 1;
        long long nmax = 0;
        for (int b = 0; b < nbatches; ++b) {
            if (rays[b].count > 0 && (rays[b].format != VM_RAYS_OHMB1 || rays[b].on_device ||
                                      !rays[b].records))
                prefetch = false;
            nmax = std::max<long long>(nmax, rays[b].count);
        }
        const unsigned base = m->batch_no;  // each batch stamps its own counter
        if (!prefetch) {
            for (int b = 0; b < nbatches; ++b) {
                m->batch_no = base + (unsigned)b;
                const int rc = vm_integrate(m, rays + b, mode, exec, out + b);
                if (rc) return rc;
            }
            return VM_OK;
        }
        CK(cudaSetDevice(m->device));
        if ((size_t)nmax * 40 > m->ring_bytes) {
            for (int r = 0; r < vm_map::RING; ++r) {
                cudaFree(m->d_ring[r]);
                m->d_ring[r] = nullptr;
                CK(cudaMalloc((void **)&m->d_ring[r], (size_t)nmax * 40));
                if (!m->ev_ring[r]) CK(cudaEventCreateWithFlags(&m->ev_ring[r], cudaEventDisableTiming));
                if (!m->ev_ring_up[r])
                    CK(cudaEventCreateWithFlags(&m->ev_ring_up[r], cudaEventDisableTiming));
            }
            m->ring_bytes = (size_t)nmax * 40;
        }
        auto upload = [&](int b) -> int {
            const int r = b % vm_map::RING;
            if (rays[b].count > 0)
                CK(cudaMemcpyAsync(m->d_ring[r], rays[b].records, (size_t)rays[b].count * 40,
                                   cudaMemcpyHostToDevice, m->copy_stream));
            CK(cudaEventRecord(m->ev_ring_up[r], m->copy_stream));
            return VM_OK;
        };
        int rc = upload(0);
        if (rc) return rc;
        for (int b = 0; b < nbatches; ++b) {
            CK(cudaStreamWaitEvent(m->stream, m->ev_ring_up[b % vm_map::RING], 0));
            // the slot of batch b+1 was last used by batch b+1-RING, which is done
            if (b + 1 < nbatches && (rc = upload(b + 1))) return rc;
            vm_rays r = rays[b];
            r.records = m->d_ring[b % vm_map::RING];
            r.on_device = 1;
            m->batch_no = base + (unsigned)b;
            if ((rc = vm_integrate(m, &r, mode, exec, out + b))) return rc;
        }
        return VM_OK;
    }
    CK(cudaSetDevice(m->device));
    (void)cudaGetLastError();
    return integrate_pipelined(m, rays, nbatches, mode, out);
}

// ---------------------------------------------------------------- exporters

int vm_export_select(vm_map *m, const int32_t *slots, int64_t nslots, int32_t kind,
                     double threshold, int64_t *count_out, int32_t *ridx_out, int32_t *li_out,
                     int64_t cap) {
    if (!m || (!slots && nslots > 0) || !count_out) return fail(VM_ERR_ARG, "null argument");
    if (kind < EX_OCCUPIED || kind > EX_DECAY) return fail(VM_ERR_ARG, "unknown export kind");
    static const int need[4] = {L_OCC, L_COUNT, L_TSDF, L_DDIST};
    if (!m->slab[need[kind]] || (kind == EX_DECAY && !m->slab[L_DHITS]))
        return fail(VM_ERR_ARG, "map lacks the layers of this export");
    CK(cudaSetDevice(m->device));
    *count_out = 0;
    if (nslots <= 0) return VM_OK;
    for (int64_t i = 0; i < nslots; ++i)
        if (slots[i] < 0 || slots[i] >= m->nreg) return fail(VM_ERR_ARG, "slot out of range");
    cudaStream_t s = m->stream;
    int *d_slots = nullptr;
    unsigned long long *d_cnt = nullptr;
    CK(cudaMalloc((void **)&d_slots, nslots * sizeof(int)));
    CK(cudaMalloc((void **)&d_cnt, nslots * sizeof(unsigned long long)));
    std::vector<unsigned long long> cnt(nslots);
    int rc = VM_OK;
    DevMap dm = make_dm(m);
    do {
        if (cudaMemcpyAsync(d_slots, slots, nslots * sizeof(int), cudaMemcpyHostToDevice, s) ||
            cudaMemsetAsync(d_cnt, 0, nslots * sizeof(unsigned long long), s)) {
            rc = fail(VM_ERR_CUDA, "export copy");
            break;
        }
        k_export_count<<<(unsigned)nslots, EX_BLOCK, 0, s>>>(dm, d_slots, kind, threshold, d_cnt);
        if (cudaMemcpyAsync(cnt.data(), d_cnt, nslots * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s) ||
            cudaStreamSynchronize(s)) {
            rc = fail(VM_ERR_CUDA, std::string("export count: ") + cudaGetErrorString(cudaGetLastError()));
            break;
        }
        unsigned long long total = 0;
        for (int64_t i = 0; i < nslots; ++i) {
            const unsigned long long c = cnt[i];
            cnt[i] = total;
            total += c;
        }
        *count_out = (int64_t)total;
        if (!ridx_out || !li_out || (int64_t)total > cap || total == 0) break;
        int *d_ridx = nullptr, *d_li = nullptr;
        if (cudaMalloc((void **)&d_ridx, total * sizeof(int)) ||
            cudaMalloc((void **)&d_li, total * sizeof(int))) {
            cudaFree(d_ridx);
            rc = fail(VM_ERR_OOM, "export buffers");
            break;
        }
        cudaMemcpyAsync(d_cnt, cnt.data(), nslots * sizeof(unsigned long long), cudaMemcpyHostToDevice, s);
        k_export_write<<<(unsigned)nslots, EX_BLOCK, 0, s>>>(dm, d_slots, kind, threshold, d_cnt,
                                                             d_ridx, d_li);
        cudaMemcpyAsync(ridx_out, d_ridx, total * sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(li_out, d_li, total * sizeof(int), cudaMemcpyDeviceToHost, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        cudaFree(d_ridx);
        cudaFree(d_li);
        if (e != cudaSuccess) rc = fail(VM_ERR_CUDA, std::string("export write: ") + cudaGetErrorString(e));
    } while (0);
    cudaFree(d_slots);
    cudaFree(d_cnt);
    return rc;
}

int vm_export_gather(vm_map *m, int32_t layer, const int32_t *slots, int64_t nslots,
                     const int32_t *ridx, const int32_t *li, int64_t n, void *out) {
    if (!m || !slots || (n > 0 && (!ridx || !li || !out))) return fail(VM_ERR_ARG, "null argument");
    if (layer < 1 || layer > L_TSDF || !m->slab[layer]) return fail(VM_ERR_ARG, "layer not in map");
    CK(cudaSetDevice(m->device));
    if (n <= 0) return VM_OK;
    const int bytes = (int)(m->bpr[layer] / (size_t)m->vpr);
    cudaStream_t s = m->stream;
    int *d_slots = nullptr, *d_ridx = nullptr, *d_li = nullptr;
    unsigned char *d_out = nullptr;
    int rc = VM_OK;
    if (cudaMalloc((void **)&d_slots, nslots * sizeof(int)) ||
        cudaMalloc((void **)&d_ridx, n * sizeof(int)) || cudaMalloc((void **)&d_li, n * sizeof(int)) ||
        cudaMalloc((void **)&d_out, (size_t)n * bytes)) {
        rc = fail(VM_ERR_OOM, "export gather buffers");
    } else {
        cudaMemcpyAsync(d_slots, slots, nslots * sizeof(int), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_ridx, ridx, n * sizeof(int), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_li, li, n * sizeof(int), cudaMemcpyHostToDevice, s);
        DevMap dm = make_dm(m);
        const long long blocks = std::min<long long>((n * bytes + 255) / 256, (long long)m->num_sms * 16);
        k_export_gather<<<(unsigned)std::max<long long>(1, blocks), 256, 0, s>>>(
            dm, layer, bytes, d_slots, d_ridx, d_li, n, d_out);
        cudaMemcpyAsync(out, d_out, (size_t)n * bytes, cudaMemcpyDeviceToHost, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = fail(VM_ERR_CUDA, std::string("export gather: ") + cudaGetErrorString(e));
    }
    cudaFree(d_slots);
    cudaFree(d_ridx);
    cudaFree(d_li);
    cudaFree(d_out);
    return rc;
}

int vm_walk_voxels(double ox, double oy, double oz, double ex, double ey, double ez, double cell,
                   int64_t cap, int64_t *coords_out, double *t0_out, double *t1_out,
                   int64_t *n_out) {
    if (!(cell > 0) || cap < 0 || !n_out) return fail(VM_ERR_ARG, "bad walk arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(VM_ERR_NODEV, "no CUDA device available");
    std::lock_guard<std::mutex> lk(g_walk_mu);
    static long long *d_c = nullptr;
    static double *d_t0 = nullptr, *d_t1 = nullptr;
    static long long *d_n = nullptr;
    static long long d_cap = 0;
    if (cap > d_cap || !d_n) {
        cudaFree(d_c);
        cudaFree(d_t0);
        cudaFree(d_t1);
        long long c = std::max<long long>(cap, 4096);
        CK(cudaMalloc(&d_c, c * 3 * sizeof(long long)));
        CK(cudaMalloc(&d_t0, c * sizeof(double)));
        CK(cudaMalloc(&d_t1, c * sizeof(double)));
        if (!d_n) CK(cudaMalloc(&d_n, sizeof(long long)));
        d_cap = c;
    }
    k_walk_one<<<1, 1>>>(ox, oy, oz, ex, ey, ez, cell, d_c, d_t0, d_t1, cap, d_n);
    int rc = check_launch("walk_one");
    if (rc) return rc;
    long long n = 0;
    CK(cudaMemcpy(&n, d_n, sizeof(long long), cudaMemcpyDeviceToHost));
    *n_out = n;
    if (n > cap) return fail(VM_ERR_ARG, "walk overflow");
    if (n) {
        CK(cudaMemcpy(coords_out, d_c, n * 3 * sizeof(long long), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(t0_out, d_t0, n * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(t1_out, d_t1, n * sizeof(double), cudaMemcpyDeviceToHost));
    }
    return VM_OK;
}

int vm_ndt_hypot(const double *ab, int64_t n, double *out) {
    if (n < 0 || (n > 0 && (!ab || !out))) return fail(VM_ERR_ARG, "bad hypot arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(VM_ERR_NODEV, "no CUDA device available");
    if (n == 0) return VM_OK;
    double *d = nullptr;
    CK(cudaMalloc(&d, (size_t)n * 3 * sizeof(double)));
    cudaError_t e = cudaMemcpy(d, ab, (size_t)n * 2 * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        k_py_hypot<<<(unsigned)((n + BLOCK - 1) / BLOCK), BLOCK>>>(d, d + 2 * n, n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpy(out, d + 2 * n, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(VM_ERR_CUDA, cudaGetErrorString(e));
    return VM_OK;
}

int vm_kernels_integrate_occupancy(const double *origins, const double *ends,
                                   const uint8_t *has_sample, int64_t n, const int64_t *tkeys,
                                   const int32_t *tvals, int64_t tsize, void *const *occ_ptrs,
                                   void *const *mean_ptrs, void *const *count_ptrs,
                                   void *const *dhit_ptrs, void *const *ddist_ptrs,
                                   double voxel_size, int64_t region_dim, double hit_delta,
                                   double miss_delta, double clamp_min, double clamp_max,
                                   int32_t retry_limit, int32_t walk_cap, int64_t *stats_out,
                                   void *stream) {
    (void)retry_limit;  // no mutex fallback on the GPU: retries are only counted
    if (!stats_out) return fail(VM_ERR_ARG, "null stats_out");
    std::memset(stats_out, 0, 4 * sizeof(int64_t));
    if (n < 0 || tsize <= 0 || (tsize & (tsize - 1)) != 0)
        return fail(VM_ERR_ARG, "n must be >= 0 and tsize a power of two");
    if (!(voxel_size > 0) || region_dim < 1 || region_dim > 1024)
        return fail(VM_ERR_ARG, "bad voxel_size / region_dim");
    if ((mean_ptrs == nullptr) != (count_ptrs == nullptr) ||
        (dhit_ptrs == nullptr) != (ddist_ptrs == nullptr))
        return fail(VM_ERR_ARG, "mean/count and decay pointer arrays come in pairs");
    if (n == 0) return VM_OK;
    if (!origins || !ends || !has_sample || !tkeys || !tvals || !occ_ptrs)
        return fail(VM_ERR_ARG, "null device array");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *d_st = nullptr;
    CK(cudaMallocAsync((void **)&d_st, 4 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(d_st, 0, 4 * sizeof(unsigned long long), s));
    CompatArgs a{};
    a.o = origins;
    a.e = ends;
    a.has = has_sample;
    a.n = n;
    a.tkeys = (const long long *)tkeys;
    a.tvals = tvals;
    a.tmask = (unsigned long long)tsize - 1;
    a.occ = occ_ptrs;
    a.mean = mean_ptrs;
    a.cnt = count_ptrs;
    a.dhit = dhit_ptrs;
    a.ddist = ddist_ptrs;
    a.vox = voxel_size;
    a.dim = (int)region_dim;
    a.hit = (float)hit_delta;
    a.miss = (float)miss_delta;
    a.cmin = (float)clamp_min;
    a.cmax = (float)clamp_max;
    a.walk_cap = walk_cap;
    a.stats = d_st;
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned grid = (unsigned)std::max<long long>(
        1, std::min<long long>((n + BLOCK - 1) / BLOCK, (long long)sms * 8));
    k_compat_occupancy<<<grid, BLOCK, 0, s>>>(a);
    int rc = check_launch("compat_occupancy");
    if (rc) return rc;
    unsigned long long h[4];
    CK(cudaMemcpyAsync(h, d_st, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d_st, s));
    CK(cudaStreamSynchronize(s));
    for (int i = 0; i < 4; ++i) stats_out[i] = (int64_t)h[i];
    return VM_OK;
}

}  // extern "C"

// =================================================================== sharding
// Region-sharded integration (vm_shard.cuh has the protocol).  Deterministic
// occupancy only; every rank passes the whole batch and walks its slice.

namespace {

template <class F>
int with_src(vm_map *m, F &&f) {
    if (m->sb.format == VM_RAYS_OHMB1) return f(SrcOHMB1{(const unsigned char *)m->sb.rays});
    return f(SrcF64{m->sb.o, m->sb.e, m->sb.h, m->sb.it});
}

int shard_headroom(vm_map *m, long long extra) {
    const long long need = m->nreg + extra + std::max<long long>(512, 2 * m->max_growth);
    if (need > m->cap) return grow_pool(m, std::max(2 * m->cap, need));
    return VM_OK;
}

int read_cursor(vm_map *m, int *cursor) {
    CK(cudaMemcpyAsync(m->h_stats + NUM_STATS, m->d_cursor, sizeof(int), cudaMemcpyDeviceToHost,
                       m->stream));
    CK(cudaStreamSynchronize(m->stream));
    *cursor = *(const int *)(m->h_stats + NUM_STATS);
    return VM_OK;
}

DevMap shard_dm(vm_map *m) {
    DevMap dm = make_dm(m);
    dm.order_bits = m->sb.order_bits;
    dm.ray_lo = m->sb.lo;
    dm.marked = m->d_smarked;
    dm.nmarked = m->d_shard_cnt;
    dm.marked_cap = m->smarked_cap;
    dm.walk_slot0 = m->sb.walk_slot0;
    dm.gx = m->d_gx;
    dm.ngx = m->d_ngx;
    dm.gx_cap = m->gx_cap;
    return dm;
}

}  // namespace

extern "C" {

int vm_shard_config(vm_map *m, int32_t rank, int32_t world) {
    if (!m || world < 1 || world > 4096 || rank < 0 || rank >= world)
        return fail(VM_ERR_ARG, "bad shard rank / world");
    if (m->sb.open) return fail(VM_ERR_ARG, "a sharded batch is in flight");
    CK(cudaSetDevice(m->device));
    cudaFree(m->d_shard_cnt);
    m->d_shard_cnt = nullptr;
    CK(cudaMalloc((void **)&m->d_shard_cnt, (2 + (size_t)world) * sizeof(unsigned long long)));
    m->shard_rank = rank;
    m->shard_world = world;
    return VM_OK;
}

int vm_shard_owner(int64_t packed_key, int32_t world) { return region_owner(packed_key, world); }

int vm_shard_begin(vm_map *m, const vm_rays *rays, int32_t mode, int32_t exec, int64_t *counts_out) {
    if (!m || !rays || !counts_out) return fail(VM_ERR_ARG, "null argument");
    if ((mode != VM_MODE_OCCUPANCY && mode != VM_MODE_NDT_OM) || exec != VM_EXEC_DETERMINISTIC)
        return fail(VM_ERR_ARG, "sharded maps integrate deterministic occupancy or NDT-OM");
    if ((m->mask & MODE_MASK[mode]) != MODE_MASK[mode]) return fail(VM_ERR_ARG, "map lacks layers");
    if (!m->d_shard_cnt) return fail(VM_ERR_ARG, "call vm_shard_config first");
    CK(cudaSetDevice(m->device));
    auto &sb = m->sb;
    sb = vm_map::ShardBatch{};
    const long long n_all = rays->count;
    if (n_all <= 0) return fail(VM_ERR_ARG, "empty batch");
    // the whole batch on the device (the fold reads any ray's end point)
    sb.format = rays->format;
    if (rays->format == VM_RAYS_OHMB1) {
        const unsigned char *p = (const unsigned char *)rays->records;
        if (!p) return fail(VM_ERR_ARG, "null records");
        if (!rays->on_device) {
            int rc = ensure_buf(&m->d_rays, &m->rays_bytes, (size_t)n_all * 40);
            if (rc) return rc;
            CK(cudaMemcpyAsync(m->d_rays, p, (size_t)n_all * 40, cudaMemcpyHostToDevice, m->stream));
            p = m->d_rays;
        }
        sb.rays = p;
    } else {
        if (!rays->on_device) return fail(VM_ERR_ARG, "sharded f64 rays must be device arrays");
        sb.o = rays->origins;
        sb.e = rays->ends;
        sb.h = rays->has_sample;
        sb.it = rays->intensity;
    }
    const int W = m->shard_world, rk = m->shard_rank;
    sb.n_all = n_all;
    sb.lo = n_all * rk / W;
    sb.n = n_all * (rk + 1) / W - sb.lo;
    sb.maxseg = (int)std::ceil(m->cfg.max_ray_range / m->cfg.segment_length) + 1;
    const unsigned long long order_span = ((unsigned long long)n_all * sb.maxseg) << 1;
    if (order_span >= (1ULL << 32)) return fail(VM_ERR_ARG, "batch too large for 32-bit ray order keys");
    sb.order_bits = std::max(1, bitlen(order_span));
    const long long n = std::max<long long>(sb.n, 1);
    sb.ndt = mode == VM_MODE_NDT_OM;
    int rc;
    if (sb.ndt) {
        // records: the slice's samples and walk records plus imported ones
        if ((rc = ensure_records(m, std::max<size_t>(m->rec_cap, (size_t)n_all * 8 + 1)))) return rc;
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_rec_t, &m->rec_t_cap, m->rec_cap))) return rc;
        if ((rc = ensure_buf(&m->d_gx, &m->gx_cap, (size_t)n * 16 + 1))) return rc;
        if (!m->d_ngx) CK(cudaMalloc((void **)&m->d_ngx, sizeof(unsigned long long)));
        CK(cudaMemsetAsync(m->d_ngx, 0, sizeof(unsigned long long), m->stream));
    } else {
        if ((rc = ensure_buf(&m->d_segs, &m->seg_cap, (size_t)n * sb.maxseg + 1))) return rc;
        if ((rc = ensure_buf(&m->d_perm, &m->perm_cap, m->seg_cap))) return rc;
        if ((rc = ensure_buf(&m->d_seg_bk, &m->seg_bk_cap, m->seg_cap))) return rc;
        if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, (size_t)n + 1))) return rc;
        if ((rc = ensure_records(m, std::max<size_t>(m->rec_cap, rec_floor(m, n_all)))))
            return rc;
    }
    sb.launches0 = m->launches;
    sb.nreg0 = m->nreg;
    CK(cudaMemsetAsync(m->d_shard_cnt, 0, (2 + (size_t)W) * sizeof(unsigned long long), m->stream));
    for (;;) {
        const long long headroom = std::max<long long>(512, 2 * m->max_growth);
        if ((rc = shard_headroom(m, 0))) return rc;
        m->epoch += 1;
        DevMap dm = shard_dm(m);
        CK(cudaMemsetAsync(m->d_stats, 0, NUM_STATS * sizeof(unsigned long long), m->stream));
        static const int box_init[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
        CK(cudaMemcpyAsync(m->d_rbox, box_init, sizeof(box_init), cudaMemcpyHostToDevice, m->stream));
        CK(cudaEventRecord(m->ev_start, m->stream));
        if (sb.n > 0) {
            rc = with_src(m, [&](auto src) {
                return launch_discover(m, dm, src, sb.n, mode, 1, sb.ndt ? 0 : 1, 1, m->stream);
            });
            if (rc) return rc;
        }
        const int margin = 64 + (int)std::min<long long>(1 << 20, headroom / 4);
        k_guard<<<1, 1, 0, m->stream>>>(dm, margin);
        m->launches += 2;
        if (!sb.ndt) {
            k_seg_scan<<<1, SEG_BUCKETS, 0, m->stream>>>(dm);
            k_seg_scatter<<<(unsigned)((n * sb.maxseg + BLOCK - 1) / BLOCK), BLOCK, 0, m->stream>>>(dm);
            m->launches += 2;
        }
        CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaMemcpyAsync(m->h_stats + NUM_STATS, m->d_cursor, sizeof(int), cudaMemcpyDeviceToHost,
                           m->stream));
        CK(cudaMemcpyAsync((int *)(m->h_stats + NUM_STATS) + 1, m->d_go, sizeof(int),
                           cudaMemcpyDeviceToHost, m->stream));
        // the slice's new sample voxels, read with the guard's verdict (one sync)
        CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 2, m->d_shard_cnt, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaStreamSynchronize(m->stream));
        const int cursor = *(const int *)(m->h_stats + NUM_STATS);
        const int go = *((const int *)(m->h_stats + NUM_STATS) + 1);
        if (m->h_stats[S_RANGE_ERR]) {
            m->nreg = cursor;
            return fail(VM_ERR_RANGE, "ray coordinates outside the packable region range");
        }
        if (!go) {
            m->max_growth = std::max<long long>(m->max_growth, cursor - m->nreg);
            if ((rc = grow_pool(m, std::max<long long>(2 * m->cap, cursor + 2 * margin + headroom))))
                return rc;
            m->nreg = cursor;
            continue;
        }
        m->nreg = cursor;
        break;
    }
    if (sb.ndt) {
        // requests: every ghost region of the slice's prefetch set (touched
        // list; its length came back with the guard's stats)
        counts_out[0] = (int64_t)m->h_stats[S_WALK_TOUCHED];
        counts_out[1] = 0;
        sb.nmarks = 0;
        sb.open = true;
        return VM_OK;
    }
    sb.nmarks = std::min<unsigned long long>(m->h_stats[NUM_STATS + 2], m->smarked_cap);
    counts_out[0] = (int64_t)(m->nreg - sb.nreg0);  // new regions (bound on the requests)
    counts_out[1] = (int64_t)sb.nmarks;
    sb.open = true;
    return VM_OK;
}

int vm_shard_lists(vm_map *m, int64_t *req_out, int64_t req_cap, int64_t *marks_out,
                   int64_t marks_cap, int64_t *counts_out) {
    if (!m || !m->sb.open || m->sb.walked || !counts_out)
        return fail(VM_ERR_ARG, "no discovered sharded batch");
    CK(cudaSetDevice(m->device));
    auto &sb = m->sb;
    const int W = m->shard_world;
    int rc;
    if ((long long)sb.nmarks > marks_cap || (!sb.ndt && req_cap < m->nreg - sb.nreg0))
        return fail(VM_ERR_ARG, "vm_shard_lists: buffers smaller than vm_shard_begin's counts");
    CK(cudaMemsetAsync(m->d_shard_cnt + 2, 0, (size_t)W * sizeof(unsigned long long), m->stream));
    DevMap dm = shard_dm(m);
    if (sb.ndt)
        k_shard_ndt_req<<<m->num_sms * 2, BLOCK, 0, m->stream>>>(dm, (long long *)req_out,
                                                                 m->d_shard_cnt + 2,
                                                                 (unsigned long long)req_cap);
    else
        k_shard_lists<<<m->num_sms * 2, BLOCK, 0, m->stream>>>(
            dm, (int)sb.nreg0, (int)m->nreg, (long long *)req_out, m->d_shard_cnt + 2,
            (unsigned long long)req_cap, (long long *)marks_out, sb.nmarks);
    m->launches += 1;
    if ((rc = check_launch("shard lists"))) return rc;
    std::vector<unsigned long long> nreq((size_t)W);
    CK(cudaMemcpyAsync(nreq.data(), m->d_shard_cnt + 2, (size_t)W * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    counts_out[0] = (int64_t)sb.nmarks;
    for (int d = 0; d < W; ++d) counts_out[1 + d] = (int64_t)nreq[d];
    return VM_OK;
}

int vm_shard_prepare(vm_map *m, const int64_t *req_in, int64_t nreq, const int64_t *marks_in,
                     int64_t nmarks) {
    if (!m || !m->sb.open || m->sb.walked) return fail(VM_ERR_ARG, "no sharded batch to prepare");
    CK(cudaSetDevice(m->device));
    int rc;
    if ((rc = shard_headroom(m, nreq))) return rc;
    DevMap dm = shard_dm(m);
    if (nreq > 0) {
        k_shard_prepare<<<(unsigned)std::min<long long>((nreq + BLOCK - 1) / BLOCK, 4096), BLOCK, 0,
                          m->stream>>>(dm, (const long long *)req_in, nreq);
        m->launches += 1;
    }
    // every rank's sample voxels, kept for the ghost clean-up in finish
    // (region key, li) pairs: two int2 slots per mark
    if ((rc = ensure_buf(&m->d_smarked, &m->smarked_cap, 2 * (size_t)std::max<int64_t>(nmarks, 0) + 2)))
        return rc;
    if (nmarks > 0) {
        CK(cudaMemcpyAsync(m->d_smarked, marks_in, (size_t)nmarks * 16, cudaMemcpyDeviceToDevice,
                           m->stream));
        k_shard_stamp<<<(unsigned)std::min<long long>((nmarks + BLOCK - 1) / BLOCK, 4096), BLOCK, 0,
                        m->stream>>>(dm, (const long long *)m->d_smarked, nmarks);
        m->launches += 1;
    }
    m->sb.nmarks = (unsigned long long)std::max<int64_t>(nmarks, 0);
    k_rgrid<<<16, BLOCK, 0, m->stream>>>(dm);
    m->launches += 1;
    if ((rc = check_launch("shard prepare"))) return rc;
    int cursor;
    if ((rc = read_cursor(m, &cursor))) return rc;
    m->nreg = cursor;
    m->sb.walk_slot0 = cursor;
    return VM_OK;
}

int vm_shard_ndt_bits(vm_map *m, const int64_t *req_in, int64_t nreq, uint32_t *bits_out) {
    if (!m || !m->sb.open || m->sb.walked || !m->sb.ndt)
        return fail(VM_ERR_ARG, "no discovered sharded NDT batch");
    if (nreq > 0 && (!req_in || !bits_out)) return fail(VM_ERR_ARG, "null argument");
    CK(cudaSetDevice(m->device));
    int rc;
    if ((rc = shard_headroom(m, nreq))) return rc;
    DevMap dm = shard_dm(m);
    if (nreq > 0) {
        const int words = (m->vpr + 31) / 32;
        k_shard_ndt_bits<<<(unsigned)std::min<long long>(nreq, 4096), BLOCK, 0, m->stream>>>(
            dm, (const long long *)req_in, nreq, bits_out, words);
        m->launches += 1;
        if ((rc = check_launch("shard ndt bits"))) return rc;
    }
    int cursor;
    if ((rc = read_cursor(m, &cursor))) return rc;
    m->nreg = cursor;
    return VM_OK;
}

int vm_shard_ndt_mark(vm_map *m, const int64_t *keys, const uint32_t *bits, int64_t n) {
    if (!m || !m->sb.open || m->sb.walked || !m->sb.ndt)
        return fail(VM_ERR_ARG, "no discovered sharded NDT batch");
    if (n > 0 && (!keys || !bits)) return fail(VM_ERR_ARG, "null argument");
    CK(cudaSetDevice(m->device));
    DevMap dm = shard_dm(m);
    if (n > 0) {
        const int words = (m->vpr + 31) / 32;
        k_shard_ndt_mark<<<(unsigned)std::min<long long>(n, 4096), BLOCK, 0, m->stream>>>(
            dm, (const long long *)keys, bits, n, words);
        m->launches += 1;
    }
    m->sb.walk_slot0 = (int)m->nreg;
    return check_launch("shard ndt mark");
}

int vm_shard_walk(vm_map *m) {
    if (!m || !m->sb.open || m->sb.walked) return fail(VM_ERR_ARG, "no sharded batch to walk");
    CK(cudaSetDevice(m->device));
    int rc;
    if ((rc = shard_headroom(m, 0))) return rc;
    DevMap dm = shard_dm(m);
    CK(cudaMemsetAsync(m->d_work, 0, sizeof(unsigned long long), m->stream));
    CK(cudaEventRecord(m->ev_w0, m->stream));
    if (m->sb.n > 0 && m->sb.ndt) {
        dm.ray_order = 0;
        const long long n = m->sb.n;
        rc = with_src(m, [&](auto src) {
            k_walk_ndt<false, true, false><<<(unsigned)((n + BLOCK - 1) / BLOCK), BLOCK, 0,
                                             m->stream>>>(dm, src, n);
            return check_launch("shard ndt walk");
        });
        if (rc) return rc;
        m->launches += 1;
    } else if (m->sb.n > 0) {
        const dim3 pgrid((unsigned)std::max<long long>(
            1, std::min<long long>((long long)WK_BLOCKS * m->num_sms, (m->sb.n * 3 + BLOCK - 1) / BLOCK)));
        rc = with_src(m, [&](auto src) {
            using S = decltype(src);
            DevMap d2 = dm;
            d2.walk_det_launched = 1;
            cudaError_t e = launch_wd<false, S>(pgrid, m->stream, d2, src);
            if (e == cudaSuccess)
                e = launch_w3<M_OCC, true, false, S>(pgrid, sizeof(WalkSmem), m->stream, d2, src);
            if (e != cudaSuccess)
                return fail(VM_ERR_CUDA, std::string("shard walk shared-memory opt-in: ") +
                                             cudaGetErrorString(e));
            return check_launch("shard walk");
        });
        if (rc) return rc;
        m->launches += 2;
    }
    CK(cudaEventRecord(m->ev_w1, m->stream));
    m->sb.walked = true;
    return VM_OK;
}

int vm_shard_export(vm_map *m, void *out, int64_t cap_per_dest, int64_t *per_dest_out) {
    if (!m || !m->sb.open || !m->sb.walked || !per_dest_out)
        return fail(VM_ERR_ARG, "no walked sharded batch to export");
    CK(cudaSetDevice(m->device));
    const int W = m->shard_world;
    CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 2, m->d_stats + S_RECORDS, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, m->stream));
    if (m->sb.ndt)  // the ghost-visit count, in the same round trip
        CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 3, m->d_ngx, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    const unsigned long long R = m->h_stats[NUM_STATS + 2];
    if (R > m->rec_cap) return fail(VM_ERR_OOM, "record buffer overflow in a sharded batch");
    m->sb.R = R;
    DevMap dm = shard_dm(m);
    CK(cudaMemsetAsync(m->d_shard_cnt + 2, 0, (size_t)W * sizeof(unsigned long long), m->stream));
    const unsigned long long cap = (unsigned long long)std::max<int64_t>(cap_per_dest, 0);
    if (m->sb.ndt) {
        const unsigned long long ng = m->h_stats[NUM_STATS + 3];
        if (ng > m->gx_cap) return fail(VM_ERR_OOM, "ghost visit buffer overflow in a sharded batch");
        k_shard_ndt_export<<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm, R, (ShardItemN *)out,
                                                                    m->d_shard_cnt + 2, cap);
        m->launches += 1;
    } else if (R > 0)
        k_shard_export_rec<<<(unsigned)std::min<unsigned long long>((R + BLOCK - 1) / BLOCK, 4096),
                             BLOCK, 0, m->stream>>>(dm, m->d_rec, (long long)R, (ShardItem *)out,
                                                    m->d_shard_cnt + 2, cap);
    if (!m->sb.ndt) {
        k_shard_export_cnt<<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm, (ShardItem *)out,
                                                                    m->d_shard_cnt + 2, cap);
        m->launches += 2;
    }
    int rc;
    if ((rc = check_launch("shard export"))) return rc;
    std::vector<unsigned long long> cnt((size_t)W);
    CK(cudaMemcpyAsync(cnt.data(), m->d_shard_cnt + 2, (size_t)W * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    bool over = false;
    for (int d = 0; d < W; ++d) {
        per_dest_out[d] = (int64_t)cnt[d];
        over = over || cnt[d] > cap;
    }
    if (over) return fail(VM_ERR_ARG, "export buffer too small (per_dest_out holds the sizes)");
    return VM_OK;
}

int vm_shard_import(vm_map *m, const void *in, int64_t n) {
    if (!m || !m->sb.open || !m->sb.walked) return fail(VM_ERR_ARG, "no sharded batch to import into");
    CK(cudaSetDevice(m->device));
    int rc;
    if (n > 0) {
        const unsigned g = (unsigned)std::min<long long>((n + BLOCK - 1) / BLOCK, 8192);
        {
            DevMap dm = shard_dm(m);
            if (m->sb.ndt)
                k_shard_ndt_import_regions<<<g, BLOCK, 0, m->stream>>>(dm, (const ShardItemN *)in, n);
            else
                k_shard_import_regions<<<g, BLOCK, 0, m->stream>>>(dm, (const ShardItem *)in, n);
        }
        int cursor;
        if ((rc = read_cursor(m, &cursor))) return rc;
        m->nreg = cursor;
        if ((rc = shard_headroom(m, 0))) return rc;  // covers every slot pass 1 handed out
        DevMap dm = shard_dm(m);
        if (m->sb.ndt) {
            rc = with_src(m, [&](auto src) {
                k_shard_ndt_import<<<g, BLOCK, 0, m->stream>>>(dm, src, (const ShardItemN *)in, n);
                return VM_OK;
            });
            if (rc) return rc;
        } else {
            k_shard_import<<<g, BLOCK, 0, m->stream>>>(dm, (const ShardItem *)in, n);
        }
        m->launches += 2;
        if ((rc = check_launch("shard import"))) return rc;
    }
    return VM_OK;  // vm_shard_finish reads the region cursor
}

int vm_shard_finish(vm_map *m, vm_stats *out) {
    if (!m || !m->sb.open || !m->sb.walked || !out) return fail(VM_ERR_ARG, "no sharded batch to finish");
    CK(cudaSetDevice(m->device));
    auto &sb = m->sb;
    int rc;
    // region cursor, stats and (NDT) the voxel-index count in one round trip
    CK(cudaMemcpyAsync(m->h_stats + NUM_STATS, m->d_cursor, sizeof(int), cudaMemcpyDeviceToHost,
                       m->stream));
    CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, m->stream));
    if (sb.ndt)
        CK(cudaMemcpyAsync(m->h_stats + NUM_STATS + 2, m->d_shard_cnt, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    const int cursor = *(const int *)(m->h_stats + NUM_STATS);
    m->nreg = cursor;
    const unsigned long long Rtot = std::min<unsigned long long>(m->h_stats[S_RECORDS], m->rec_cap);
    if (m->h_stats[S_RECORDS] > m->rec_cap) return fail(VM_ERR_OOM, "record buffer overflow on import");
    if (sb.ndt) {
        // ghost state out, then the single-GPU tail: resolve, buckets, fold
        DevMap dm = shard_dm(m);
        k_shard_ndt_clear<<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
        CK(cudaEventRecord(m->ev_k1, m->stream));
        k_resolve<true, false><<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
        CK(cudaEventRecord(m->ev_res, m->stream));
        if (m->h_stats[NUM_STATS + 2] > m->smarked_cap)
            return fail(VM_ERR_OOM, "voxel index overflow in a sharded NDT batch");
        rc = with_src(m, [&](auto src) {
            return launch_ndt_fold(m, dm, src, sb.n_all, sb.maxseg, false, m->ev_sort);
        });
        if (rc) return rc;
        m->launches += 2;
        CK(cudaEventRecord(m->ev_end, m->stream));
        CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, m->stream));
        CK(cudaStreamSynchronize(m->stream));
        if ((rc = check_launch("shard finish"))) return rc;
        const unsigned long long *hs = m->h_stats;
        std::memset(out, 0, sizeof(*out));
        out->rays_in = sb.n;
        out->rays_processed = (int64_t)hs[S_PROCESSED];
        out->segments = (int64_t)hs[S_SEGMENTS];
        out->voxel_visits = (int64_t)hs[S_VISITS];
        out->region_misses = (int64_t)hs[S_RMISS];
        out->regions_touched = (int64_t)hs[S_PREF_TOUCHED];
        out->records = (int64_t)Rtot;
        out->regions_total = cursor;
        out->new_regions = cursor - sb.nreg0;
        out->touched_regions_walk = (int64_t)hs[S_WALK_TOUCHED];
        out->launches = m->launches - sb.launches0;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, m->ev_start, m->ev_end) == cudaSuccess) out->gpu_ms = ms;
        if (cudaEventElapsedTime(&ms, m->ev_w0, m->ev_w1) == cudaSuccess) out->walk_ms = ms;
        if (cudaEventElapsedTime(&ms, m->ev_k1, m->ev_res) == cudaSuccess) out->resolve_ms = ms;
        if (cudaEventElapsedTime(&ms, m->ev_res, m->ev_sort) == cudaSuccess) out->sort_ms = ms;
        if (cudaEventElapsedTime(&ms, m->ev_sort, m->ev_end) == cudaSuccess) out->fold_ms = ms;
        m->max_growth = std::max<long long>(m->max_growth, cursor - sb.nreg0);
        sb.open = false;
        return VM_OK;
    }
    const int vbits = std::max(1, bitlen((unsigned long long)(cursor + 1) * m->vpr));
    const int end_bit = std::min(64, sb.order_bits + vbits);
    DevMap dm = shard_dm(m);
    dm.rec_invalid = (1ULL << vbits) - 1;
    const unsigned long long invalid_key = dm.rec_invalid << sb.order_bits;
    k_shard_clear<<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm, m->d_rec, (long long)sb.R, invalid_key,
                                                          (const long long *)m->d_smarked,
                                                          (long long)sb.nmarks);
    CK(cudaEventRecord(m->ev_k1, m->stream));
    k_resolve<false, false><<<m->num_sms * 8, BLOCK, 0, m->stream>>>(dm);
    CK(cudaEventRecord(m->ev_res, m->stream));
    cub::DoubleBuffer<unsigned long long> db(m->d_rec, m->d_rec2);
    if (Rtot > 1) {
        if ((rc = ensure_sort_tmp(m))) return rc;
        size_t bytes = m->sort_tmp_bytes;
        CK(cub::DeviceRadixSort::SortKeys(m->d_sort_tmp, bytes, db, (int)Rtot, 0, end_bit, m->stream));
    }
    CK(cudaEventRecord(m->ev_sort, m->stream));
    rc = with_src(m, [&](auto src) {
        return launch_fold(m, dm, src, db.Current(), m->d_val, (long long)Rtot, M_OCC);
    });
    if (rc) return rc;
    m->launches += 2;
    CK(cudaEventRecord(m->ev_end, m->stream));
    CK(cudaMemcpyAsync(m->h_stats, m->d_stats, NUM_STATS * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    if ((rc = check_launch("shard finish"))) return rc;
    const unsigned long long *hs = m->h_stats;
    std::memset(out, 0, sizeof(*out));
    out->rays_in = sb.n;
    out->rays_processed = (int64_t)hs[S_PROCESSED];
    out->segments = (int64_t)hs[S_SEGMENTS];
    out->voxel_visits = (int64_t)hs[S_VISITS];
    out->region_misses = (int64_t)hs[S_RMISS];
    out->regions_touched = (int64_t)hs[S_PREF_TOUCHED];
    out->records = (int64_t)Rtot;
    out->marked_voxels = (int64_t)sb.nmarks;
    out->regions_total = cursor;
    out->new_regions = cursor - sb.nreg0;
    out->touched_regions_walk = (int64_t)hs[S_WALK_TOUCHED];
    out->launches = m->launches - sb.launches0;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, m->ev_start, m->ev_end) == cudaSuccess) out->gpu_ms = ms;
    if (cudaEventElapsedTime(&ms, m->ev_w0, m->ev_w1) == cudaSuccess) out->walk_ms = ms;
    if (cudaEventElapsedTime(&ms, m->ev_k1, m->ev_res) == cudaSuccess) out->resolve_ms = ms;
    if (cudaEventElapsedTime(&ms, m->ev_res, m->ev_sort) == cudaSuccess) out->sort_ms = ms;
    if (cudaEventElapsedTime(&ms, m->ev_sort, m->ev_end) == cudaSuccess) out->fold_ms = ms;
    m->max_growth = std::max<long long>(m->max_growth, cursor - sb.nreg0);
    sb.open = false;
    return VM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// L2-atomic ceiling probe (vm_probe_red_rate): the roofline of the walk's
// per-visit RED.ADD, measured on the device at hand.
namespace {
__global__ void __launch_bounds__(256) k_red_probe(unsigned *buf, unsigned mask, int per_thread) {
    unsigned x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
#pragma unroll 8
    for (int i = 0; i < per_thread; ++i) {
        x = x * 1664525u + 1013904223u;  // LCG: one IMAD per RED
        red_add(buf + ((x >> 7) & mask), 1u);
    }
}
}  // namespace

int vm_probe_red_rate(int32_t device, int64_t footprint_bytes, int32_t reps, double *out) {
    if (!out || footprint_bytes < 4096 || reps < 1) return fail(VM_ERR_ARG, "bad probe arguments");
    CK(cudaSetDevice(device));
    unsigned long long words = 1;
    while (words * 2 * 4 <= (unsigned long long)footprint_bytes) words <<= 1;
    unsigned *buf = nullptr;
    CK(cudaMalloc(&buf, words * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * 8, per = 1024;
    double best = 0.0;
    cudaMemset(buf, 0, words * 4);
    k_red_probe<<<blocks, 256>>>(buf, (unsigned)(words - 1), per);  // warm-up
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        k_red_probe<<<blocks, 256>>>(buf, (unsigned)(words - 1), per);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms > 0.f) best = std::max(best, (double)blocks * 256.0 * per / (ms * 1e-3));
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    if (err != cudaSuccess) return fail(VM_ERR_CUDA, std::string("red probe: ") + cudaGetErrorString(err));
    *out = best;
    return VM_OK;
}
