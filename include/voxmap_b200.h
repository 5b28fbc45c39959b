/*
 * voxmap_b200.h -- C ABI of the B200-native ray-integration path.
 *
 * Drop-in boundary for the reference package `voxmap` 0.1.0, whose only
 * native boundary is the Cython extension `voxmap._kernels`
 * (/root/reference/pkg/setup.py:5-13, src/voxmap/_kernels.pyx).  Plain C
 * types only: pointers, sizes, ints and doubles.  No torch types.
 *
 * Two layers:
 *
 *  1. `vm_kernels_*`, `vm_walk_voxels`, `vm_hash_mix`: one-to-one
 *     replacements of the `_kernels` entry points, same argument meaning
 *     (segment arrays, open-addressing region table with splitmix64 keys,
 *     per-layer region pointer arrays), except that every array is a
 *     DEVICE pointer and the work runs on a CUDA stream.
 *
 *  2. `vm_map_*`, `vm_integrate`: the device-resident map runtime that
 *     `engine.submit_batch` (engine.py:175-210) calls.  It owns the
 *     region table, the per-layer region pools in HBM and the batch
 *     pipeline (preprocess -> region discovery -> DDA walk -> resolve /
 *     sort+fold), and reproduces the reference's sequential semantics
 *     (engine.py:213-237) in VM_EXEC_DETERMINISTIC mode.
 *
 * All functions return VM_OK (0) or an error code; vm_last_error() gives
 * a thread-local message.  Errors never leave a half-applied batch: a
 * batch either integrates completely or the map is unchanged.
 */
#ifndef VOXMAP_B200_H
#define VOXMAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VM_OK 0
#define VM_ERR_ARG 1     /* bad argument (reference: ValueError)            */
#define VM_ERR_CUDA 2    /* CUDA runtime failure                            */
#define VM_ERR_OOM 3     /* device allocation failed (reference: MemoryError) */
#define VM_ERR_RANGE 4   /* region coordinate outside the 21-bit packing,
                            keys.py:76-86 (reference: ValueError)           */
#define VM_ERR_NODEV 5   /* no CUDA device                                  */

/* Map geometry and sensor model: MapConfig fields (config.py:8-28).  The
 * log-odds deltas are passed precomputed (occupancy.py:20-35). */
typedef struct vm_config {
    double voxel_size;
    int32_t region_dim;
    int32_t _pad;
    double hit_delta;
    double miss_delta;
    double clamp_min;
    double clamp_max;
    double max_ray_range;
    double segment_length;
    double tsdf_truncation;
    double tsdf_max_weight;
    double ndt_sensor_noise;
    double ndt_reset_threshold;
    double ndt_miss_likelihood_threshold;
} vm_config;

/* Batch statistics: BatchStats (engine.py:33-64) plus device counters. */
typedef struct vm_stats {
    int64_t rays_in;
    int64_t rays_processed;
    int64_t segments;
    int64_t voxel_visits;
    int64_t cas_retries;
    int64_t cas_failures;     /* always 0: no mutex fallback on the GPU */
    int64_t region_misses;
    int64_t regions_touched;  /* prefetch set size, engine.py:99-118 */
    int64_t records;          /* order-keyed records sorted this batch */
    int64_t marked_voxels;    /* sample voxels (deterministic mode) */
    int64_t regions_total;    /* regions in the map after the batch */
    int64_t new_regions;
    int64_t replays;          /* batch re-runs after a pool growth */
    int64_t touched_regions_walk;
    int64_t launches;         /* kernels of this library launched for the batch */
    double gpu_ms;            /* device time of the whole batch (CUDA events) */
    double walk_ms;           /* device time of the DDA walk kernel */
    double discover_ms;       /* preprocess + region discovery (+ dense grid) */
    double resolve_ms;        /* order-free miss counts -> log-odds */
    double sort_ms;           /* record sort */
    double fold_ms;           /* in-order record fold + cleanup */
} vm_stats;

enum { VM_MODE_OCCUPANCY = 0, VM_MODE_DECAY = 1, VM_MODE_NDT_OM = 2, VM_MODE_NDT_TM = 3,
       VM_MODE_TSDF = 4 };
enum { VM_EXEC_CAS = 0, VM_EXEC_DETERMINISTIC = 1 };
enum { VM_RAYS_OHMB1 = 0, VM_RAYS_F64 = 1 };

/* Layer ids (layers.py:22-31); layer_mask bit (1 << id). */
enum { VM_LAYER_OCCUPANCY = 1, VM_LAYER_MEAN = 2, VM_LAYER_MEAN_COUNT = 3,
       VM_LAYER_COV_SQRT = 4, VM_LAYER_HIT_COUNT = 5, VM_LAYER_MISS_COUNT = 6,
       VM_LAYER_INTENSITY = 7, VM_LAYER_DECAY_HITS = 8, VM_LAYER_DECAY_DISTANCE = 9,
       VM_LAYER_TSDF = 10 };

/* A ray batch.  VM_RAYS_OHMB1: `records` points at packed 40-byte OHMB1
 * records (rayset.py:19-27: f64 timestamp, f32 origin[3], f32 end[3],
 * f32 intensity, u32 flags), converted to f64 exactly as to_ray_samples
 * does (rayset.py:74-84).  VM_RAYS_F64: RaySample arrays (traversal.py:20-42):
 * origins/ends [n][3] f64, has_sample u8[n], intensity f32[n] (may be NULL).
 * on_device: 0 = host pointers (copied in on the map stream; pinned memory
 * overlaps), 1 = device pointers. */
typedef struct vm_rays {
    int32_t format;
    int32_t on_device;
    int64_t count;
    const void *records;
    const double *origins;
    const double *ends;
    const uint8_t *has_sample;
    const float *intensity;
} vm_rays;

typedef struct vm_map vm_map;

/* ---- map runtime (replaces store.VoxelMap's buffers, store.py:28-80) ---- */

/* Create a device map on `device` with the given layers.  initial_regions
 * sizes the HBM region pool (it grows by doubling between batches). */
int vm_map_create(const vm_config *cfg, uint32_t layer_mask, int32_t device,
                  int64_t initial_regions, vm_map **out);
int vm_map_destroy(vm_map *map);
/* Drop every region (the map becomes empty; pool capacity is kept). */
int vm_map_reset(vm_map *map);
/* Use an external CUDA stream (cudaStream_t) for all map work; NULL = own stream. */
int vm_map_set_stream(vm_map *map, void *cuda_stream);

/* Region recency and eviction (store.py:28-39, 112-174).
 * vm_map_set_batch_counter: the VoxelMap.batch_counter value the next batch
 *   stamps on every region its prefetch touches (engine.py:99-118 refreshes
 *   Region.last_access the same way); a pipelined sequence counts on from it.
 * vm_map_region_last_access: those stamps for slots [first, first + count).
 * vm_map_set_spill: the spill directory and the host map's layer order (the
 *   OHMS1 payload order).
 * vm_map_evict_regions: write each region in keys[] to
 *   <dir>/region_<x>_<y>_<z>.bin -- b"OHMS1", <3q I> key and layer count, u32
 *   layer ids, zlib level 6 of the layer bytes, byte-compatible with the
 *   reference's _write_spill -- drop it from HBM and compact the pool (slots
 *   stay dense and creation-ordered; host mirrors must be re-read).  A failed
 *   write keeps the region.  *evicted_out counts the regions spilled.
 * A batch whose prefetch reaches a spilled region reloads it first (the
 *   guard refuses the attempt, the runtime reloads, the batch replays);
 *   vm_map_reload_region / vm_map_ensure_regions reload on demand.  Reloading
 *   consumes the file. */
int vm_map_set_batch_counter(vm_map *map, uint32_t counter);
int vm_map_region_last_access(vm_map *map, int64_t first, int64_t count, uint32_t *out);
int vm_map_set_spill(vm_map *map, const char *dir, const int32_t *layer_ids, int32_t n);
int vm_map_evict_regions(vm_map *map, const int64_t *keys, int64_t n, int64_t *evicted_out);
int vm_map_reload_region(vm_map *map, int64_t key, int32_t *slot_out);
int vm_map_spilled_keys(vm_map *map, int64_t *out, int64_t cap, int64_t *n_out);
int vm_map_region_count(const vm_map *map, int64_t *out);
/* Packed region keys (keys.py:76-86) of slots [first, first+count), in slot
 * (creation) order. */
int vm_map_region_keys(const vm_map *map, int64_t first, int64_t count, int64_t *keys_out);
/* get_or_create_region (store.py:67-80) for host-driven region creation. */
int vm_map_ensure_regions(vm_map *map, const int64_t *packed_keys, int64_t n,
                          int32_t *slots_out);
/* Region slot of a packed key or -1 (store.py:67-77 without create). */
int vm_map_find_region(vm_map *map, int64_t packed_key, int32_t *slot_out);
/* Copy one region's layer buffer (region_dim^3 * components elements)
 * device->host / host->device on the map stream (synchronous). */
int vm_map_read_layer(vm_map *map, int32_t slot, int32_t layer_id, void *host_dst,
                      int64_t bytes);
int vm_map_write_layer(vm_map *map, int32_t slot, int32_t layer_id, const void *host_src,
                       int64_t bytes);
/* Device pointer of a region's layer buffer (valid until the next batch
 * that grows the pool). */
int vm_map_layer_ptr(vm_map *map, int32_t slot, int32_t layer_id, void **dev_ptr_out);

/* ---- the hot path: submit_batch (engine.py:175-210) ---- */

/* Integrate one batch: clip + segment (traversal.py:140-178), region
 * prefetch (engine.py:99-118), DDA walk and layer updates.  exec =
 * VM_EXEC_DETERMINISTIC reproduces sequential_reference (engine.py:213-216)
 * bit-for-bit on occupancy / mean / mean_count / decay_hits / tsdf;
 * VM_EXEC_CAS is the paper's atomic compare-and-swap update
 * (_kernels.pyx:233-357).  Synchronous: returns after the batch is
 * complete and `out` is filled. */
int vm_integrate(vm_map *map, const vm_rays *rays, int32_t mode, int32_t exec,
                 vm_stats *out);

/* Exporters (exporters.py:14-159).  vm_export_select: the voxels a format
 * keeps, in the reference's order (regions as given -- the caller passes the
 * slots of the sorted region keys, exporters.py:33-41 -- then local index).
 * kind: 0 occupied (log-odds > threshold, :53), 1 NDT (mean_count > 0, :88),
 * 2 TSDF (weight != 0, :131), 3 decay (hits or distance != 0, :149).
 * *count_out is always set; ridx/li are filled when cap >= the count.
 * vm_export_gather: the layer records of the selected voxels (host out). */
int vm_export_select(vm_map *map, const int32_t *slots, int64_t nslots, int32_t kind,
                     double threshold, int64_t *count_out, int32_t *ridx_out, int32_t *li_out,
                     int64_t cap);
int vm_export_gather(vm_map *map, int32_t layer, const int32_t *slots, int64_t nslots,
                     const int32_t *ridx, const int32_t *li, int64_t n, void *out);

/* A sequence of batches, integrated in order with the same result as one
 * vm_integrate call per batch (out[i] = that call's stats).  Deterministic
 * occupancy over OHMB1 records is pipelined: every batch is enqueued with no
 * host round trip, host records are uploaded while earlier batches compute,
 * and the call syncs once at the end.  Other modes loop over vm_integrate.
 * Replaces the reference CLI's offline replay loop over submit_batch
 * (cli.py:122-127, engine.py:175-210). */
int vm_integrate_many(vm_map *map, const vm_rays *rays, int32_t nbatches, int32_t mode,
                      int32_t exec, vm_stats *out);

/* ---- `_kernels` one-to-one entry points (device pointers) ---- */

/* _kernels.walk_voxels_native (_kernels.pyx:214-228): walk one segment on
 * the GPU; coords_out [cap][3] i64, t0/t1 [cap] f64 host buffers.
 * Returns VM_ERR_ARG if the walk needs more than cap visits. */
int vm_walk_voxels(double ox, double oy, double oz, double ex, double ey, double ez,
                   double cell, int64_t cap, int64_t *coords_out, double *t0_out,
                   double *t1_out, int64_t *n_out);

/* math.hypot as ndt.cholupdate3 calls it (ndt.py:37-52; CPython 3.12
 * vector_norm): the device restatement the NDT fold runs, on n pairs
 * ab[2n] (host buffer) into out[n] (host buffer).  A parity probe. */
int vm_ndt_hypot(const double *ab, int64_t n, double *out);

/* _kernels.hash_mix (_kernels.pyx:105-110,127-129): splitmix64 finalizer. */
uint64_t vm_hash_mix(int64_t key);

/* _kernels.integrate_occupancy (_kernels.pyx:376-470): CAS occupancy
 * (+ mean when mean_ptrs/count_ptrs are non-NULL, + decay when
 * dhit_ptrs/ddist_ptrs are non-NULL) over n segments.  tkeys/tvals: the
 * open-addressing region table of engine._build_region_table
 * (engine.py:121-147), tsize a power of two.  *_ptrs: device arrays of
 * per-region device buffer pointers.  stats_out[4] = (cas_retries,
 * cas_failures, region_misses, visits).  stream: cudaStream_t or NULL. */
int vm_kernels_integrate_occupancy(const double *origins, const double *ends,
                                   const uint8_t *has_sample, int64_t n,
                                   const int64_t *tkeys, const int32_t *tvals, int64_t tsize,
                                   void *const *occ_ptrs, void *const *mean_ptrs,
                                   void *const *count_ptrs, void *const *dhit_ptrs,
                                   void *const *ddist_ptrs, double voxel_size,
                                   int64_t region_dim, double hit_delta, double miss_delta,
                                   double clamp_min, double clamp_max, int32_t retry_limit,
                                   int32_t walk_cap, int64_t *stats_out, void *stream);

/* ---- region-sharded integration over G GPUs ----
 *
 * Map `rank` of `world` owns the regions with vm_shard_owner(key, world) ==
 * rank (2 x 2 x 2 region blocks hashed over the ranks) and walks the slice
 * [rank*N/world, (rank+1)*N/world) of each batch; every rank passes the whole
 * batch.  Deterministic occupancy only.  One batch = begin, exchange A
 * (requests all-to-all, marks all-gather), prepare, walk, export, exchange B
 * (items all-to-all), import, finish.  All int64_t / void buffers below are
 * DEVICE buffers except counts_out / per_dest_out (host).  The union of the
 * ranks' owned regions equals the single-GPU map, bit for bit. */
int vm_shard_config(vm_map *map, int32_t rank, int32_t world);
int vm_shard_owner(int64_t packed_key, int32_t world);
/* Discover the slice: counts_out[2] = (#new regions, #new sample voxels). */
int vm_shard_begin(vm_map *map, const vm_rays *rays, int32_t mode, int32_t exec, int64_t *counts_out);
/* req_out: world segments of req_cap (>= #new regions) packed keys -- the new
 * regions owned by rank d (creation requests) go to segment d; marks_out:
 * (packed key, li) int64 pairs of the slice's new sample voxels;
 * counts_out[1 + world] = (#marks, #requests for rank 0 .. world-1). */
int vm_shard_lists(vm_map *map, int64_t *req_out, int64_t req_cap, int64_t *marks_out,
                   int64_t marks_cap, int64_t *counts_out);
/* req_in: requests addressed to this rank; marks_in: every rank's marks. */
int vm_shard_prepare(vm_map *map, const int64_t *req_in, int64_t nreq, const int64_t *marks_in,
                     int64_t nmarks);
/* NDT-OM batches (vm_shard_ndt.cuh): vm_shard_lists' req_out holds every
 * ghost region of the slice's prefetch set, per owner.  The owner answers a
 * request list with the regions' Gaussian bitmaps -- ceil(vpr / 32) u32 words
 * per region, bit li set when voxel li holds >= 3 samples -- creating the
 * regions it lacks; the requester marks its ghost voxels from them. */
int vm_shard_ndt_bits(vm_map *map, const int64_t *req_in, int64_t nreq, uint32_t *bits_out);
int vm_shard_ndt_mark(vm_map *map, const int64_t *keys, const uint32_t *bits, int64_t n);
int vm_shard_walk(vm_map *map);
/* out: world segments of cap_per_dest 16-byte items (region key, li | kind
 * << 31, count or ray order | hit) -- 32-byte items for NDT-OM batches
 * (region key, li | kind << 30, count or segment order, chord t0, t1);
 * per_dest_out[world] gets the sizes
 * (VM_ERR_ARG if a segment overflowed: retry with a larger cap). */
int vm_shard_export(vm_map *map, void *out, int64_t cap_per_dest, int64_t *per_dest_out);
int vm_shard_import(vm_map *map, const void *in, int64_t n);
int vm_shard_finish(vm_map *map, vm_stats *out);

/* Ceiling probe for the contended walk path (not a reference interface):
 * fire-and-forget u32 reductions (RED.ADD, the walk's per-visit update) at
 * pseudo-random word addresses inside a `footprint_bytes` buffer on `device`
 * -- small enough to stay in L2, as the walk's touched scratch words do.
 * reds_per_s_out: the measured L2 atomic throughput (best of `reps` launches). */
int vm_probe_red_rate(int32_t device, int64_t footprint_bytes, int32_t reps, double *reds_per_s_out);

const char *vm_last_error(void);
int vm_device_count(int32_t *out);
/* Build-time identification string (arch, flags). */
const char *vm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* VOXMAP_B200_H */
