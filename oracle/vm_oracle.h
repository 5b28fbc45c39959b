/*
 * vm_oracle.h -- CPU restatement of the reference's ray-integration path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA
 * product path (paper_2206_06079_b200/csrc).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product never links or calls it.
 *
 * It restates, in plain C, the *sequential* executor of the reference
 * package `voxmap` 0.1.0:
 *   engine._preprocess / prefetch_regions / _run_sequential
 *       (/root/reference/pkg/src/voxmap/engine.py:82-118,222-237)
 *   traversal._walk_grid / clip_ray / segment_ray
 *       (/root/reference/pkg/src/voxmap/traversal.py:52-111,140-178)
 *   reference.integrate_occupancy_segment / ndt_phase1_segment /
 *       apply_ndt_hits / integrate_tsdf_ray / sample_buckets
 *       (/root/reference/pkg/src/voxmap/reference.py:35-186)
 *   subvoxel.py:16-49, ndt.py:37-106, tsdf.py:21-26, keys.py:76-86.
 *
 * Pinned against golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py).  Known deliberate deviation: the NDT miss
 * likelihood uses the adjugate inverse of the reference's native kernel
 * (_kernels.pyx:473-525) instead of numpy.linalg.inv (ndt.py:86), so NDT
 * phase-1 values are tolerance-graded, never bit-graded.
 */
#ifndef VM_ORACLE_H
#define VM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double voxel_size;
    int32_t region_dim;
    int32_t _pad;
    double hit_delta;      /* prob_to_logodds(p_hit), computed by the caller */
    double miss_delta;     /* prob_to_logodds(p_miss) */
    double clamp_min;
    double clamp_max;
    double max_ray_range;
    double segment_length;
    double tsdf_truncation;
    double tsdf_max_weight;
    double ndt_sensor_noise;
    double ndt_reset_threshold;
    double ndt_miss_likelihood_threshold;
} orc_config;

enum { ORC_MODE_OCCUPANCY = 0, ORC_MODE_DECAY = 1, ORC_MODE_NDT_OM = 2,
       ORC_MODE_NDT_TM = 3, ORC_MODE_TSDF = 4,
       /* checker aid, not a reference mode: per-voxel hit / miss visit counts
        * of the occupancy walk into the hit_count / miss_count layers */
       ORC_MODE_COUNTS = 5 };

/* stats layout: rays_in, rays_processed, segments, voxel_visits,
 * cas_retries, cas_failures, region_misses, regions_touched */
#define ORC_NSTATS 8

typedef struct orc_map orc_map;

orc_map *orc_map_create(const orc_config *cfg, uint32_t layer_mask);
void orc_map_destroy(orc_map *m);
int64_t orc_map_region_count(const orc_map *m);
/* region coordinates (n x 3, int64) in creation order; returns count written */
int64_t orc_map_regions(const orc_map *m, int64_t *coords_out, int64_t cap);
/* pointer to a layer buffer of region (rx,ry,rz), or NULL if absent */
void *orc_map_layer(orc_map *m, int64_t rx, int64_t ry, int64_t rz, int32_t layer_id);
/* ensure region exists (used to seed maps from host data) */
void *orc_map_layer_create(orc_map *m, int64_t rx, int64_t ry, int64_t rz, int32_t layer_id);

/* sequential_reference(vmap, rays, mode): rays as f64 origins/ends (n x 3),
 * u8 has_sample, f32 intensity.  Returns 0 on success. */
int orc_integrate(orc_map *m, const double *origins, const double *ends,
                  const uint8_t *has_sample, const float *intensity, int64_t n,
                  int32_t mode, int64_t *stats_out);

/* traversal._walk_grid; returns visit count or -1 if cap exceeded */
int64_t orc_walk(double ox, double oy, double oz, double ex, double ey, double ez,
                 double cell, int64_t *coords, double *t0, double *t1, int64_t cap);

/* engine._preprocess (clip, optional segmentation); returns #segments,
 * or -1 if cap is exceeded.  seg_ray gets the input ray index. */
int64_t orc_preprocess(const orc_config *cfg, const double *origins, const double *ends,
                       const uint8_t *has_sample, int64_t n, int32_t segment,
                       double *seg_o, double *seg_e, uint8_t *seg_has, int64_t *seg_ray,
                       int64_t cap, int64_t *processed_out);

/* engine.prefetch_regions (engine.py:99-118) over pre-built segments:
 * distinct region coords (n x 3) touched by the coarse region DDA, in
 * first-touch order.  Returns the count, or -1 if cap is exceeded. */
int64_t orc_prefetch_regions(const orc_config *cfg, const double *seg_o, const double *seg_e,
                             const uint8_t *seg_has, int64_t n, double extra_reach,
                             int64_t *coords_out, int64_t cap);

double orc_norm3(double x, double y, double z);
double orc_py_hypot(double a, double b);
uint64_t orc_hash_mix(int64_t key);

#ifdef __cplusplus
}
#endif
#endif
