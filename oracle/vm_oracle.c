/*
 * vm_oracle.c -- CPU restatement of voxmap's sequential integration path.
 * TEST INFRASTRUCTURE ONLY (see vm_oracle.h).  Built with
 * -ffp-contract=off so every a*b+c rounds twice unless fma() is written
 * out, exactly like the numpy ufunc / CPython float arithmetic it restates.
 */
#include "vm_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* layers (layers.py:22-31)                                            */

static const int LAYER_ELEM[11] = {0, 4, 4, 4, 4, 4, 4, 4, 4, 8, 4};
static const int LAYER_COMP[11] = {0, 1, 1, 1, 6, 1, 1, 2, 1, 1, 2};
enum { L_OCC = 1, L_MEAN = 2, L_COUNT = 3, L_COV = 4, L_HIT = 5, L_MISS = 6,
       L_INTENS = 7, L_DHITS = 8, L_DDIST = 9, L_TSDF = 10 };

/* ------------------------------------------------------------------ */
/* arithmetic helpers                                                  */

/* RaySample.length = np.linalg.norm -> sqrt(ddot(v, v)); OpenBLAS 0.3.30
 * (Haswell kernel) accumulates with FMA: traversal.py:40-42. */
double orc_norm3(double x, double y, double z)
{
    return sqrt(fma(z, z, fma(y, y, x * x)));
}

/* float(a @ b) for 3-vectors (tsdf proj, reference.py:170): same ddot */
static double dot3(const double *a, const double *b)
{
    return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

/* CPython 3.12 math.hypot (vector_norm, Modules/mathmodule.c), used by
 * ndt.cholupdate3 (ndt.py:42). */
static double py_vector_norm2(double x0, double x1, double max)
{
    if (isinf(max)) return max;
    if (max == 0.0) return max;
    int max_e;
    frexp(max, &max_e);
    if (max_e < -1023) {
        return DBL_MIN * py_vector_norm2(x0 / DBL_MIN, x1 / DBL_MIN, max / DBL_MIN);
    }
    double scale = ldexp(1.0, -max_e);
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    double v[2] = {x0, x1};
    for (int i = 0; i < 2; i++) {
        double x = v[i] * scale;
        double hi = x * x, lo = fma(x, x, -hi);
        double s = csum + hi;
        double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    double h = sqrt(csum - 1.0 + (frac1 + frac2));
    {
        double hi = -h * h, lo = fma(-h, h, -hi);
        double s = csum + hi;
        double sl = (csum - s) + hi;
        csum = s;
        frac1 += lo;
        frac2 += sl;
    }
    double x = csum - 1.0 + (frac1 + frac2);
    h += x / (2.0 * h);
    return h / scale;
}

double orc_py_hypot(double a, double b)
{
    double x0 = fabs(a), x1 = fabs(b);
    double max = 0.0;
    if (x0 > max) max = x0;
    if (x1 > max) max = x1;
    if (isnan(a) || isnan(b)) return NAN;
    return py_vector_norm2(x0, x1, max);
}

/* _kernels.pyx:105-110 splitmix64 finalizer */
uint64_t orc_hash_mix(int64_t key)
{
    uint64_t h = (uint64_t)key + 0x9E3779B97F4A7C15ULL;
    h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ULL;
    h = (h ^ (h >> 27)) * 0x94D049BB133111EBULL;
    return h ^ (h >> 31);
}

/* keys.py:76-86 */
static int64_t pack_region(int64_t rx, int64_t ry, int64_t rz)
{
    const int64_t B = 1 << 20, M = (1 << 21) - 1;
    return (((rx + B) & M) << 42) | (((ry + B) & M) << 21) | ((rz + B) & M);
}

/* Python divmod for ints (reference.py:26-32, keys.py:41-47) */
static void divmod64(int64_t a, int64_t d, int64_t *q, int64_t *r)
{
    int64_t qq = a / d, rr = a % d;
    if (rr != 0 && ((rr < 0) != (d < 0))) { qq -= 1; rr += d; }
    *q = qq;
    *r = rr;
}

static float clamped_add(float l, float d32, float cmin, float cmax)
{
    /* reference.py:22-23: np.clip(buf[idx] + delta32, f32(cmin), f32(cmax)) */
    volatile float s = l + d32;
    float v = s;
    if (v < cmin) v = cmin;
    if (v > cmax) v = cmax;
    return v;
}

/* subvoxel.py:16-23 */
static uint32_t pack_mean(const double off[3])
{
    uint32_t packed = 0;
    for (int a = 0; a < 3; a++) {
        double f = floor(off[a] * 1024.0);
        int q;
        if (f < 0.0) q = 0;
        else if (f > 1023.0) q = 1023;
        else q = (int)f;
        packed |= (uint32_t)q << (10 * a);
    }
    return packed;
}

/* subvoxel.py:26-31 */
static void unpack_mean(uint32_t packed, double out[3])
{
    for (int a = 0; a < 3; a++)
        out[a] = ((double)((packed >> (10 * a)) & 1023u) + 0.5) / 1024.0;
}

/* subvoxel.py:34-49 */
static void update_packed_mean(uint32_t *packed, uint32_t *count, const double s[3])
{
    uint32_t n = *count;
    if (n >= 0xFFFFFFFFu) return;
    if (n == 0) {
        *packed = pack_mean(s);
        *count = 1;
        return;
    }
    double m[3];
    unpack_mean(*packed, m);
    double div = (double)n + 1.0;
    for (int a = 0; a < 3; a++) m[a] = m[a] + (s[a] - m[a]) / div;
    *packed = pack_mean(m);
    *count = n + 1;
}

/* ------------------------------------------------------------------ */
/* map (store.py:28-80): hash of packed region key -> region           */

typedef struct {
    int64_t rx, ry, rz;
    void *buf[11];
} orc_region;

struct orc_map {
    orc_config cfg;
    uint32_t layer_mask;
    int64_t vpr; /* voxels per region */
    orc_region *regions;
    int64_t nreg, capreg;
    int64_t *tkeys;
    int64_t *tvals;
    int64_t tcap;
};

static void table_insert(orc_map *m, int64_t key, int64_t idx)
{
    uint64_t mask = (uint64_t)m->tcap - 1;
    uint64_t h = orc_hash_mix(key) & mask;
    while (m->tkeys[h] != -1) h = (h + 1) & mask;
    m->tkeys[h] = key;
    m->tvals[h] = idx;
}

static int64_t table_find(const orc_map *m, int64_t key)
{
    uint64_t mask = (uint64_t)m->tcap - 1;
    uint64_t h = orc_hash_mix(key) & mask;
    while (m->tkeys[h] != -1) {
        if (m->tkeys[h] == key) return m->tvals[h];
        h = (h + 1) & mask;
    }
    return -1;
}

static void table_grow(orc_map *m)
{
    int64_t ncap = m->tcap ? m->tcap * 2 : 1024;
    free(m->tkeys);
    free(m->tvals);
    m->tcap = ncap;
    m->tkeys = (int64_t *)malloc(sizeof(int64_t) * ncap);
    m->tvals = (int64_t *)malloc(sizeof(int64_t) * ncap);
    for (int64_t i = 0; i < ncap; i++) m->tkeys[i] = -1;
    for (int64_t i = 0; i < m->nreg; i++)
        table_insert(m, pack_region(m->regions[i].rx, m->regions[i].ry, m->regions[i].rz), i);
}

orc_map *orc_map_create(const orc_config *cfg, uint32_t layer_mask)
{
    orc_map *m = (orc_map *)calloc(1, sizeof(orc_map));
    m->cfg = *cfg;
    m->layer_mask = layer_mask;
    m->vpr = (int64_t)cfg->region_dim * cfg->region_dim * cfg->region_dim;
    table_grow(m);
    return m;
}

void orc_map_destroy(orc_map *m)
{
    if (!m) return;
    for (int64_t i = 0; i < m->nreg; i++)
        for (int l = 1; l <= 10; l++) free(m->regions[i].buf[l]);
    free(m->regions);
    free(m->tkeys);
    free(m->tvals);
    free(m);
}

int64_t orc_map_region_count(const orc_map *m) { return m->nreg; }

int64_t orc_map_regions(const orc_map *m, int64_t *out, int64_t cap)
{
    int64_t n = m->nreg < cap ? m->nreg : cap;
    for (int64_t i = 0; i < n; i++) {
        out[3 * i] = m->regions[i].rx;
        out[3 * i + 1] = m->regions[i].ry;
        out[3 * i + 2] = m->regions[i].rz;
    }
    return n;
}

static orc_region *get_region(orc_map *m, int64_t rx, int64_t ry, int64_t rz, int create)
{
    int64_t key = pack_region(rx, ry, rz);
    int64_t idx = table_find(m, key);
    if (idx >= 0) return &m->regions[idx];
    if (!create) return NULL;
    if (m->nreg == m->capreg) {
        m->capreg = m->capreg ? m->capreg * 2 : 64;
        m->regions = (orc_region *)realloc(m->regions, sizeof(orc_region) * m->capreg);
    }
    orc_region *r = &m->regions[m->nreg];
    memset(r, 0, sizeof(*r));
    r->rx = rx;
    r->ry = ry;
    r->rz = rz;
    for (int l = 1; l <= 10; l++)
        if (m->layer_mask & (1u << l))
            r->buf[l] = calloc((size_t)m->vpr * LAYER_COMP[l], LAYER_ELEM[l]);
    m->nreg++;
    if (m->nreg * 2 > m->tcap) table_grow(m);
    else table_insert(m, key, m->nreg - 1);
    return r;
}

void *orc_map_layer(orc_map *m, int64_t rx, int64_t ry, int64_t rz, int32_t layer_id)
{
    orc_region *r = get_region(m, rx, ry, rz, 0);
    if (!r || layer_id < 1 || layer_id > 10) return NULL;
    return r->buf[layer_id];
}

void *orc_map_layer_create(orc_map *m, int64_t rx, int64_t ry, int64_t rz, int32_t layer_id)
{
    orc_region *r = get_region(m, rx, ry, rz, 1);
    if (layer_id < 1 || layer_id > 10) return NULL;
    return r->buf[layer_id];
}

/* reference.py:26-32 */
static orc_region *region_and_local(orc_map *m, const int64_t g[3], int64_t *li)
{
    int64_t d = m->cfg.region_dim, r[3], l[3];
    for (int a = 0; a < 3; a++) divmod64(g[a], d, &r[a], &l[a]);
    *li = l[0] + d * (l[1] + d * l[2]);
    return get_region(m, r[0], r[1], r[2], 1);
}

/* ------------------------------------------------------------------ */
/* traversal._walk_grid (traversal.py:52-111)                          */

int64_t orc_walk(double ox, double oy, double oz, double ex, double ey, double ez,
                 double cell, int64_t *coords, double *t0, double *t1, int64_t cap)
{
    double o[3] = {ox, oy, oz};
    double v[3] = {ex - ox, ey - oy, ez - oz};
    int64_t cur[3] = {(int64_t)floor(ox / cell), (int64_t)floor(oy / cell),
                      (int64_t)floor(oz / cell)};
    int64_t last[3] = {(int64_t)floor(ex / cell), (int64_t)floor(ey / cell),
                       (int64_t)floor(ez / cell)};
    int64_t step[3] = {0, 0, 0};
    double tmax[3] = {INFINITY, INFINITY, INFINITY};
    double tdel[3] = {INFINITY, INFINITY, INFINITY};
    for (int a = 0; a < 3; a++) {
        if (v[a] > 0) {
            step[a] = 1;
            tmax[a] = ((double)(cur[a] + 1) * cell - o[a]) / v[a];
            tdel[a] = cell / v[a];
        } else if (v[a] < 0) {
            step[a] = -1;
            tmax[a] = ((double)cur[a] * cell - o[a]) / v[a];
            tdel[a] = -cell / v[a];
        }
    }
    int64_t remaining = 0;
    for (int a = 0; a < 3; a++) remaining += llabs(cur[a] - last[a]);
    double tprev = 0.0;
    int64_t n = 0;
    for (;;) {
        if (n >= cap) return -1;
        if (cur[0] == last[0] && cur[1] == last[1] && cur[2] == last[2]) {
            memcpy(&coords[3 * n], cur, sizeof(cur));
            t0[n] = tprev;
            t1[n] = 1.0;
            return n + 1;
        }
        if (remaining <= 0) {
            memcpy(&coords[3 * n], last, sizeof(last));
            t0[n] = tprev;
            t1[n] = 1.0;
            return n + 1;
        }
        int axis = 0;
        if (tmax[1] < tmax[axis]) axis = 1;
        if (tmax[2] < tmax[axis]) axis = 2;
        double tn = tmax[axis];
        if (tprev > tn) tn = tprev;  /* max(t_max, t_prev): returns t_max unless t_prev larger */
        if (tn > 1.0) tn = 1.0;      /* min(., 1.0) */
        memcpy(&coords[3 * n], cur, sizeof(cur));
        t0[n] = tprev;
        t1[n] = tn;
        cur[axis] += step[axis];
        tmax[axis] += tdel[axis];
        tprev = tn;
        n++;
        remaining--;
    }
}

/* growable walk scratch */
typedef struct {
    int64_t *c;
    double *t0, *t1;
    int64_t cap;
} walkbuf;

static int64_t walk_bound(const double o[3], const double e[3], double cell)
{
    int64_t b = 0;
    for (int a = 0; a < 3; a++)
        b += llabs((int64_t)floor(e[a] / cell) - (int64_t)floor(o[a] / cell));
    return b + 2;
}

static int64_t walk(walkbuf *w, const double o[3], const double e[3], double cell)
{
    int64_t need = walk_bound(o, e, cell);
    if (need > w->cap) {
        w->cap = need * 2;
        w->c = (int64_t *)realloc(w->c, sizeof(int64_t) * 3 * w->cap);
        w->t0 = (double *)realloc(w->t0, sizeof(double) * w->cap);
        w->t1 = (double *)realloc(w->t1, sizeof(double) * w->cap);
    }
    return orc_walk(o[0], o[1], o[2], e[0], e[1], e[2], cell, w->c, w->t0, w->t1, w->cap);
}

static void walkbuf_free(walkbuf *w)
{
    free(w->c);
    free(w->t0);
    free(w->t1);
}

/* ------------------------------------------------------------------ */
/* preprocessing: engine._preprocess + clip_ray + segment_ray          */

typedef struct {
    double o[3], e[3];
    uint8_t has;
    float intensity;
    int64_t ray;
} segment_t;

static double seg_len(const double o[3], const double e[3])
{
    return orc_norm3(e[0] - o[0], e[1] - o[1], e[2] - o[2]);
}

/* emits into out (may be NULL to count); returns #segments for this ray,
 * or 0 if the ray is dropped (length == 0) */
static int64_t preprocess_ray(const orc_config *cfg, const double o_in[3], const double e_in[3],
                              uint8_t has, float intensity, int64_t ray, int segment,
                              segment_t *out)
{
    double o[3] = {o_in[0], o_in[1], o_in[2]};
    double e[3] = {e_in[0], e_in[1], e_in[2]};
    double L = seg_len(o, e);
    if (L == 0.0) return 0;
    /* clip_ray, traversal.py:140-150 */
    if (L > cfg->max_ray_range) {
        double d[3];
        for (int a = 0; a < 3; a++) d[a] = (e[a] - o[a]) / L;
        for (int a = 0; a < 3; a++) e[a] = o[a] + d[a] * cfg->max_ray_range;
        has = 0;
        L = seg_len(o, e);
    }
    if (!segment || L <= cfg->segment_length) {
        if (out) {
            memcpy(out[0].o, o, sizeof(o));
            memcpy(out[0].e, e, sizeof(e));
            out[0].has = has;
            out[0].intensity = intensity;
            out[0].ray = ray;
        }
        return 1;
    }
    /* segment_ray, traversal.py:153-178 */
    double seg = cfg->segment_length;
    int64_t count = (int64_t)ceil(L / seg);
    double d[3];
    for (int a = 0; a < 3; a++) d[a] = (e[a] - o[a]) / L;
    if (out) {
        for (int64_t i = 0; i < count; i++) {
            double t0 = (double)i * seg;
            double t1 = (double)(i + 1) * seg;
            if (L < t1) t1 = L; /* min((i+1)*seg, length) */
            int is_last = i == count - 1;
            for (int a = 0; a < 3; a++) {
                out[i].o[a] = o[a] + d[a] * t0;
                out[i].e[a] = is_last ? e[a] : o[a] + d[a] * t1;
            }
            out[i].has = is_last ? has : 0;
            out[i].intensity = intensity;
            out[i].ray = ray;
        }
    }
    return count;
}

int64_t orc_preprocess(const orc_config *cfg, const double *origins, const double *ends,
                       const uint8_t *has_sample, int64_t n, int32_t segment,
                       double *seg_o, double *seg_e, uint8_t *seg_has, int64_t *seg_ray,
                       int64_t cap, int64_t *processed_out)
{
    int64_t ns = 0, processed = 0;
    segment_t tmp[64];
    for (int64_t i = 0; i < n; i++) {
        int64_t k = preprocess_ray(cfg, &origins[3 * i], &ends[3 * i], has_sample[i], 0.0f, i,
                                   segment, NULL);
        if (k == 0) continue;
        processed++;
        if (k > 64 || ns + k > cap) return -1;
        preprocess_ray(cfg, &origins[3 * i], &ends[3 * i], has_sample[i], 0.0f, i, segment, tmp);
        for (int64_t j = 0; j < k; j++, ns++) {
            memcpy(&seg_o[3 * ns], tmp[j].o, 24);
            memcpy(&seg_e[3 * ns], tmp[j].e, 24);
            seg_has[ns] = tmp[j].has;
            seg_ray[ns] = tmp[j].ray;
        }
    }
    if (processed_out) *processed_out = processed;
    return ns;
}

/* ------------------------------------------------------------------ */
/* integrators (reference.py)                                          */

/* reference.py:35-64 */
static int64_t integrate_occupancy_segment(orc_map *m, walkbuf *w, const segment_t *s, int decay)
{
    const orc_config *cfg = &m->cfg;
    int64_t n = walk(w, s->o, s->e, cfg->voxel_size);
    float hit32 = (float)cfg->hit_delta, miss32 = (float)cfg->miss_delta;
    float cmin = (float)cfg->clamp_min, cmax = (float)cfg->clamp_max;
    double length = seg_len(s->o, s->e);
    for (int64_t i = 0; i < n; i++) {
        int64_t li;
        const int64_t *g = &w->c[3 * i];
        orc_region *r = region_and_local(m, g, &li);
        float *occ = (float *)r->buf[L_OCC];
        int sample_hit = s->has && i == n - 1;
        if (sample_hit) {
            occ[li] = clamped_add(occ[li], hit32, cmin, cmax);
            if (r->buf[L_MEAN]) {
                double off[3];
                for (int a = 0; a < 3; a++) off[a] = s->e[a] / cfg->voxel_size - (double)g[a];
                update_packed_mean(&((uint32_t *)r->buf[L_MEAN])[li],
                                   &((uint32_t *)r->buf[L_COUNT])[li], off);
            }
        } else {
            occ[li] = clamped_add(occ[li], miss32, cmin, cmax);
        }
        if (decay) {
            ((double *)r->buf[L_DDIST])[li] += (w->t1[i] - w->t0[i]) * length;
            if (sample_hit) ((uint32_t *)r->buf[L_DHITS])[li] += 1;
        }
    }
    return n;
}

/* _kernels.pyx:473-525: exp(-0.5 m^2) via adjugate inverse (deliberate
 * deviation from ndt.py:73-95's numpy.linalg.inv; tolerance-graded) */
static double gaussian_miss_weight(const double mu[3], const float cov6[6], double sigma2,
                                   const double o[3], const double v[3], double t0, double t1)
{
    double s0 = cov6[0], s1 = cov6[1], s2 = cov6[2], s3 = cov6[3], s4 = cov6[4], s5 = cov6[5];
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

/* reference.py:97-104 */
static void reset_voxel(orc_region *r, int64_t li, int tm)
{
    ((uint32_t *)r->buf[L_COUNT])[li] = 0;
    ((uint32_t *)r->buf[L_MEAN])[li] = 0;
    memset(&((float *)r->buf[L_COV])[li * 6], 0, 6 * sizeof(float));
    if (tm) {
        ((uint32_t *)r->buf[L_HIT])[li] = 0;
        ((uint32_t *)r->buf[L_MISS])[li] = 0;
        memset(&((float *)r->buf[L_INTENS])[li * 2], 0, 2 * sizeof(float));
    }
}

/* reference.py:67-94 */
static int64_t ndt_phase1_segment(orc_map *m, walkbuf *w, const segment_t *s, int tm)
{
    const orc_config *cfg = &m->cfg;
    int64_t n = walk(w, s->o, s->e, cfg->voxel_size);
    float cmin = (float)cfg->clamp_min, cmax = (float)cfg->clamp_max;
    float fthresh = (float)cfg->ndt_reset_threshold;
    double sigma2 = cfg->ndt_sensor_noise * cfg->ndt_sensor_noise;
    double v[3] = {s->e[0] - s->o[0], s->e[1] - s->o[1], s->e[2] - s->o[2]};
    for (int64_t i = 0; i < n; i++) {
        if (s->has && i == n - 1) continue;
        int64_t li;
        const int64_t *g = &w->c[3 * i];
        orc_region *r = region_and_local(m, g, &li);
        float *occ = (float *)r->buf[L_OCC];
        uint32_t *cnt = (uint32_t *)r->buf[L_COUNT];
        uint32_t ns = cnt[li];
        double gw = 1.0;
        if (ns >= 3) {
            double off[3], mu[3];
            unpack_mean(((uint32_t *)r->buf[L_MEAN])[li], off);
            for (int a = 0; a < 3; a++) mu[a] = ((double)g[a] + off[a]) * cfg->voxel_size;
            gw = gaussian_miss_weight(mu, &((float *)r->buf[L_COV])[li * 6], sigma2, s->o, v,
                                      w->t0[i], w->t1[i]);
        }
        occ[li] = clamped_add(occ[li], (float)(gw * cfg->miss_delta), cmin, cmax);
        if (tm && (ns < 3 || gw >= cfg->ndt_miss_likelihood_threshold))
            ((uint32_t *)r->buf[L_MISS])[li] += 1;
        if (occ[li] < fthresh && cnt[li] > 0) reset_voxel(r, li, tm);
    }
    return n;
}

/* ndt.py:37-52 */
static void cholupdate3(double L[3][3], double x[3])
{
    for (int k = 0; k < 3; k++) {
        double r = orc_py_hypot(L[k][k], x[k]);
        if (r == 0.0) continue;
        double c = L[k][k] / r, s = x[k] / r;
        L[k][k] = r;
        for (int i = k + 1; i < 3; i++) {
            double lik = L[i][k];
            L[i][k] = c * lik + s * x[i];
            x[i] = c * x[i] - s * lik;
        }
    }
}

/* ndt.py:55-70 */
static void update_gaussian(uint64_t *n, double mu[3], double S[3][3], const double x[3])
{
    if (*n == 0) {
        *n = 1;
        for (int a = 0; a < 3; a++) mu[a] = x[a];
        memset(S, 0, sizeof(double) * 9);
        return;
    }
    uint64_t nn = *n + 1;
    double d[3];
    for (int a = 0; a < 3; a++) d[a] = x[a] - mu[a];
    for (int a = 0; a < 3; a++) mu[a] = mu[a] + d[a] / (double)nn;
    double sq = sqrt((double)*n);
    double L[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) L[i][j] = S[i][j] * sq;
    double f = sqrt((double)*n / (double)nn);
    double xx[3];
    for (int a = 0; a < 3; a++) xx[a] = d[a] * f;
    cholupdate3(L, xx);
    double sn = sqrt((double)nn);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) S[i][j] = L[i][j] / sn;
    *n = nn;
}

typedef struct {
    int64_t g[3];
    int64_t order;
    double pos[3];
    float intensity;
} ndt_sample;

static int cmp_sample(const void *pa, const void *pb)
{
    const ndt_sample *a = (const ndt_sample *)pa, *b = (const ndt_sample *)pb;
    for (int k = 0; k < 3; k++) {
        if (a->g[k] < b->g[k]) return -1;
        if (a->g[k] > b->g[k]) return 1;
    }
    return (a->order > b->order) - (a->order < b->order);
}

/* reference.py:107-150 (apply_ndt_hits) over sample_buckets (178-186) */
static void apply_ndt_hits(orc_map *m, ndt_sample *smp, int64_t ns, int tm)
{
    const orc_config *cfg = &m->cfg;
    float hit32 = (float)cfg->hit_delta;
    float cmin = (float)cfg->clamp_min, cmax = (float)cfg->clamp_max;
    qsort(smp, (size_t)ns, sizeof(ndt_sample), cmp_sample);
    int64_t i = 0;
    while (i < ns) {
        int64_t j = i;
        while (j < ns && !memcmp(smp[j].g, smp[i].g, sizeof(smp[i].g))) j++;
        int64_t li;
        orc_region *r = region_and_local(m, smp[i].g, &li);
        float *occ = (float *)r->buf[L_OCC];
        uint32_t *mb = (uint32_t *)r->buf[L_MEAN];
        uint32_t *cb = (uint32_t *)r->buf[L_COUNT];
        float *cov = (float *)r->buf[L_COV];
        uint64_t n = cb[li];
        double mu[3] = {0, 0, 0};
        if (n > 0) {
            double off[3];
            unpack_mean(mb[li], off);
            for (int a = 0; a < 3; a++) mu[a] = ((double)smp[i].g[a] + off[a]) * cfg->voxel_size;
        }
        double S[3][3] = {{cov[li * 6], 0, 0},
                          {cov[li * 6 + 1], cov[li * 6 + 2], 0},
                          {cov[li * 6 + 3], cov[li * 6 + 4], cov[li * 6 + 5]}};
        for (int64_t k = i; k < j; k++) {
            occ[li] = clamped_add(occ[li], hit32, cmin, cmax);
            if (tm) {
                float *ib = (float *)r->buf[L_INTENS];
                /* ndt.py:98-106 */
                double val = smp[k].intensity;
                double mean = ib[li * 2], m2 = ib[li * 2 + 1];
                double nn = (double)(n + 1);
                double d = val - mean;
                double mean_new = mean + d / nn;
                double m2_new = m2 + d * (val - mean_new);
                ib[li * 2] = (float)mean_new;
                ib[li * 2 + 1] = (float)m2_new;
            }
            update_gaussian(&n, mu, S, smp[k].pos);
        }
        if (tm) ((uint32_t *)r->buf[L_HIT])[li] += (uint32_t)(j - i);
        cb[li] = n > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)n;
        double frac[3];
        for (int a = 0; a < 3; a++) {
            double f = mu[a] / cfg->voxel_size - (double)smp[i].g[a];
            const double hi = 1.0 - 1.0 / 2048.0;
            if (f < 0.0) f = 0.0;
            if (f > hi) f = hi;
            frac[a] = f;
        }
        mb[li] = pack_mean(frac);
        cov[li * 6] = (float)S[0][0];
        cov[li * 6 + 1] = (float)S[1][0];
        cov[li * 6 + 2] = (float)S[1][1];
        cov[li * 6 + 3] = (float)S[2][0];
        cov[li * 6 + 4] = (float)S[2][1];
        cov[li * 6 + 5] = (float)S[2][2];
        i = j;
    }
}

/* reference.py:153-175 */
static int64_t integrate_tsdf_ray(orc_map *m, walkbuf *w, const segment_t *s)
{
    const orc_config *cfg = &m->cfg;
    double length = seg_len(s->o, s->e);
    if (!s->has || length == 0.0) return 0;
    double d[3], p0[3], p1[3];
    for (int a = 0; a < 3; a++) d[a] = (s->e[a] - s->o[a]) / length;
    double tau = cfg->tsdf_truncation;
    double ts = length - tau;
    if (!(ts > 0.0)) ts = 0.0; /* max(0.0, length - tau) */
    double te = length + tau;
    for (int a = 0; a < 3; a++) {
        p0[a] = s->o[a] + d[a] * ts;
        p1[a] = s->o[a] + d[a] * te;
    }
    int64_t n = walk(w, p0, p1, cfg->voxel_size);
    for (int64_t i = 0; i < n; i++) {
        int64_t li;
        const int64_t *g = &w->c[3 * i];
        orc_region *r = region_and_local(m, g, &li);
        float *buf = (float *)r->buf[L_TSDF];
        double c[3], cmo[3];
        for (int a = 0; a < 3; a++) {
            c[a] = ((double)g[a] + 0.5) * cfg->voxel_size;
            cmo[a] = c[a] - s->o[a];
        }
        double proj = dot3(cmo, d);
        double dv = length - proj;
        if (dv < -tau) dv = -tau;
        if (dv > tau) dv = tau;
        double wgt = buf[li * 2 + 1];
        double nd = (wgt * (double)buf[li * 2] + dv) / (wgt + 1.0);
        double nw = wgt + 1.0;
        if (nw > cfg->tsdf_max_weight) nw = cfg->tsdf_max_weight;
        buf[li * 2] = (float)nd;
        buf[li * 2 + 1] = (float)nw;
    }
    return n;
}

/* engine.prefetch_regions (engine.py:99-118) */
static int64_t prefetch_regions(orc_map *m, walkbuf *w, const segment_t *segs, int64_t ns,
                                double extra)
{
    const orc_config *cfg = &m->cfg;
    double rsize = (double)cfg->region_dim * cfg->voxel_size;
    int64_t before = m->nreg;
    /* touched = set(); count distinct: use a scratch map of keys */
    int64_t tcap = 1024;
    while (tcap < 4 * ns + 1024) tcap <<= 1;
    int64_t *seen = (int64_t *)malloc(sizeof(int64_t) * tcap);
    for (int64_t i = 0; i < tcap; i++) seen[i] = -1;
    int64_t touched = 0;
    int64_t (*keys)[3] = NULL;
    int64_t kcap = 0;
    for (int64_t k = 0; k < ns; k++) {
        const segment_t *s = &segs[k];
        double pe[3] = {s->e[0], s->e[1], s->e[2]};
        double L = seg_len(s->o, s->e);
        if (extra > 0.0 && s->has && L > 0.0) {
            for (int a = 0; a < 3; a++) {
                double d = (s->e[a] - s->o[a]) / L;
                pe[a] = s->e[a] + d * extra;
            }
        }
        int64_t n = walk(w, s->o, pe, rsize);
        for (int64_t i = 0; i < n; i++) {
            const int64_t *rc = &w->c[3 * i];
            int64_t key = pack_region(rc[0], rc[1], rc[2]);
            uint64_t mask = (uint64_t)tcap - 1, h = orc_hash_mix(key) & mask;
            int found = 0;
            while (seen[h] != -1) {
                if (seen[h] == key) { found = 1; break; }
                h = (h + 1) & mask;
            }
            if (found) continue;
            seen[h] = key;
            if (touched == kcap) {
                kcap = kcap ? kcap * 2 : 256;
                keys = realloc(keys, sizeof(*keys) * kcap);
            }
            memcpy(keys[touched], rc, 24);
            touched++;
            if (touched * 2 > tcap) {
                /* rehash */
                int64_t ncap = tcap * 2;
                int64_t *ns2 = (int64_t *)malloc(sizeof(int64_t) * ncap);
                for (int64_t q = 0; q < ncap; q++) ns2[q] = -1;
                for (int64_t q = 0; q < touched; q++) {
                    int64_t kk = pack_region(keys[q][0], keys[q][1], keys[q][2]);
                    uint64_t mm = (uint64_t)ncap - 1, hh = orc_hash_mix(kk) & mm;
                    while (ns2[hh] != -1) hh = (hh + 1) & mm;
                    ns2[hh] = kk;
                }
                free(seen);
                seen = ns2;
                tcap = ncap;
            }
        }
    }
    for (int64_t q = 0; q < touched; q++) get_region(m, keys[q][0], keys[q][1], keys[q][2], 1);
    (void)before;
    free(seen);
    free(keys);
    return touched;
}

int64_t orc_prefetch_regions(const orc_config *cfg, const double *seg_o, const double *seg_e,
                             const uint8_t *seg_has, int64_t n, double extra_reach,
                             int64_t *coords_out, int64_t cap)
{
    orc_map *m = orc_map_create(cfg, 0);
    segment_t *segs = (segment_t *)malloc(sizeof(segment_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) {
        memcpy(segs[i].o, &seg_o[3 * i], 24);
        memcpy(segs[i].e, &seg_e[3 * i], 24);
        segs[i].has = seg_has[i];
    }
    walkbuf w = {0};
    prefetch_regions(m, &w, segs, n, extra_reach);
    walkbuf_free(&w);
    free(segs);
    int64_t k = m->nreg;
    if (k > cap) {
        orc_map_destroy(m);
        return -1;
    }
    orc_map_regions(m, coords_out, k);
    orc_map_destroy(m);
    return k;
}

int orc_integrate(orc_map *m, const double *origins, const double *ends,
                  const uint8_t *has_sample, const float *intensity, int64_t n, int32_t mode,
                  int64_t *stats)
{
    const orc_config *cfg = &m->cfg;
    memset(stats, 0, sizeof(int64_t) * ORC_NSTATS);
    stats[0] = n;
    int segment = mode != ORC_MODE_TSDF;
    segment_t *segs = NULL;
    int64_t ns = 0, scap = 0, processed = 0;
    segment_t tmp[64];
    for (int64_t i = 0; i < n; i++) {
        float inten = intensity ? intensity[i] : 0.0f;
        int64_t k = preprocess_ray(cfg, &origins[3 * i], &ends[3 * i], has_sample[i], inten, i,
                                   segment, NULL);
        if (k == 0) continue;
        if (k > 64) return -1;
        processed++;
        preprocess_ray(cfg, &origins[3 * i], &ends[3 * i], has_sample[i], inten, i, segment, tmp);
        if (ns + k > scap) {
            scap = (ns + k) * 2;
            segs = (segment_t *)realloc(segs, sizeof(segment_t) * scap);
        }
        memcpy(&segs[ns], tmp, sizeof(segment_t) * k);
        ns += k;
    }
    stats[1] = processed;
    stats[2] = ns;
    if (ns == 0) {
        free(segs);
        return 0;
    }
    walkbuf w = {0};
    double extra = mode == ORC_MODE_TSDF ? cfg->tsdf_truncation : 0.0;
    stats[7] = prefetch_regions(m, &w, segs, ns, extra);
    int64_t visits = 0;
    if (mode == ORC_MODE_OCCUPANCY || mode == ORC_MODE_DECAY) {
        for (int64_t k = 0; k < ns; k++)
            visits += integrate_occupancy_segment(m, &w, &segs[k], mode == ORC_MODE_DECAY);
    } else if (mode == ORC_MODE_NDT_OM || mode == ORC_MODE_NDT_TM) {
        int tm = mode == ORC_MODE_NDT_TM;
        for (int64_t k = 0; k < ns; k++) visits += ndt_phase1_segment(m, &w, &segs[k], tm);
        int64_t nsmp = 0;
        for (int64_t k = 0; k < ns; k++) nsmp += segs[k].has ? 1 : 0;
        ndt_sample *smp = (ndt_sample *)malloc(sizeof(ndt_sample) * (nsmp ? nsmp : 1));
        int64_t q = 0;
        for (int64_t k = 0; k < ns; k++) {
            if (!segs[k].has) continue;
            for (int a = 0; a < 3; a++) {
                smp[q].g[a] = (int64_t)floor(segs[k].e[a] / cfg->voxel_size);
                smp[q].pos[a] = segs[k].e[a];
            }
            smp[q].order = k;
            smp[q].intensity = segs[k].intensity;
            q++;
        }
        apply_ndt_hits(m, smp, nsmp, tm);
        free(smp);
    } else if (mode == ORC_MODE_TSDF) {
        for (int64_t k = 0; k < ns; k++) visits += integrate_tsdf_ray(m, &w, &segs[k]);
    } else if (mode == ORC_MODE_COUNTS) {
        /* the visits integrate_occupancy_segment would make, counted per voxel:
         * the bounds of the CAS order envelope (tests/test_gpu_parity.py) */
        for (int64_t k = 0; k < ns; k++) {
            int64_t nv = walk(&w, segs[k].o, segs[k].e, cfg->voxel_size);
            for (int64_t i = 0; i < nv; i++) {
                int64_t li;
                orc_region *r = region_and_local(m, &w.c[3 * i], &li);
                if (segs[k].has && i == nv - 1) ((uint32_t *)r->buf[L_HIT])[li] += 1;
                else ((uint32_t *)r->buf[L_MISS])[li] += 1;
            }
            visits += nv;
        }
    } else {
        walkbuf_free(&w);
        free(segs);
        return -2;
    }
    stats[3] = visits;
    walkbuf_free(&w);
    free(segs);
    return 0;
}
