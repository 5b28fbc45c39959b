// vm_shard.cuh -- region-sharded integration across GPUs.
//
// G maps, one per GPU.  Map r owns the regions with region_owner(key) == r
// (2 x 2 x 2 region blocks hashed over the ranks) and walks the slice
// [r*N/G, (r+1)*N/G) of every batch; every rank holds the whole batch (the
// in-order fold needs any ray's end point).  Regions a rank's rays reach but
// another rank owns are "ghost" regions in its map: scratch only.
//
// Per batch (vm_shard_* in vm_runtime.cu, driven by sharded.py):
//   begin    discover the slice; list the new ghost regions (creation
//            requests for their owners) and the slice's new sample voxels
//   -- exchange A: requests all-to-all, sample voxels all-gather --
//   prepare  create requested regions, stamp every rank's sample voxels
//            into the local regions that hold them (owned or ghost)
//   walk     the deterministic walk of the slice
//   export   ghost payload per owner: order-free miss counts of ghost voxels
//            and the order-keyed records of ghost sample voxels
//   -- exchange B: payload all-to-all --
//   import   counts into the owner's scratch, records into its record buffer
//   finish   drop ghost state; resolve, sort, fold as on one GPU
//
// Items are 16 bytes: region key, then local index | kind << 31, then the
// miss count or the record's ray order | hit.
#pragma once

#include "vm_kernels.cuh"

namespace vm {

struct ShardItem {
    long long rkey;
    unsigned li_kind;  // li | kind << 31 (0: miss count, 1: record)
    unsigned val;
};
static_assert(sizeof(ShardItem) == 16, "ShardItem layout");

// begin: creation requests for the new ghost regions [s0, s1) and the
// slice's new sample voxels as (region key, li) pairs
__global__ void k_shard_lists(const __grid_constant__ DevMap m, int s0, int s1, long long *req,
                              unsigned long long *nreq, unsigned long long req_cap,
                              long long *marks, unsigned long long n_marks) {
    // req: world segments of req_cap keys, nreq[d] = requests for rank d
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long s = s0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; s < s1; s += stride) {
        const long long key = m.slot_keys[s];
        const int d = region_owner(key, m.shard_world);
        if (d == m.shard_rank) continue;
        const unsigned long long k = atomicAdd(nreq + d, 1ULL);
        if (k < req_cap) req[(unsigned long long)d * req_cap + k] = key;
    }
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)n_marks;
         i += stride) {
        const int2 sl = m.marked[i];
        marks[2 * i] = m.slot_keys[sl.x];
        marks[2 * i + 1] = sl.y;
    }
}

// prepare: regions other ranks created in this map's partition, then the
// sample-voxel stamps of every rank
__global__ void k_shard_prepare(const __grid_constant__ DevMap m, const long long *req, long long nreq) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nreq; i += stride)
        region_slot(m, req[i]);
}

__global__ void k_shard_stamp(const __grid_constant__ DevMap m, const long long *marks, long long nmarks) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nmarks; i += stride) {
        const int s = region_find(m, marks[2 * i]);
        if (s < 0 || s >= m.cap) continue;
        const int li = (int)marks[2 * i + 1];
        atomicOr(reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]) + (size_t)s * m.vpr + li, MARK_FLAG);
        // the walk's brick summary (see k_discover)
        atomicOr(m.bmask + s, m.brick_shift >= 0 ? 1u << brick_of(li, m.bsh) : 0xFFFFFFFFu);
    }
}

// ghost slot test (slot key owned by another rank)
__device__ __forceinline__ bool is_ghost(const DevMap &m, int slot) {
    return region_owner(m.slot_keys[slot], m.shard_world) != m.shard_rank;
}

// per-destination append into fixed segments of `cap_per` items
__device__ __forceinline__ void shard_emit(ShardItem *out, unsigned long long *cnt,
                                          unsigned long long cap_per, int dest, const ShardItem &it) {
    const unsigned long long k = atomicAdd(cnt + dest, 1ULL);
    if (k < cap_per) out[(unsigned long long)dest * cap_per + k] = it;
}

// export 1: records of ghost voxels
__global__ void k_shard_export_rec(const __grid_constant__ DevMap m, const unsigned long long *rec,
                                   long long R, ShardItem *out, unsigned long long *cnt,
                                   unsigned long long cap_per) {
    const unsigned long long omask = (1ULL << m.order_bits) - 1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = rec[i];
        const unsigned vid = (unsigned)(k >> m.order_bits);
        const int slot = (int)(vid / (unsigned)m.vpr);
        if (!is_ghost(m, slot)) continue;
        const long long key = m.slot_keys[slot];
        ShardItem it{key, (vid % (unsigned)m.vpr) | 0x80000000u, (unsigned)(k & omask)};
        shard_emit(out, cnt, cap_per, region_owner(key, m.shard_world), it);
    }
}

// slot of work item t over the regions the walk touched (grid cells, then
// touched-list regions outside the grid, like k_resolve); -1 to skip
__device__ __forceinline__ int touched_slot(const DevMap &m, unsigned long long t, bool grid,
                                            long long gx, long long gy, long long gz,
                                            unsigned long long ncell) {
    const int *b = m.rbox;
    if (t < ncell) {
        const int slot = m.rgrid[t];
        return slot >= 0 && slot < m.cap ? slot : -1;
    }
    const int slot = m.touched[t - ncell];
    if (grid) {
        int r[3];
        unpack_region(m.slot_keys[slot], r);
        const long long ux = r[0] - b[0], uy = r[1] - b[1], uz = r[2] - b[2];
        if (ux >= 0 && ux < gx && uy >= 0 && uy < gy && uz >= 0 && uz < gz &&
            m.rgrid[ux + gx * (uy + gy * uz)] == slot)
            return -1;  // covered by its grid cell
    }
    return slot;
}

#define VM_TOUCHED_REGIONS(BODY)                                                              \
    {                                                                                         \
        unsigned long long nt_ = *((volatile unsigned long long *)(m.stats + S_WALK_TOUCHED)); \
        if (nt_ > (unsigned long long)m.touched_cap) nt_ = m.touched_cap;                      \
        const bool grid_ = *((volatile unsigned long long *)(m.stats + S_RGRID)) != 0;          \
        const int *b_ = m.rbox;                                                               \
        const long long gx_ = grid_ ? b_[3] - b_[0] + 1 : 0, gy_ = grid_ ? b_[4] - b_[1] + 1 : 0, \
                        gz_ = grid_ ? b_[5] - b_[2] + 1 : 0;                                  \
        const unsigned long long ncell_ = (unsigned long long)(gx_ * gy_ * gz_);               \
        for (unsigned long long t_ = blockIdx.x; t_ < ncell_ + nt_; t_ += gridDim.x) {          \
            const int slot = touched_slot(m, t_, grid_, gx_, gy_, gz_, ncell_);               \
            if (slot < 0 || !is_ghost(m, slot)) continue;                                     \
            BODY                                                                              \
        }                                                                                     \
    }

// export 2: order-free miss counts of the ghost regions the walk touched
__global__ void __launch_bounds__(BLOCK) k_shard_export_cnt(const __grid_constant__ DevMap m,
                                                             ShardItem *out, unsigned long long *cnt,
                                                             unsigned long long cap_per) {
    const unsigned *scr0 = reinterpret_cast<const unsigned *>(m.slab[L_SCRATCH]);
    VM_TOUCHED_REGIONS({
        const long long key = m.slot_keys[slot];
        const int dest = region_owner(key, m.shard_world);
        const unsigned *scr = scr0 + (size_t)slot * m.vpr;
        for (int li = threadIdx.x; li < m.vpr; li += blockDim.x) {
            const unsigned c = scr[li];
            if (c == 0u || (c & MARK_FLAG)) continue;  // MARK'ed: its visits are records
            shard_emit(out, cnt, cap_per, dest, ShardItem{key, (unsigned)li, c});
        }
    })
}

// after a successful export: zero the touched ghost scratch, drop the ghost
// stamps of this batch and the ghost records
__global__ void __launch_bounds__(BLOCK) k_shard_clear(const __grid_constant__ DevMap m,
                                                        unsigned long long *rec, long long R,
                                                        unsigned long long invalid_key,
                                                        const long long *marks, long long nmarks) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < R;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned vid = (unsigned)(rec[i] >> m.order_bits);
        if (is_ghost(m, (int)(vid / (unsigned)m.vpr))) rec[i] = invalid_key;
    }
    unsigned *scr0 = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nmarks;
         i += (long long)gridDim.x * blockDim.x) {
        const int s = region_find(m, marks[2 * i]);
        if (s >= 0 && s < m.cap && is_ghost(m, s)) {
            scr0[(size_t)s * m.vpr + marks[2 * i + 1]] = 0u;
            m.bmask[s] = 0u;
        }
    }
    VM_TOUCHED_REGIONS({
        unsigned *scr = scr0 + (size_t)slot * m.vpr;
        for (int li = threadIdx.x; li < m.vpr; li += blockDim.x)
            if (scr[li]) scr[li] = 0u;
    })
}

// import pass 1: make sure every region the items address exists (a ghost
// region another rank's walk entered may be new here); the host grows the
// pool to the cursor before pass 2
__global__ void k_shard_import_regions(const __grid_constant__ DevMap m, const ShardItem *in,
                                       long long n) {
    long long prev = -1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long key = in[i].rkey;
        if (key != prev) region_slot(m, key);
        prev = key;
    }
}

// import pass 2: counts into the owner's scratch, records appended
__global__ void k_shard_import(const __grid_constant__ DevMap m, const ShardItem *in, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const ShardItem it = in[i];
        const int s = region_find(m, it.rkey);
        if (s < 0 || s >= m.cap) continue;
        if (stamp_epoch(m.slot_touch + s, m.epoch)) {
            const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
            if (t < (unsigned long long)m.touched_cap) m.touched[t] = s;
        }
        const unsigned li = it.li_kind & 0x7FFFFFFFu;
        const unsigned long long vid = (unsigned long long)s * m.vpr + li;
        if (it.li_kind & 0x80000000u) {
            const unsigned long long k = atomicAdd(m.stats + S_RECORDS, 1ULL);
            if (k < m.rec_cap) m.rec[k] = (vid << m.order_bits) | it.val;
        } else {
            red_add(reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]) + vid, it.val);
        }
    }
}

}  // namespace vm
