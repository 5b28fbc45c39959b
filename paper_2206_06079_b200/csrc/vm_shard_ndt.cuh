// vm_shard_ndt.cuh -- region-sharded NDT-OM.
//
// NDT phase 1 weighs a miss through a voxel by the voxel's Gaussian
// (_kernels.pyx:602-648), which only the voxel's owner holds.  The protocol
// keeps the reference's phase barrier (engine.py:285: every phase-1 update
// of the batch before any phase-2 update) and sends as little as possible:
//
//   begin    discover the slice (clip, segment, prefetch, phase-2 records of
//            the slice's samples)
//   request  every ghost region the slice prefetched, to its owner
//   -- exchange A: requests all-to-all --
//   bits     the owner answers each request with the region's Gaussian
//            bitmap (count >= 3 at the start of the batch, 1 bit per voxel)
//   -- exchange A': bitmaps back --
//   mark     GAUSS_FLAG into the requester's ghost scratch words
//   walk     the NDT walk of the slice: an owned voxel as on one GPU; a ghost
//            voxel with GAUSS_FLAG (or in a region without a bitmap) becomes
//            a 32-byte visit item (segment order, chord t0 / t1) for its
//            owner; any other ghost visit is an order-free miss count
//   export   visit items, ghost miss counts, the phase-2 records of ghost
//            sample voxels -- all per owner
//   -- exchange B: items all-to-all --
//   import   the owner files each visit as a phase-1 record of its own
//            Gaussian voxel; k_ndt_weigh weighs it from the segment (every
//            rank holds the whole batch) exactly like its own walk's records
//   finish   drop the ghost state; resolve, bucket, fold as on one GPU
//
// Every record carries its global segment order, so each owner folds the
// same sequence the single-GPU fold sees: the union of the owned regions
// equals the single-GPU map (tests/test_gpu_sharded.py).
#pragma once

#include "vm_ndt.cuh"
#include "vm_shard.cuh"

namespace vm {

// request list: the ghost regions this slice prefetched (touched list)
__global__ void k_shard_ndt_req(const __grid_constant__ DevMap m, long long *req,
                                unsigned long long *nreq, unsigned long long req_cap) {
    unsigned long long nt = *((volatile unsigned long long *)(m.stats + S_WALK_TOUCHED));
    if (nt > (unsigned long long)m.touched_cap) nt = m.touched_cap;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        const int slot = m.touched[t];
        if (slot < 0 || slot >= m.cap) continue;
        const long long key = m.slot_keys[slot];
        const int d = region_owner(key, m.shard_world);
        if (d == m.shard_rank) continue;
        const unsigned long long k = atomicAdd(nreq + d, 1ULL);
        if (k < req_cap) req[(unsigned long long)d * req_cap + k] = key;
    }
}

// owner: create each requested region if new, answer with its bitmap
// (words per region = ceil(vpr / 32)); one warp per 32 voxels
__global__ void __launch_bounds__(BLOCK) k_shard_ndt_bits(const __grid_constant__ DevMap m,
                                                          const long long *req, long long nreq,
                                                          unsigned *bits, int words) {
    const int lane = threadIdx.x & 31;
    for (long long r = blockIdx.x; r < nreq; r += gridDim.x) {
        const int slot = region_slot(m, req[r]);
        const unsigned *cnt = slot >= 0 && slot < m.cap ? layer_at<unsigned>(m, L_COUNT, slot) : nullptr;
        for (int w = threadIdx.x >> 5; w < words; w += blockDim.x >> 5) {
            const int li = w * 32 + lane;
            const bool g = cnt && li < m.vpr && cnt[li] >= 3u;
            const unsigned b = __ballot_sync(0xffffffffu, g);
            if (lane == 0) bits[(size_t)r * words + w] = b;
        }
    }
}

// requester: GAUSS_FLAG into the ghost scratch words (zero between batches)
__global__ void __launch_bounds__(BLOCK) k_shard_ndt_mark(const __grid_constant__ DevMap m,
                                                          const long long *keys, const unsigned *bits,
                                                          long long n, int words) {
    for (long long r = blockIdx.x; r < n; r += gridDim.x) {
        const int slot = region_find(m, keys[r]);
        if (slot < 0 || slot >= m.cap) continue;
        unsigned *scr = layer_at<unsigned>(m, L_SCRATCH, slot);
        for (int w = threadIdx.x; w < words; w += blockDim.x) {
            unsigned b = bits[(size_t)r * words + w];
            while (b) {
                const int j = __ffs(b) - 1;
                b &= b - 1;
                scr[w * 32 + j] = GAUSS_FLAG;
            }
        }
    }
}

__device__ __forceinline__ void shard_emit_n(ShardItemN *out, unsigned long long *cnt,
                                             unsigned long long cap_per, int dest, const ShardItemN &it) {
    const unsigned long long k = atomicAdd(cnt + dest, 1ULL);
    if (k < cap_per) out[(unsigned long long)dest * cap_per + k] = it;
}

// export: the walk's ghost visit items, ghost miss counts, and the phase-2
// records the slice's discover filed for ghost sample voxels
__global__ void __launch_bounds__(BLOCK) k_shard_ndt_export(const __grid_constant__ DevMap m,
                                                            unsigned long long R, ShardItemN *out,
                                                            unsigned long long *cnt,
                                                            unsigned long long cap_per) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long ng = min(*((volatile unsigned long long *)m.ngx), m.gx_cap);
    const ShardItemN *gx = reinterpret_cast<const ShardItemN *>(m.gx);
    for (unsigned long long k = tid; k < ng; k += stride) {
        const ShardItemN it = gx[k];
        shard_emit_n(out, cnt, cap_per, region_owner(it.rkey, m.shard_world), it);
    }
    const unsigned long long M = min(*((volatile unsigned long long *)m.nmarked), m.marked_cap);
    for (unsigned long long i = tid; i < R; i += stride) {
        const unsigned long long k = m.rec[i];
        if (!((k >> 31) & 1ULL)) continue;  // phase-1 records are the slice's own voxels
        const unsigned mi = (unsigned)(k >> 32);
        if (mi >= M) continue;
        const int2 sl = m.marked[mi];
        if (sl.x < 0 || !is_ghost(m, sl.x)) continue;
        const long long key = m.slot_keys[sl.x];
        shard_emit_n(out, cnt, cap_per, region_owner(key, m.shard_world),
                     ShardItemN{key, (unsigned)sl.y | (1u << 30), (unsigned)k & 0x7FFFFFFFu, 0.0, 0.0});
    }
    const unsigned *scr0 = reinterpret_cast<const unsigned *>(m.slab[L_SCRATCH]);
    VM_TOUCHED_REGIONS({
        const long long key = m.slot_keys[slot];
        const int dest = region_owner(key, m.shard_world);
        const unsigned *scr = scr0 + (size_t)slot * m.vpr;
        for (int li = threadIdx.x; li < m.vpr; li += blockDim.x) {
            const unsigned c = scr[li] & ~GAUSS_FLAG;
            if (c) shard_emit_n(out, cnt, cap_per, dest, ShardItemN{key, (unsigned)li, c, 0.0, 0.0});
        }
    })
}

// drop the ghost state of the batch: scratch words (counts, GAUSS_FLAG) of
// the ghost regions the walk touched and the ghost sample voxels' indices
__global__ void __launch_bounds__(BLOCK) k_shard_ndt_clear(const __grid_constant__ DevMap m) {
    const unsigned long long M = min(*((volatile unsigned long long *)m.nmarked), m.marked_cap);
    for (unsigned long long mi = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; mi < M;
         mi += (unsigned long long)gridDim.x * blockDim.x) {
        const int2 sl = m.marked[mi];
        if (sl.x < 0 || !is_ghost(m, sl.x)) continue;
        layer_at<unsigned>(m, m.nidx, sl.x)[sl.y] = 0u;
        m.marked[mi] = make_int2(-1, -1);  // the fold skips the bucket
    }
    unsigned *scr0 = reinterpret_cast<unsigned *>(m.slab[L_SCRATCH]);
    VM_TOUCHED_REGIONS({
        unsigned *scr = scr0 + (size_t)slot * m.vpr;
        for (int li = threadIdx.x; li < m.vpr; li += blockDim.x)
            if (scr[li]) scr[li] = 0u;
    })
}

// owner, pass 1: every region the items address exists afterwards
__global__ void k_shard_ndt_import_regions(const __grid_constant__ DevMap m, const ShardItemN *in,
                                           long long n) {
    long long prev = -1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long key = in[i].rkey;
        if (key != prev) region_slot(m, key);
        prev = key;
    }
}

// owner, pass 2 (regions exist): file counts, samples and weighed visits
template <class Src>
__global__ void __launch_bounds__(BLOCK) k_shard_ndt_import(const __grid_constant__ DevMap m, Src src,
                                                            const ShardItemN *in, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const ShardItemN it = in[i];
        const int s = region_find(m, it.rkey);
        if (s < 0 || s >= m.cap) continue;
        if (stamp_epoch(m.slot_touch + s, m.epoch)) {
            const unsigned long long t = atomicAdd(m.stats + S_WALK_TOUCHED, 1ULL);
            if (t < (unsigned long long)m.touched_cap) m.touched[t] = s;
        }
        const int li = (int)(it.li_kind & 0x3FFFFFFFu);
        const unsigned kind = it.li_kind >> 30;
        unsigned *scr = layer_at<unsigned>(m, L_SCRATCH, s) + li;
        if (kind == 0u) {
            red_add(scr, it.val);
            continue;
        }
        if (kind == 1u) {
            const unsigned long long k = atomicAdd(m.stats + S_RECORDS, 1ULL);
            if (k < m.rec_cap) {
                m.rec[k] = ndt_key(ndt_index(m, s, li), 1u, it.val);
                m.recval[k] = 0u;
            }
            continue;
        }
        // a phase-1 visit: a record of this rank's Gaussian voxel
        const unsigned ns = layer_at<unsigned>(m, L_COUNT, s)[li];
        if (ns < 3u) {
            red_add(scr, 1u);
            continue;
        }
        // (k_ndt_weigh weighs it with this rank's Gaussian, like its own records)
        const unsigned long long k = atomicAdd(m.stats + S_RECORDS, 1ULL);
        if (k < m.rec_cap) {
            m.rec[k] = ndt_key(ndt_index(m, s, li), 0u, it.val);
            m.rec_t[k] = make_double2(it.t0, it.t1);
        }
    }
}

}  // namespace vm
