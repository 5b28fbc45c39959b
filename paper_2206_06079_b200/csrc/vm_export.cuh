// vm_export.cuh -- voxel selection and gather for the map exporters
// (exporters.py:44-159): the reference walks every voxel of every region in
// sorted-region, local-index order in Python (exporters.py:33-41); here one
// block per region counts the voxels a format keeps, a second pass writes
// their local indices in the same order (block-wide ordered compaction), and
// a gather copies the layers the format prints.
#pragma once

#include "vm_kernels.cuh"

namespace vm {

enum ExportKind { EX_OCCUPIED = 0, EX_NDT = 1, EX_TSDF = 2, EX_DECAY = 3 };

constexpr int EX_BLOCK = 256;

// exporters.py:53 (`l <= threshold` is skipped: a float32 against a Python
// float, which NumPy 2 compares in float32 -- NEP 50), :88 (mean_count == 0),
// :131 (tsdf weight == 0), :149 (no hits and no distance)
__device__ __forceinline__ bool ex_keep(const DevMap &m, int kind, int slot, int li,
                                        double threshold) {
    const size_t v = (size_t)slot * m.vpr + li;
    switch (kind) {
    case EX_OCCUPIED:
        return !(reinterpret_cast<const float *>(m.slab[L_OCC])[v] <= (float)threshold);
    case EX_NDT:
        return reinterpret_cast<const unsigned *>(m.slab[L_COUNT])[v] != 0u;
    case EX_TSDF:
        return reinterpret_cast<const float *>(m.slab[L_TSDF])[2 * v + 1] != 0.0f;
    default:
        return reinterpret_cast<const double *>(m.slab[L_DDIST])[v] != 0.0 ||
               reinterpret_cast<const unsigned *>(m.slab[L_DHITS])[v] != 0u;
    }
}

__global__ void __launch_bounds__(EX_BLOCK) k_export_count(const __grid_constant__ DevMap m,
                                                           const int *slots, int kind,
                                                           double threshold,
                                                           unsigned long long *counts) {
    const int slot = slots[blockIdx.x];
    unsigned c = 0;
    for (int li = threadIdx.x; li < m.vpr; li += blockDim.x) c += ex_keep(m, kind, slot, li, threshold);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    __shared__ unsigned ws[EX_BLOCK / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (int w = 0; w < EX_BLOCK / 32; ++w) t += ws[w];
        counts[blockIdx.x] = t;
    }
}

// Ordered compaction: thread t owns the contiguous run of local indices
// [t * per, (t + 1) * per); a block scan of the per-thread counts gives every
// kept voxel its position within the region.
__global__ void __launch_bounds__(EX_BLOCK) k_export_write(const __grid_constant__ DevMap m,
                                                           const int *slots, int kind,
                                                           double threshold,
                                                           const unsigned long long *offsets,
                                                           int *ridx, int *li_out) {
    const int slot = slots[blockIdx.x];
    const int per = (m.vpr + EX_BLOCK - 1) / EX_BLOCK;
    const int l0 = threadIdx.x * per, l1 = min(m.vpr, l0 + per);
    unsigned c = 0;
    for (int li = l0; li < l1; ++li) c += ex_keep(m, kind, slot, li, threshold);
    __shared__ unsigned sc[EX_BLOCK];
    sc[threadIdx.x] = c;
    __syncthreads();
    for (int o = 1; o < EX_BLOCK; o <<= 1) {  // inclusive Hillis-Steele scan
        const unsigned x = threadIdx.x >= (unsigned)o ? sc[threadIdx.x - o] : 0u;
        __syncthreads();
        sc[threadIdx.x] += x;
        __syncthreads();
    }
    unsigned long long pos = offsets[blockIdx.x] + sc[threadIdx.x] - c;
    for (int li = l0; li < l1; ++li) {
        if (!ex_keep(m, kind, slot, li, threshold)) continue;
        ridx[pos] = (int)blockIdx.x;
        li_out[pos] = li;
        ++pos;
    }
}

// out[i] = the `bytes`-byte record of voxel (slots[ridx[i]], li[i]) of a layer
__global__ void k_export_gather(const __grid_constant__ DevMap m, int layer, int bytes,
                                const int *slots, const int *ridx, const int *li, long long n,
                                unsigned char *out) {
    const long long total = n * bytes;
    const unsigned char *base = reinterpret_cast<const unsigned char *>(m.slab[layer]);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const long long i = k / bytes;
        const int b = (int)(k - i * bytes);
        const size_t v = (size_t)slots[ridx[i]] * m.vpr + li[i];
        out[k] = base[v * bytes + b];
    }
}

}  // namespace vm
