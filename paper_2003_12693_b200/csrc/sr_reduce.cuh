// sr_reduce.cuh -- deterministic reductions for the NEXT-1 monitor: every CTA writes
// its partial sums (fp64) to its own slot in a fixed order -- lanes by a fixed xor-shuffle tree,
// warps in index order -- and k_reduce_partials sums the slots of each image in a fixed order.  No
// atomics: the monitor values, and so iterate_until's stop decision, are bitwise run-to-run
// reproducible.
#pragma once
#include <cuda_runtime.h>

namespace srsb {

// Sum v[0..NV) over the CTA (blockDim = power of two, <= 1024) into dst[0..NV) (thread 0 writes):
// lanes by a fixed fp32 xor-shuffle tree (as the former per-warp atomics did), warps in index order
// in fp64.  Must be reached by every thread of the CTA (it synchronizes).
template <int NV>
__device__ __forceinline__ void block_partials(const float (&v)[NV], double* dst) {
    __shared__ double red[32][NV];
    const int nt = blockDim.x * blockDim.y * blockDim.z;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nw = nt < 32 ? nt : 32;                       // lanes per warp that exist
    const unsigned mask = nw == 32 ? 0xffffffffu : ((1u << nw) - 1u);
    float d[NV];
#pragma unroll
    for (int k = 0; k < NV; k++) d[k] = v[k];
    for (int o = nw / 2; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < NV; k++) d[k] += __shfl_xor_sync(mask, d[k], o);
    if ((tid & 31) == 0)
#pragma unroll
        for (int k = 0; k < NV; k++) red[tid >> 5][k] = (double)d[k];
    __syncthreads();
    if (tid == 0) {
        const int nwarps = (nt + 31) / 32;
#pragma unroll
        for (int k = 0; k < NV; k++) {
            double s = 0.0;
            for (int w = 0; w < nwarps; w++) s += red[w][k];
            dst[k] = s;
        }
    }
}

// out[img * out_stride + k] = sum over j = 0..nblk-1 (in order of a fixed 32-lane tree) of
// part[(img * nblk + j) * nv + k]; one warp per (img, k): grid = nimg * nv, block = 32.
static __global__ void k_reduce_partials(const double* __restrict__ part, int nblk, int nv, double* __restrict__ out,
                                  int out_stride) {
    const int img = blockIdx.x / nv, k = blockIdx.x - img * nv, lane = threadIdx.x;
    double s = 0.0;
    for (int j = lane; j < nblk; j += 32) s += part[((long long)img * nblk + j) * nv + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[(long long)img * out_stride + k] = s;
}

}  // namespace srsb
