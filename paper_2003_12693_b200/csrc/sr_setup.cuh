// sr_setup.cuh -- one-time kernels of Algorithm 1 step (1): edge indicator Eq. (1)
// and w^0 = grad phi^0, b^0 = 0.  Included by srsb.cu only.
//
// Layout as in sr_stencil.cuh: pointers address local row 0 of image 0, image planes are `plane`
// floats apart, local rows -gh .. M + gh - 1 exist (ghost rows).  Boundary rules use GLOBAL rows
// (row_off + local row, Mg rows), so a slab computes exactly what the whole image computes,
// provided its ghost rows hold the neighbouring slabs' rows.
#pragma once
#include <cuda_runtime.h>
#include "sr_reduce.cuh"

namespace srsb {

struct EdgeArgs {
    int M, N, r;         // local rows, columns, blur radius ceil(3 sigma) <= 8
    int Mg, row_off;     // global rows, global index of local row 0
    int ext;             // extra rows computed above / below the local rows (row pass of the blur)
    long long plane;     // floats per image plane
    float k[17];         // normalized Gaussian taps, k[t + r]
    float rho;
    int s;
};

// Eq. (1) step 1: f_s = G_sigma * f along rows (replicate padding at the image's columns), for
// local rows -ext .. M + ext - 1 (grid.y = M + 2 ext).
__global__ void k_blur_rows(const float* __restrict__ f, float* __restrict__ out, EdgeArgs a) {
    const int img = blockIdx.z;
    const int i = (int)blockIdx.y - a.ext, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.N) return;
    const int gi = i + a.row_off;
    if (gi < 0 || gi >= a.Mg) return;
    const float* src = f + img * a.plane + (long long)i * a.N;
    float acc = 0.f;
    for (int t = -a.r; t <= a.r; t++) {
        const int jj = min(max(j + t, 0), a.N - 1);
        acc = fmaf(a.k[t + a.r], __ldg(src + jj), acc);
    }
    out[img * a.plane + (long long)i * a.N + j] = acc;
}

// Eq. (1) step 1 along columns (replicate padding at the GLOBAL first/last row), for local rows
// -ext .. M + ext - 1.
__global__ void k_blur_cols(const float* __restrict__ in, float* __restrict__ out, EdgeArgs a) {
    const int img = blockIdx.z;
    const int i = (int)blockIdx.y - a.ext, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.N) return;
    const int gi = i + a.row_off;
    if (gi < 0 || gi >= a.Mg) return;
    const float* src = in + img * a.plane;
    float acc = 0.f;
    for (int t = -a.r; t <= a.r; t++) {
        const int ii = min(max(gi + t, 0), a.Mg - 1) - a.row_off;   // local (possibly ghost) row
        acc = fmaf(a.k[t + a.r], __ldg(src + (long long)ii * a.N + j), acc);
    }
    out[img * a.plane + (long long)i * a.N + j] = acc;
}

// Eq. (1) step 2: central differences (replicate padding), g = 1/(1 + rho |grad|^s), local rows.
__global__ void k_edge_g(const float* __restrict__ fs, float* __restrict__ g, EdgeArgs a) {
    const int img = blockIdx.z;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.N) return;
    const int gi = i + a.row_off;
    const float* src = fs + img * a.plane;
    const int ip = min(gi + 1, a.Mg - 1) - a.row_off, im = max(gi - 1, 0) - a.row_off;
    const int jp = min(j + 1, a.N - 1), jm = max(j - 1, 0);
    const float gx = 0.5f * (__ldg(src + (long long)ip * a.N + j) - __ldg(src + (long long)im * a.N + j));
    const float gy = 0.5f * (__ldg(src + (long long)i * a.N + jp) - __ldg(src + (long long)i * a.N + jm));
    const float m2 = gx * gx + gy * gy;
    const float mag = (a.s == 2) ? m2 : sqrtf(m2);
    g[img * a.plane + (long long)i * a.N + j] = 1.f / (1.f + a.rho * mag);
}

// Alg. 1 (1): w = grad phi0 (Eq. 35, zero on the last global row / column), b = 0.  Reads the
// ghost row below the slab (the next slab's first row).
__global__ void k_init_w(const float* __restrict__ phi, float* __restrict__ w, float* __restrict__ bv, int N,
                         int Mg, int row_off, long long plane) {
    const int img = blockIdx.z;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const float* p = phi + img * plane;
    const long long o = (long long)i * N + j;
    const float c = p[o];
    float* w1 = w + img * 2 * plane;
    float* b1 = bv + img * 2 * plane;
    w1[o] = (i + row_off < Mg - 1) ? p[o + N] - c : 0.f;
    w1[plane + o] = (j < N - 1) ? p[o + 1] - c : 0.f;
    b1[o] = 0.f;
    b1[plane + o] = 0.f;
}

// NEXT-1 outer convergence: per image sum (phi - prev)^2 and sum prev^2 over the local rows, then
// prev = phi.  grid (blocks, batch); out = per-CTA partials [img][blockIdx.x][2] (stride unused).
__global__ void k_phi_change(const float* __restrict__ phi, float* __restrict__ prev, double* __restrict__ out,
                             int M, int N, long long plane, int stride) {
    const int img = blockIdx.y;
    const float* p = phi + img * plane;
    float* q = prev + img * plane;
    float d2 = 0.f, o2 = 0.f;
    const long long n = (long long)M * N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float a = p[i], b = q[i];
        d2 += (a - b) * (a - b);
        o2 += b * b;
        q[i] = a;
    }
    const float pv[2] = {d2, o2};   // per-CTA partials, reduced in a fixed order (k_reduce_partials)
    block_partials<2>(pv, out + ((long long)img * gridDim.x + blockIdx.x) * 2);
}

}  // namespace srsb
