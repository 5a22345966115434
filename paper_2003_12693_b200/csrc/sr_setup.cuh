// sr_setup.cuh -- one-time kernels of Algorithm 1 step (1): edge indicator Eq. (1)
// and w^0 = grad phi^0, b^0 = 0.  Included by srsb.cu only.
#pragma once
#include <cuda_runtime.h>

namespace srsb {

// ---------------------------------------------------------------- one-time kernels

struct EdgeArgs {
    int M, N, r;     // blur radius ceil(3 sigma) <= 8
    float k[17];     // normalized Gaussian taps, k[t + r]
    float rho;
    int s;
};

// Eq. (1) step 1: f_s = G_sigma * f, rows (replicate padding)
__global__ void k_blur_rows(const float* __restrict__ f, float* __restrict__ out, EdgeArgs a) {
    const size_t plane = (size_t)a.M * a.N;
    const int img = blockIdx.z;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.N) return;
    const float* src = f + img * plane + (size_t)i * a.N;
    float acc = 0.f;
    for (int t = -a.r; t <= a.r; t++) {
        const int jj = min(max(j + t, 0), a.N - 1);
        acc = fmaf(a.k[t + a.r], __ldg(src + jj), acc);
    }
    out[img * plane + (size_t)i * a.N + j] = acc;
}

// Eq. (1) step 1 (columns)
__global__ void k_blur_cols(const float* __restrict__ in, float* __restrict__ out, EdgeArgs a) {
    const size_t plane = (size_t)a.M * a.N;
    const int img = blockIdx.z;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.N) return;
    const float* src = in + img * plane;
    float acc = 0.f;
    for (int t = -a.r; t <= a.r; t++) {
        const int ii = min(max(i + t, 0), a.M - 1);
        acc = fmaf(a.k[t + a.r], __ldg(src + (size_t)ii * a.N + j), acc);
    }
    out[img * plane + (size_t)i * a.N + j] = acc;
}

// Eq. (1) step 2: central differences (replicate padding), g = 1/(1 + rho |grad|^s)
__global__ void k_edge_g(const float* __restrict__ fs, float* __restrict__ g, EdgeArgs a) {
    const size_t plane = (size_t)a.M * a.N;
    const int img = blockIdx.z;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.N) return;
    const float* src = fs + img * plane;
    const int ip = min(i + 1, a.M - 1), im = max(i - 1, 0), jp = min(j + 1, a.N - 1), jm = max(j - 1, 0);
    const float gx = 0.5f * (__ldg(src + (size_t)ip * a.N + j) - __ldg(src + (size_t)im * a.N + j));
    const float gy = 0.5f * (__ldg(src + (size_t)i * a.N + jp) - __ldg(src + (size_t)i * a.N + jm));
    const float m2 = gx * gx + gy * gy;
    const float mag = (a.s == 2) ? m2 : sqrtf(m2);
    g[img * plane + (size_t)i * a.N + j] = 1.f / (1.f + a.rho * mag);
}

// Alg. 1 (1): w = grad phi0 (Eq. 35, zero on the last row / column), b = 0
__global__ void k_init_w(const float* __restrict__ phi, float* __restrict__ w, float* __restrict__ bv, int M, int N) {
    const size_t plane = (size_t)M * N;
    const int img = blockIdx.z;
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const float* p = phi + img * plane;
    const size_t o = (size_t)i * N + j;
    const float c = p[o];
    float* w1 = w + img * 2 * plane;
    float* b1 = bv + img * 2 * plane;
    w1[o] = (i < M - 1) ? p[o + N] - c : 0.f;
    w1[plane + o] = (j < N - 1) ? p[o + 1] - c : 0.f;
    b1[o] = 0.f;
    b1[plane + o] = 0.f;
}

}  // namespace srsb
