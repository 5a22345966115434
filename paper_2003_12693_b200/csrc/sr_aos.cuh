// sr_aos.cuh -- AOS variant of the phi sub-problem:
//   phi = 1/2 [ (I - c A_1)^{-1} + (I - c A_2)^{-1} ] F,   c = 2 tau mu,
// A_1 / A_2 the 1-D second differences along columns / rows with Neumann (reflecting) ends.  The
// coefficients are constant, so the LR factors (cp_i, r_i) of each direction are computed once on
// the host ("LR decomposition will only need to happen once") and every line is solved by
// forward substitution y_i = r_i (f_i - a y_{i-1}) and back substitution x_i = y_i - cp_i x_{i+1},
// a = -c.
//
// Both recurrences are first-order affine maps v -> A v + B, so a line splits into segments: each
// segment composes its maps, the compositions are scanned across segments (exact, only the
// rounding order changes), and each segment re-runs its recurrence from the scanned input.
//
//   k_aos_vert_reg<L>: columns (M <= 2048).  CTA = CW columns x CH row-chunks of L rows, the chunk
//                      held in registers (F read once, Xv written once: 8 B/px); scan across the
//                      chunks of a column through shared memory.
//   k_aos_vert       : fallback for M > 2048: one thread per column marching down the rows
//                      (F -> Y -> Xv, 16 B/px).
//   k_aos_horiz      : rows.  One warp per row staged in shared memory (padded so each lane's
//                      segment starts in its own bank), the r factors staged once per CTA; scans
//                      across lanes with shuffles; phi = (Xv + Xh) / 2, optionally clamped
//                      (north-star projection after the last sweep).
#pragma once
#include <cuda_runtime.h>

namespace srsb {

struct AosArgs {
    int M, N;
    long long plane;   // floats per image plane (ghost rows included)
    float a;           // -2 tau mu
    float clip;        // > 0: clamp phi to [-clip, clip]
};

__global__ void __launch_bounds__(128) k_aos_vert(const float* __restrict__ F, float* __restrict__ Y,
                                                  float* __restrict__ Xv, const float* __restrict__ cp,
                                                  const float* __restrict__ r, AosArgs q) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, img = blockIdx.y;
    if (j >= q.N) return;
    const float* f = F + img * q.plane + j;
    float* y = Y + img * q.plane + j;
    float* x = Xv + img * q.plane + j;
    float prev = 0.f;
#pragma unroll 8
    for (int i = 0; i < q.M; i++) {
        prev = __ldg(&r[i]) * (f[(long long)i * q.N] - q.a * prev);
        y[(long long)i * q.N] = prev;
    }
    float next = prev;   // x_{M-1} = y_{M-1}
    x[(long long)(q.M - 1) * q.N] = next;
#pragma unroll 8
    for (int i = q.M - 2; i >= 0; i--) {
        next = y[(long long)i * q.N] - __ldg(&cp[i]) * next;
        x[(long long)i * q.N] = next;
    }
}

// affine map v -> A v + B; compose(second, first) = second o first
struct Aff {
    float A, B;
};
__device__ __forceinline__ Aff compose(Aff s, Aff f) { return {s.A * f.A, fmaf(s.A, f.B, s.B)}; }

constexpr int AOS_VT = 512;        // threads per CTA of k_aos_vert_reg
constexpr int AOS_VREG_MAXM = 2048;

// blockDim = (CW, CH), CH * L = M, grid = (N / CW, batch).  Dynamic smem: 4 * CH * CW floats.
template <int L>
__global__ void __launch_bounds__(AOS_VT) k_aos_vert_reg(const float* __restrict__ F, float* __restrict__ Xv,
                                                         const float* __restrict__ cp, const float* __restrict__ r,
                                                         AosArgs q) {
    extern __shared__ float sv[];
    const int CW = blockDim.x, CH = blockDim.y, x = threadIdx.x, yc = threadIdx.y;
    const int j = blockIdx.x * CW + x, img = blockIdx.y, i0 = yc * L;
    float* sA = sv;
    float* sB = sv + CH * CW;
    const long long base = img * q.plane + (long long)i0 * q.N + j;
    float v[L];
#pragma unroll
    for (int t = 0; t < L; t++) v[t] = __ldg(F + base + (long long)t * q.N);
    // forward: y_i = alpha_i y_{i-1} + beta_i, alpha_i = -a r_i, beta_i = r_i f_i
    Aff seg = {1.f, 0.f};
#pragma unroll
    for (int t = 0; t < L; t++) {
        const float ri = __ldg(r + i0 + t);
        seg = compose(Aff{-q.a * ri, ri * v[t]}, seg);
    }
    // inclusive scan over the chunks of this column (top to bottom)
    Aff inc = seg;
    for (int d = 1; d < CH; d <<= 1) {
        sA[yc * CW + x] = inc.A;
        sB[yc * CW + x] = inc.B;
        __syncthreads();
        if (yc >= d) inc = compose(inc, Aff{sA[(yc - d) * CW + x], sB[(yc - d) * CW + x]});
        __syncthreads();
    }
    sB[yc * CW + x] = inc.B;
    __syncthreads();
    float yv = yc > 0 ? sB[(yc - 1) * CW + x] : 0.f;   // the maps applied to y_{-1} = 0
#pragma unroll
    for (int t = 0; t < L; t++) {
        yv = __ldg(r + i0 + t) * (v[t] - q.a * yv);
        v[t] = yv;
    }
    // backward: x_i = -cp_i x_{i+1} + y_i (cp_{M-1} := 0), scanned bottom to top
    float* sA2 = sv + 2 * CH * CW;
    float* sB2 = sv + 3 * CH * CW;
    Aff segb = {1.f, 0.f};
#pragma unroll
    for (int t = L - 1; t >= 0; t--) {
        const float ci = (i0 + t == q.M - 1) ? 0.f : __ldg(cp + i0 + t);
        segb = compose(Aff{-ci, v[t]}, segb);
    }
    Aff incb = segb;
    for (int d = 1; d < CH; d <<= 1) {
        sA2[yc * CW + x] = incb.A;
        sB2[yc * CW + x] = incb.B;
        __syncthreads();
        if (yc + d < CH) incb = compose(incb, Aff{sA2[(yc + d) * CW + x], sB2[(yc + d) * CW + x]});
        __syncthreads();
    }
    sB2[yc * CW + x] = incb.B;
    __syncthreads();
    float xv = yc + 1 < CH ? sB2[(yc + 1) * CW + x] : 0.f;   // x_M = 0
#pragma unroll
    for (int t = L - 1; t >= 0; t--) {
        const float ci = (i0 + t == q.M - 1) ? 0.f : __ldg(cp + i0 + t);
        xv = v[t] - ci * xv;
        Xv[base + (long long)t * q.N] = xv;
    }
}

constexpr int aos_horiz_wpb(int N) { return N <= 2048 ? 8 : 4; }
inline size_t aos_horiz_smem(int N) {
    const int S = N >= 32 ? N / 32 : 1;
    return (size_t)(aos_horiz_wpb(N) + 1) * (N + N / S) * sizeof(float);
}

// Padded shared index: element j of a row sits at j + j / S, so lane l's segment starts at
// l (S + 1): with S even the 32 segment starts fall in 32 different banks.
__device__ __forceinline__ int aos_pad(int j, int S) { return j + j / S; }

// grid = (ceil(M / wpb), batch), blockDim = 32 wpb.  Dynamic smem: (wpb + 1) * (N + N / S) floats.
__global__ void __launch_bounds__(256) k_aos_horiz(const float* __restrict__ F, const float* __restrict__ Xv,
                                                   float* __restrict__ phi, const float* __restrict__ cp,
                                                   const float* __restrict__ r, AosArgs q) {
    extern __shared__ float row_s[];
    const int N = q.N;
    const int S = N >= 32 ? N / 32 : 1;          // segment length per lane
    const int NP = N + N / S;                    // padded row length
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    float* rs = row_s + wpb * NP;                // r factors, padded like the rows
    for (int j = threadIdx.x; j < N; j += blockDim.x) rs[aos_pad(j, S)] = __ldg(r + j);
    __syncthreads();
    const int m = blockIdx.x * wpb + wi, img = blockIdx.y;
    if (m >= q.M) return;
    float* row = row_s + wi * NP;
    const float* f = F + img * q.plane + (long long)m * N;
    for (int j = lane; j < N; j += 32) row[aos_pad(j, S)] = f[j];
    __syncwarp();
    const int j0 = lane * S, p0 = lane * (S + 1);
    const bool active = j0 < N;
    // forward: y_j = alpha_j y_{j-1} + beta_j, alpha_j = -a r_j, beta_j = r_j f_j
    Aff seg = {1.f, 0.f};
    if (active)
        for (int t = 0; t < S; t++) {
            const float rj = rs[p0 + t];
            seg = compose(Aff{-q.a * rj, rj * row[p0 + t]}, seg);
        }
    Aff inc = seg;   // inclusive scan over lanes, left to right
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const float A = __shfl_up_sync(0xffffffffu, inc.A, d), B = __shfl_up_sync(0xffffffffu, inc.B, d);
        if (lane >= d) inc = compose(inc, Aff{A, B});
    }
    float yin = __shfl_up_sync(0xffffffffu, inc.B, 1);   // maps applied to y_{-1} = 0 -> B
    if (lane == 0) yin = 0.f;
    if (active) {
        float y = yin;
        for (int t = 0; t < S; t++) {
            y = rs[p0 + t] * (row[p0 + t] - q.a * y);
            row[p0 + t] = y;
        }
    }
    // backward: x_j = -cp_j x_{j+1} + y_j (cp_{N-1} := 0), scanned right to left; cp_j = a r_j
    Aff segb = {1.f, 0.f};
    if (active)
        for (int t = S - 1; t >= 0; t--) {
            const float cj = (j0 + t == N - 1) ? 0.f : q.a * rs[p0 + t];
            segb = compose(Aff{-cj, row[p0 + t]}, segb);
        }
    Aff incb = segb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const float A = __shfl_down_sync(0xffffffffu, incb.A, d), B = __shfl_down_sync(0xffffffffu, incb.B, d);
        if (lane + d < 32) incb = compose(incb, Aff{A, B});
    }
    float xin = __shfl_down_sync(0xffffffffu, incb.B, 1);  // x entering from the right (x_N = 0)
    if (lane == 31 || (lane + 1) * S >= N) xin = 0.f;
    if (active) {
        float x = xin;
        for (int t = S - 1; t >= 0; t--) {
            const float cj = (j0 + t == N - 1) ? 0.f : q.a * rs[p0 + t];
            x = row[p0 + t] - cj * x;
            row[p0 + t] = x;
        }
    }
    __syncwarp();
    const float* xv = Xv + img * q.plane + (long long)m * N;
    float* out = phi + img * q.plane + (long long)m * N;
    for (int j = lane; j < N; j += 32) {
        float v = 0.5f * (__ldg(xv + j) + row[aos_pad(j, S)]);
        if (q.clip > 0.f) v = fminf(fmaxf(v, -q.clip), q.clip);
        out[j] = v;
    }
}

}  // namespace srsb
