// sr_tri.cuh -- column pass of the phi solve as a cyclic tridiagonal solve (sm_100a).
//
// After the row R2C pass, Eq. (31)-(33) decouple per spectrum column k2 into
//     c x_i - a (x_{i-1} + x_{i+1}) = d_i   (i cyclic in [0, M)),
//     a = tau mu,  c = 1 + tau mu (4 - 2 cos(2 pi k2 / N)),
// the real-space form along i of dividing by the symbol 1 + tau mu (4 - 2 cos z1 - 2 cos z2) (Eq. 32, Q10).
// k_cols_solve does that division between a forward and an inverse M-point FFT; this kernel solves the
// same system directly.  With r = 2a / (c + sqrt(c^2 - 4 a^2)) < 1 and kappa = 1 / sqrt(c^2 - 4 a^2) the
// cyclic Green's function is kappa sum_m r^|n + m M|, so
//     y_i = d_i + r y_{i-1},   z_i = d_i + r z_{i+1}   (both cyclic),   x_i = kappa (y_i + r z_{i+1}):
// two first-order recurrences, O(M) instead of O(M log M), no twiddles, no transposes through shared
// memory between radix stages -- the pass becomes a streaming kernel (8 B read + 8 B written per complex).
// Exact (the same linear system; different rounding order).  The packed slot 0 holds the real columns
// k2 = 0 (real part) and k2 = N/2 (imaginary part): the recurrences run per component with that
// component's (r, kappa), so no unpacking is needed.
//
// Parallel form.  A column is cut into chunks of L = 16 consecutive elements, one thread each.  A chunk's
// local recurrences (zero incoming) give its end values Bf (forward) and Bb (backward); the true incoming
// values are Yin_c = sum_{m >= 1} rho^{m-1} Bf_{c-m}, Zin_c = sum_{m >= 1} rho^{m-1} Bb_{c+m}, rho = r^L,
// chunk indices cyclic.  The sum stops after mmax terms, where rho^mmax < 2^-48 (weights below any fp32
// rounding of the result); if that does not happen within one wrap (mmax = C chunks) the sum over one wrap
// times 1 / (1 - rho^C) is the full cyclic series.  r, kappa / (N/2), rho, mmax and that factor come from a
// per-column table computed in fp64 on the host (TriCol).
#pragma once
#include <cuda_runtime.h>
#include <cmath>
#include "sr_tma.cuh"

namespace srsb {

// ---- host logic (fp64): constants of c x_i - a (x_{i-1} + x_{i+1}) = d_i, cut into C chunks of L
// carry terms of the chunked recurrences of sr_tri.cuh: the smallest m with rho^m < 2^-48 (rho = r^L), at most
// one wrap of C chunks (then the series is closed by 1 / (1 - rho^C))
inline int tri_carry_terms(double rho, int C, double* clos) {
    int m = 1;
    if (rho > 0.0) {
        const double v = std::ceil(-48.0 * std::log(2.0) / std::log(rho));
        m = v > (double)C ? C : (int)v;
    }
    if (m < 1) m = 1;
    if (clos) *clos = 1.0;
    if (m >= C) {
        m = C;
        if (clos) *clos = 1.0 / (1.0 - std::pow(rho, C));
    }
    return m;
}
inline double tri_ratio(double a, double cc, double* sq_out) {   // r = 2a / (c + sqrt(c^2 - 4 a^2)) of c x_i - a (x_{i-1} + x_{i+1})
    const double sq = std::sqrt(cc * cc - 4.0 * a * a);
    if (sq_out) *sq_out = sq;
    return 2.0 * a / (cc + sq);
}


struct TriCol {       // per global spectrum column k2; [0] real part, [1] imaginary part (differ only for k2 = 0)
    float r[2];       // recurrence ratio
    float ks[2];      // kappa / (N/2): Green's function scale and the row-FFT normalisation
    float rho[2];     // r^L
    float clos[2];    // 1 / (1 - rho^C) when the carry sum runs a full wrap, else 1
    int mmax;         // carry terms
    int pad_[3];
};

#ifndef SRSB_TRI_MINB
#define SRSB_TRI_MINB 2
#endif

// spec: [B][H][M] complex (G = 1: each column contiguous), solved in place.  grid (columns / cpc, B),
// block cpc * M / L threads, dynamic shared memory cpc * (M + 3 M / L) float2.
// Slab mode: the all-to-all receive buffer holds column k2l as P segments of 2^lg_seg rows,
// segment s at s * seg_stride + (k2l << lg_seg) (whole image: one segment, lg_seg = lgM); tc points at the
// entry of local column 0 (global column k2_off).  Same chunks, same sums: bitwise the whole-image result.
template <int LOGL>
__global__ void __launch_bounds__(512, SRSB_TRI_MINB) k_cols_tri(float2* __restrict__ spec, const TriCol* __restrict__ tc,
                                                                 int lgM, int lg_cpc, long long bstride, int lg_seg,
                                                                 long long seg_stride) {
    constexpr int L = 1 << LOGL;
    extern __shared__ float2 smem2[];
    const int M = 1 << lgM, lgC = lgM - LOGL, C = 1 << lgC;
    const int SC = M + C;                       // one pad slot per chunk: chunk stride L + 1 (odd) -> the
                                                // per-thread chunk walks are bank-conflict-free
    const int cpc = 1 << lg_cpc;
    const int tid = threadIdx.x, T = blockDim.x;   // T = cpc * C
    float2* data = smem2;                          // [cpc][SC]
    float2* Bf = smem2 + cpc * SC;                 // [cpc][C]
    float2* Bb = Bf + cpc * C;
    float2* g = spec + blockIdx.y * bstride + ((long long)(blockIdx.x << lg_cpc) << lg_seg);
    const int segmask = (1 << lg_seg) - 1;
    // element i of the CTA's column cl
    auto at = [&](int cl, int i) -> float2* {
        return g + (long long)(i >> lg_seg) * seg_stride + ((long long)cl << lg_seg) + (i & segmask);
    };
    // stage the CTA's cpc columns (coalesced 8-byte cp.async into the padded rows)
#pragma unroll 4
    for (int u = 0; u < L; u++) {
        const int e = tid + u * T;
        const int cl = e >> lgM, i = e & (M - 1);
        float2* dst = data + cl * SC + i + (i >> LOGL);
        SRSB_CHK(dst, 8);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(at(cl, i)) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int cl = tid >> lgC, c = tid & (C - 1);
    const TriCol* q = tc + ((blockIdx.x << lg_cpc) + cl);
    const float2 r = make_float2(__ldg(&q->r[0]), __ldg(&q->r[1]));
    const float2 rho = make_float2(__ldg(&q->rho[0]), __ldg(&q->rho[1]));
    const int mmax = __ldg(&q->mmax);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    float2* ch = data + cl * SC + c * (L + 1);
    float2 d[L];
#pragma unroll
    for (int j = 0; j < L; j++) d[j] = ch[j];
    {   // local recurrences from zero: the chunk's contribution to what follows / precedes it
        float2 y = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < L; j++) {
            y.x = fmaf(r.x, y.x, d[j].x);
            y.y = fmaf(r.y, y.y, d[j].y);
            z.x = fmaf(r.x, z.x, d[L - 1 - j].x);
            z.y = fmaf(r.y, z.y, d[L - 1 - j].y);
        }
        SRSB_CHK(&Bb[tid], 8);
        SRSB_CHK(&ch[L - 1], 8);
        Bf[tid] = y;
        Bb[tid] = z;
    }
    __syncthreads();
    float2 y = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
    {
        const float2* bf = Bf + (cl << lgC);
        const float2* bb = Bb + (cl << lgC);
        float2 wgt = make_float2(1.f, 1.f);
        for (int m = 1; m <= mmax; m++) {
            const float2 f = bf[(c - m) & (C - 1)], bk = bb[(c + m) & (C - 1)];
            y.x = fmaf(wgt.x, f.x, y.x);
            y.y = fmaf(wgt.y, f.y, y.y);
            z.x = fmaf(wgt.x, bk.x, z.x);
            z.y = fmaf(wgt.y, bk.y, z.y);
            wgt.x *= rho.x;
            wgt.y *= rho.y;
        }
        const float2 clos = make_float2(__ldg(&q->clos[0]), __ldg(&q->clos[1]));
        y.x *= clos.x;  y.y *= clos.y;
        z.x *= clos.x;  z.y *= clos.y;
    }
    // forward recurrence with the true incoming value; d[j] <- y_j
#pragma unroll
    for (int j = 0; j < L; j++) {
        y.x = fmaf(r.x, y.x, d[j].x);
        y.y = fmaf(r.y, y.y, d[j].y);
        d[j] = y;
    }
    // backward recurrence (z enters as z_{j+1}; d_j re-read from the chunk) and x_j = ks (y_j + r z_{j+1})
    const float2 ks = make_float2(__ldg(&q->ks[0]), __ldg(&q->ks[1]));
#pragma unroll
    for (int j = L - 1; j >= 0; j--) {
        const float2 dj = ch[j];
        const float2 x = make_float2(ks.x * fmaf(r.x, z.x, d[j].x), ks.y * fmaf(r.y, z.y, d[j].y));
        z.x = fmaf(r.x, z.x, dj.x);
        z.y = fmaf(r.y, z.y, dj.y);
        ch[j] = x;
    }
    __syncthreads();
#pragma unroll 4
    for (int u = 0; u < L; u++) {
        const int e = tid + u * T;
        const int cl2 = e >> lgM, i = e & (M - 1);
        *at(cl2, i) = data[cl2 * SC + i + (i >> LOGL)];
    }
}

// The same solve on a spectrum stored ROW-MAJOR in column groups of G >= 32 columns,
// spec[b][k2 / G][m][k2 % G] (G = N/2: plain row-major), which lets both row passes read and write whole
// 128-byte lines instead of transposed chunks.  Lanes run across 32 adjacent columns (every access is a
// coalesced 256-byte row segment), warp w of the CTA owns chunk ct0 + w of those columns, and the CTA
// covers W chunks of the column, not all of it: the carries from outside the tile come from the end values
// of the mmax chunks above (Bf) and below (Bb) the tile, recomputed here from their rows (L2 hits: the
// neighbouring tiles read them as data).  Chunk indices are cyclic, so the same code handles tiles that
// cover the column more than once over (tiny M).  Out of place (in -> out): a neighbour's halo read must
// see the right-hand side, not the solution.  mmax is the largest carry count over the columns
// (host-checked <= kTriRmMaxCarry, else the transposed layout is used).
constexpr int kTriRmMaxCarry = 4;
template <int LOGL>
__global__ void __launch_bounds__(512, 2) k_cols_tri_rm(const float2* __restrict__ in, float2* __restrict__ out,
                                                        const TriCol* __restrict__ tc, int lgM, int lgG, int H, int mmax,
                                                        int tc_bstride) {
    constexpr int L = 1 << LOGL;
    extern __shared__ float2 smem2[];
    const int M = 1 << lgM, C = M >> LOGL, G = 1 << lgG;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int k2 = blockIdx.x * 32 + lane;
    const size_t base = (size_t)blockIdx.z * H * M + ((size_t)(k2 >> lgG) << (lgM + lgG)) + (k2 & (G - 1));
    const float2* col = in + base;                 // element m of the column: col[m << lgG]
    const int ct0 = blockIdx.y * W, cg = ct0 + w;   // this warp's chunk
    float2* my = smem2 + (w * L) * 32 + lane;       // [W][L][32] thread-private copy of the chunk (re-read by
                                                    // the backward recurrence)
    float2* Bf = smem2 + W * L * 32;                // [mmax + W][32]: chunks ct0 - mmax .. ct0 + W - 1
    float2* Bb = Bf + (mmax + W) * 32;              // [W + mmax][32]: chunks ct0 .. ct0 + W + mmax - 1
    {
        const float2* src = col + ((size_t)(cg * L) << lgG);
#pragma unroll
        for (int j = 0; j < L; j++) {
            SRSB_CHK(my + j * 32, 8);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(my + j * 32)),
                         "l"(src + ((size_t)j << lgG)) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const TriCol* q = tc + (size_t)blockIdx.z * tc_bstride + k2;   // tc_bstride = 0: one table for every image (2-D);
                                                                   // 3-D: one table row per spectrum plane
    const float2 r = make_float2(__ldg(&q->r[0]), __ldg(&q->r[1]));
    const float2 rho = make_float2(__ldg(&q->rho[0]), __ldg(&q->rho[1]));
    for (int h = w; h < 2 * mmax; h += W) {   // halo chunks: end values only
        const bool above = h < mmax;
        const int k = above ? h : h - mmax;
        const int hc = (above ? ct0 - 1 - k : ct0 + W + k) & (C - 1);
        // rows in sweep order: ascending for a forward end value, descending for a backward one
        const float2* hp = col + ((size_t)(hc * L + (above ? 0 : L - 1)) << lgG);
        const long long step = above ? (long long)G : -(long long)G;
        float2 hv[L];
#pragma unroll
        for (int j = 0; j < L; j++) hv[j] = __ldg(hp + j * step);
        float2 e = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < L; j++) {
            e.x = fmaf(r.x, e.x, hv[j].x);
            e.y = fmaf(r.y, e.y, hv[j].y);
        }
        SRSB_CHK(above ? Bf + (mmax - 1 - k) * 32 + lane : Bb + (W + k) * 32 + lane, 8);
        if (above) Bf[(mmax - 1 - k) * 32 + lane] = e;
        else Bb[(W + k) * 32 + lane] = e;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    float2 d[L];
#pragma unroll
    for (int j = 0; j < L; j++) d[j] = my[j * 32];
    {
        float2 y = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < L; j++) {
            y.x = fmaf(r.x, y.x, d[j].x);
            y.y = fmaf(r.y, y.y, d[j].y);
            z.x = fmaf(r.x, z.x, d[L - 1 - j].x);
            z.y = fmaf(r.y, z.y, d[L - 1 - j].y);
        }
        SRSB_CHK(&Bf[(mmax + w) * 32 + lane], 8);
        SRSB_CHK(&Bb[(w + mmax) * 32 + lane], 8);
        Bf[(mmax + w) * 32 + lane] = y;
        Bb[w * 32 + lane] = z;
    }
    __syncthreads();
    float2 y = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
    {
        float2 wgt = make_float2(1.f, 1.f);
        for (int m = 1; m <= mmax; m++) {
            const float2 f = Bf[(mmax + w - m) * 32 + lane], bk = Bb[(w + m) * 32 + lane];
            y.x = fmaf(wgt.x, f.x, y.x);
            y.y = fmaf(wgt.y, f.y, y.y);
            z.x = fmaf(wgt.x, bk.x, z.x);
            z.y = fmaf(wgt.y, bk.y, z.y);
            wgt.x *= rho.x;
            wgt.y *= rho.y;
        }
        const float2 clos = make_float2(__ldg(&q->clos[0]), __ldg(&q->clos[1]));
        y.x *= clos.x;  y.y *= clos.y;
        z.x *= clos.x;  z.y *= clos.y;
    }
#pragma unroll
    for (int j = 0; j < L; j++) {
        y.x = fmaf(r.x, y.x, d[j].x);
        y.y = fmaf(r.y, y.y, d[j].y);
        d[j] = y;
    }
    const float2 ks = make_float2(__ldg(&q->ks[0]), __ldg(&q->ks[1]));
    float2* dst = out + base + ((size_t)(cg * L) << lgG);
#pragma unroll
    for (int j = L - 1; j >= 0; j--) {
        const float2 dj = my[j * 32];
        const float2 x = make_float2(ks.x * fmaf(r.x, z.x, d[j].x), ks.y * fmaf(r.y, z.y, d[j].y));
        z.x = fmaf(r.x, z.x, dj.x);
        z.y = fmaf(r.y, z.y, dj.y);
        dst[(size_t)j << lgG] = x;
    }
}

typedef void (*ColTriKernel)(float2*, const TriCol*, int, int, long long, int, long long);
typedef void (*ColTriRmKernel)(const float2*, float2*, const TriCol*, int, int, int, int, int);
ColTriRmKernel pick_col_tri_rm();   // fft_tri.cu
ColTriKernel pick_col_tri();     // fft_tri.cu
constexpr int kTriLogL = 4;      // chunk length 2^kTriLogL

}  // namespace srsb
