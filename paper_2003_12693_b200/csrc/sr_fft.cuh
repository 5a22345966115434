// sr_fft.cuh -- hand-written power-of-two FFT passes for the phi sub-problem (sm_100a).
//
// Solves (1 - tau mu Delta_per) phi = F, i.e. phi = Re F^-1( F(F) / symbol ),
// Eq. (31)-(33), with the symbol of Eq. (32) read as
// 1 + tau mu (4 - 2 cos z1 - 2 cos z2) (Q10).  Three HBM passes:
//
//   k_rows_r2c   : each image row of N reals -> N/2 + 1 bins (N/2-point complex
//                  FFT of (x[2n], x[2n+1]) + split), bins 0 and N/2 packed into
//                  slot 0 (both real); stored TRANSPOSED in column groups:
//                  spec[b][k2 / G][m][k2 % G]  (complex64)
//   k_cols_solve : per spectrum column (contiguous M complex): forward M-point FFT,
//                  multiply by 1 / (M (N/2) symbol(k1, k2)) (the packed slot 0 is
//                  unpacked to the k2 = 0 and k2 = N/2 symbols), inverse FFT, in place
//   k_rows_c2r   : transposed load, inverse real FFT, optional clamp, phi rows
//
// Inside a CTA each transform is a Stockham autosort FFT: every thread holds
// E (<= 16) complex values in registers, runs radix-R (R <= 16) butterflies in
// registers and exchanges through shared memory between stages (one padded
// SoA row per transform).  Twiddles come from fp32 tables computed in fp64 on
// the host.  No cuFFT.
#pragma once
#include <cuda_runtime.h>
#include "sr_tma.cuh"
#include "sr_reduce.cuh"

namespace srsb {

#ifndef SRSB_COLS_MAXNREG
#define SRSB_COLS_MAXNREG 96   // 64-thread column CTAs: 96 registers -> 10 CTAs / SM without spills (128: 8)
#endif
#ifndef SRSB_COLS_MAXNREG_BIG
#define SRSB_COLS_MAXNREG_BIG 64   // M >= 4096: 256 / 512-thread column CTAs, 2 resident per SM instead of 1
#endif

// L2 prefetch of the input of the CTA launched SRSB_*_PF_DIST CTAs later (about one full wave of
// resident CTAs ahead), issued by thread 0 at the start: bit 0 r2c (its 8 rows of D), bit 1 the
// contiguous-column solve (its column), bit 2 c2r (its rows of psi).  0 = off.
#ifndef SRSB_FFT_PF
#define SRSB_FFT_PF 0
#endif
#ifndef SRSB_R2C_MIRROR
#define SRSB_R2C_MIRROR 1   // r2c split: bins k and H - k from one pair of shared reads (0: one bin per pair)
#endif
#ifndef SRSB_R2C_SHFL
#define SRSB_R2C_SHFL 1     // the row-major H = 512 instances (one warp per row) do the real split through warp shuffles
                            // (C3 r2c 0.109 -> 0.097 ms; same formulas, but the compiler contracts them into other FMAs
                            // than in the shared-memory split, so not bitwise equal to SRSB_R2C_SHFL=0)
#endif
#ifndef SRSB_R2C_PF_DIST
#define SRSB_R2C_PF_DIST 592    // 148 SMs x 4 resident CTAs
#endif
#ifndef SRSB_COLS_PF_DIST
#define SRSB_COLS_PF_DIST 1480  // 148 x 10
#endif
#ifndef SRSB_C2R_PF_DIST
#define SRSB_C2R_PF_DIST 296    // 148 x 2
#endif
// 2-D grid block `ahead` launches after this one (blockIdx.x fastest); false past the grid
__device__ __forceinline__ bool block_ahead_2d(int ahead, int& bx, int& by) {
    const int lin = blockIdx.x + gridDim.x * blockIdx.y + ahead;
    if (lin >= (int)(gridDim.x * gridDim.y)) return false;
    bx = lin % gridDim.x;
    by = lin / gridDim.x;
    return true;
}

// float2 shared-memory index with one pad slot per 16 complex values (128 B): strided butterfly
// accesses with power-of-two strides <= 16 hit 16 distinct 8-byte bank pairs per half-warp.
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// scale / symbol(k1, k2) with symbol = 1 + tau mu (cm + ck) in [1, 1 + 8 tau mu] (Eq. 32, Q10).  scale =
// 1 / (M N/2) is a power of two, so scale * rcp_rn(symbol) IS the IEEE quotient (correctly rounded, Q20)
// at the cost of a correctly rounded reciprocal instead of a full division.
__device__ __forceinline__ float sym_scale(float scale, float taumu, float cm, float ck) {
    return scale * __frcp_rn(1.f + taumu * (cm + ck));
}

__host__ __device__ constexpr int brevn(int k, int bits) {
    int r = 0;
    for (int i = 0; i < bits; i++) r |= ((k >> i) & 1) << (bits - 1 - i);
    return r;
}

// d * exp(-+ 2 pi i idx / 16); idx is a compile-time constant after unrolling.
template <bool INV>
__device__ __forceinline__ float2 tw16(float2 d, int idx) {
    idx &= 15;
    if (idx == 0) return d;
    if (idx == 8) return make_float2(-d.x, -d.y);
    if (idx == 4) return INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
    if (idx == 12) return INV ? make_float2(d.y, -d.x) : make_float2(-d.y, d.x);
    const float C[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                         0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                         -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                         0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
    const float Sn[16] = {0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f,
                          1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                          0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                          -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f};
    const float c = C[idx], s = INV ? Sn[idx] : -Sn[idx];
    return make_float2(d.x * c - d.y * s, d.x * s + d.y * c);
}

// In-register DFT of size R (<= 16): radix-2 decimation in frequency, then bit reversal.
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(float2 (&x)[R]) {
#pragma unroll
    for (int len = R; len >= 2; len >>= 1) {
        const int half = len >> 1;
#pragma unroll
        for (int s = 0; s < R; s += len) {
#pragma unroll
            for (int k = 0; k < half; k++) {
                const float2 a = x[s + k], b = x[s + k + half];
                x[s + k] = make_float2(a.x + b.x, a.y + b.y);
                x[s + k + half] = tw16<INV>(make_float2(a.x - b.x, a.y - b.y), k * (16 / len));
            }
        }
    }
    constexpr int LOGR = (R >= 16) ? 4 : (R >= 8) ? 3 : (R >= 4) ? 2 : (R >= 2) ? 1 : 0;
    float2 y[R];
#pragma unroll
    for (int k = 0; k < R; k++) y[k] = x[brevn(k, LOGR)];
#pragma unroll
    for (int k = 0; k < R; k++) x[k] = y[k];
}

// CTA barrier of the FFT stages: NBAR = 0 -> __syncthreads(); NBAR > 0 -> named barrier 1 over the
// first NBAR threads (a subset of the CTA runs the transforms: k_rhs_r2c)
template <int NBAR>
__device__ __forceinline__ void fft_bar() {
    if constexpr (NBAR == 0) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"n"(NBAR) : "memory");
}

// Stockham stages of an N-point FFT (N = 2^LOGN) by T = N/E threads, thread t.
// On entry of the first stage v[u] = x[t + u T]; on exit v[u] = X[t + u T].
// sm: this transform's padded float2 shared-memory row.  tw[m] = exp(-2 pi i m / N).
template <int LOGN, int LOGE, int LOGNS, bool INV, int NBAR = 0>
__device__ __forceinline__ void fft_stages(float2 (&v)[1 << LOGE], float2* __restrict__ sm, int t,
                                           const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, E = 1 << LOGE, T = N / E;
    constexpr int LOGR = (LOGN - LOGNS < LOGE) ? (LOGN - LOGNS) : LOGE;
    constexpr int R = 1 << LOGR, Q = E / R, NS = 1 << LOGNS;
    constexpr bool LAST = (LOGNS + LOGR == LOGN);
    if constexpr (LOGNS > 0) {
#pragma unroll
        for (int q = 0; q < Q; q++)
#pragma unroll
            for (int r = 0; r < R; r++) {
                SRSB_CHK(&sm[pad16(t + q * T + r * (N / R))], 8);
                v[q + r * Q] = sm[pad16(t + q * T + r * (N / R))];
            }
        fft_bar<NBAR>();
    }
#pragma unroll
    for (int q = 0; q < Q; q++) {
        const int j = t + q * T;
        const int k = j & (NS - 1);
        float2 x[R];
#pragma unroll
        for (int r = 0; r < R; r++) x[r] = v[q + r * Q];
        if constexpr (LOGNS > 0) {
            constexpr int STRIDE = N / (NS * R);
            float2 pw[LOGR];
#pragma unroll
            for (int bb = 0; bb < LOGR; bb++) {
                const float2 w = __ldg(&tw[(k * STRIDE) << bb]);
                pw[bb] = INV ? conjf2(w) : w;
            }
#pragma unroll
            for (int r = 1; r < R; r++) {
                float2 w = make_float2(1.f, 0.f);
                bool first = true;
#pragma unroll
                for (int bb = 0; bb < LOGR; bb++)
                    if ((r >> bb) & 1) {
                        w = first ? pw[bb] : cmul(w, pw[bb]);
                        first = false;
                    }
                x[r] = cmul(x[r], w);
            }
        }
        dft_reg<R, INV>(x);
        if constexpr (LAST) {
#pragma unroll
            for (int r = 0; r < R; r++) v[q + r * Q] = x[r];
        } else {
            const int base = (j >> LOGNS) * (NS * R) + k;
#pragma unroll
            for (int r = 0; r < R; r++) {
                SRSB_CHK(&sm[pad16(base + r * NS)], 8);
                sm[pad16(base + r * NS)] = x[r];
            }
        }
    }
    if constexpr (!LAST) {
        fft_bar<NBAR>();
        fft_stages<LOGN, LOGE, LOGNS + LOGR, INV, NBAR>(v, sm, t, tw);
    }
}

struct FftRowArgs {
    long long plane;  // elements per image plane of the real fields (ghost rows included)
    int M;          // rows per image (local rows of the slab)
    int lg_rpc;     // log2 rows per CTA
    int lg_G;       // log2 column-group interleave of the spectrum
    int SR;         // float2 per shared row, padded
    float clip;     // c2r only: > 0 clamps the output to [-clip, clip]
    int accum;      // c2r only: 1 -> phi = phi + z (increment form), 0 -> phi = z
    double* stats;  // c2r monitor: per-CTA partials [image][CTA][sum (phi_new - phi_old)^2, sum phi_old^2]
                    // of this sweep (null = off); k_reduce_partials sums them per image
    int stats_stride;
};

// Row pass 1: F rows (N = 2H reals) -> transposed packed half spectrum.
template <int LOGH, int LOGE, int LRPC = -1, int LG = -1>
__global__ void __launch_bounds__((LRPC >= 0 && (((1 << LOGH) >> LOGE) << (LRPC >= 0 ? LRPC : 0)) > 512) ? 1024 : 512)
k_rows_r2c(const float* __restrict__ F, float2* __restrict__ spec,
                                                   const float2* __restrict__ twH,
                                                   const float2* __restrict__ twR, FftRowArgs a) {
    constexpr int H = 1 << LOGH, E = 1 << LOGE, T = H / E;
    extern __shared__ float2 smem2[];
    const int tid = threadIdx.x;
    const int grp = tid / T, t = tid % T;
    // LRPC / LG >= 0: rows per CTA and column interleave fixed at compile time (the launch shapes of the
    // measured configs), so the transposed addressing folds into immediate offsets
    const int lg_rpc = LRPC >= 0 ? LRPC : a.lg_rpc, lg_G = LG >= 0 ? LG : a.lg_G;
    const int rpc = 1 << lg_rpc, G = 1 << lg_G;
    const int nthr = LRPC >= 0 ? (T << LRPC) : (int)blockDim.x;   // = blockDim.x
    const int b = blockIdx.y, m0 = blockIdx.x * rpc;
    float2* sm = smem2 + grp * a.SR;
    if ((SRSB_FFT_PF & 1) && tid == 0) {
        int bx, by;
        if (block_ahead_2d(SRSB_R2C_PF_DIST, bx, by))
            bulk_prefetch_l2(F + by * a.plane + (long long)(bx * rpc) * (2 * H), (uint32_t)(rpc * 2 * H * 4));
    }
    const float2* x = reinterpret_cast<const float2*>(F + b * a.plane + (long long)(m0 + grp) * (2 * H));
    float2 v[E];
#pragma unroll
    for (int u = 0; u < E; u++) v[u] = __ldcs(x + t + u * T);
    fft_stages<LOGH, LOGE, 0, false>(v, sm, t, twH);
    if constexpr (SRSB_R2C_SHFL && LG == LOGH && LRPC >= 0 && T == 32 && E == 16) {
        // row-major spectrum, one warp per row (H = 512): thread t holds Z[t + 32 u]; the split partner
        // Z[H - k] of k = t + 32 u sits in lane (32 - t) % 32 at index 15 - u (lane 0: its own index 16 - u), so
        // the split needs no shared-memory round trip and no barrier.  Same operands, same operations as the
        // shared-memory split: bitwise equal.
        float2* o = spec + (size_t)b * H * a.M + (size_t)(m0 + grp) * H;
        const int src = (32 - t) & 31;
#pragma unroll
        for (int u = 0; u < E; u++) {
            const float2 mine = v[15 - u];
            float2 part = make_float2(__shfl_sync(0xffffffffu, mine.x, src), __shfl_sync(0xffffffffu, mine.y, src));
            if (t == 0) part = v[(16 - u) & 15];
            const int k = t + 32 * u;
            const float2 tw = __ldg(&twR[k]);
            float2 X;
            if (u == 0 && t == 0) {
                X = make_float2(v[0].x + v[0].y, v[0].x - v[0].y);   // (X[0], X[N/2]) packed
            } else {
                const float2 Zc = conjf2(part);
                const float2 Ev = make_float2(0.5f * (v[u].x + Zc.x), 0.5f * (v[u].y + Zc.y));
                const float2 D = make_float2(0.5f * (v[u].x - Zc.x), 0.5f * (v[u].y - Zc.y));
                const float2 O = make_float2(D.y, -D.x);  // -i D
                const float2 wo = cmul(tw, O);
                X = make_float2(Ev.x + wo.x, Ev.y + wo.y);
            }
            o[k] = X;
        }
        return;
    }
#pragma unroll
    for (int u = 0; u < E; u++) sm[pad16(t + u * T)] = v[u];
    __syncthreads();
    float2* out = spec + (size_t)b * H * a.M;
    // real-FFT split of bin k2 of shared row rr
    auto split = [&](int rr, int k2) -> float2 {
        const float2* row = smem2 + rr * a.SR;
        const float2 Zk = row[pad16(k2)];
        const float2 Zc = conjf2(row[pad16((H - k2) & (H - 1))]);
        if (k2 == 0) return make_float2(Zk.x + Zk.y, Zk.x - Zk.y);  // (X[0], X[N/2]) packed
        const float2 Ev = make_float2(0.5f * (Zk.x + Zc.x), 0.5f * (Zk.y + Zc.y));
        const float2 D = make_float2(0.5f * (Zk.x - Zc.x), 0.5f * (Zk.y - Zc.y));
        const float2 O = make_float2(D.y, -D.x);  // -i D
        const float2 wo = cmul(__ldg(&twR[k2]), O);
        return make_float2(Ev.x + wo.x, Ev.y + wo.y);
    };
    auto split2 = [&](float2 Za, float2 Zb, float2 tw) -> float2 {   // Zb = Z[H - k]
        const float2 Zc = conjf2(Zb);
        const float2 Ev = make_float2(0.5f * (Za.x + Zc.x), 0.5f * (Za.y + Zc.y));
        const float2 D = make_float2(0.5f * (Za.x - Zc.x), 0.5f * (Za.y - Zc.y));
        const float2 O = make_float2(D.y, -D.x);  // -i D
        const float2 wo = cmul(tw, O);
        return make_float2(Ev.x + wo.x, Ev.y + wo.y);
    };
    if constexpr (LG == LOGH && LRPC >= 0 && E >= 2 && LOGH >= 1) {
        // row-major spectrum (G = H): row m0 + rr is H contiguous complex.  Bins k2 and H - k2 from the same two
        // shared reads (the split of one is the split of the other with the operands swapped); consecutive
        // lanes store consecutive (k2) and reverse-consecutive (H - k2) bins: whole lines.  k2 = 0 emits the
        // packed (X[0], X[N/2]) slot and the self-mirrored bin H / 2.
        constexpr int LHH = LOGH - 1;
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            const int e = tid + u * nthr;
            const int k2 = e & ((1 << LHH) - 1), rr = e >> LHH;   // k2 in [0, H/2)
            const float2* r0 = smem2 + rr * a.SR;
            float2* o = out + (size_t)(m0 + rr) * H;
            if (k2 == 0) {
                const float2 A0 = r0[0], B0 = r0[pad16(H / 2)];
                o[0] = make_float2(A0.x + A0.y, A0.x - A0.y);
                o[H / 2] = split2(B0, B0, __ldg(&twR[H / 2]));
            } else {
                const float2 A0 = r0[pad16(k2)], B0 = r0[pad16(H - k2)];
                o[k2] = split2(A0, B0, __ldg(&twR[k2]));
                o[H - k2] = split2(B0, A0, __ldg(&twR[H - k2]));
            }
        }
    } else if constexpr (LG == 0 && LRPC >= 1 && E >= 4 && SRSB_R2C_MIRROR) {
        // contiguous columns, bins k2 and H - k2 from the same two shared reads per row (the split of
        // one is the split of the other with the operands swapped); rows 2 rp, 2 rp + 1 of a bin are
        // adjacent -> 16-byte stores.  k2 = 0 also emits the self-mirrored bin H / 2.
        constexpr int LRP = LRPC - 1;
#pragma unroll
        for (int u = 0; u < E / 4; u++) {
            const int e = tid + u * nthr;
            const int rp = e & ((1 << LRP) - 1), k2 = e >> LRP;   // k2 in [0, H/2)
            const float2* r0 = smem2 + (2 * rp) * a.SR;
            const float2* r1 = r0 + a.SR;
            float2 X0, X1, Y0, Y1;   // bin k2 (X) and bin H - k2 (Y; H/2 when k2 = 0)
            if (k2 == 0) {
                const float2 A0 = r0[0], A1 = r1[0];
                X0 = make_float2(A0.x + A0.y, A0.x - A0.y);  // (X[0], X[N/2]) packed
                X1 = make_float2(A1.x + A1.y, A1.x - A1.y);
                const float2 th = __ldg(&twR[H / 2]);
                const float2 B0 = r0[pad16(H / 2)], B1 = r1[pad16(H / 2)];
                Y0 = split2(B0, B0, th);
                Y1 = split2(B1, B1, th);
            } else {
                const float2 t1 = __ldg(&twR[k2]), t2 = __ldg(&twR[H - k2]);
                const float2 A0 = r0[pad16(k2)], B0 = r0[pad16(H - k2)];
                const float2 A1 = r1[pad16(k2)], B1 = r1[pad16(H - k2)];
                X0 = split2(A0, B0, t1);
                X1 = split2(A1, B1, t1);
                Y0 = split2(B0, A0, t2);
                Y1 = split2(B1, A1, t2);
            }
            const int k2m = k2 == 0 ? H / 2 : H - k2;
            *reinterpret_cast<float4*>(out + (size_t)k2 * a.M + m0 + 2 * rp) = make_float4(X0.x, X0.y, X1.x, X1.y);
            *reinterpret_cast<float4*>(out + (size_t)k2m * a.M + m0 + 2 * rp) = make_float4(Y0.x, Y0.y, Y1.x, Y1.y);
        }
    } else if constexpr (LG == 0 && LRPC >= 1) {
        // contiguous columns: rows 2 rp, 2 rp + 1 of bin k2 are adjacent -> one 16-byte store per pair
        constexpr int LRP = LRPC - 1;
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            const int e = tid + u * nthr;
            const int rp = e & ((1 << LRP) - 1), k2 = e >> LRP;
            const float2 X0 = split(2 * rp, k2), X1 = split(2 * rp + 1, k2);
            *reinterpret_cast<float4*>(out + (size_t)k2 * a.M + m0 + 2 * rp) = make_float4(X0.x, X0.y, X1.x, X1.y);
        }
    } else {
#pragma unroll
        for (int u = 0; u < E; u++) {
            const int e = tid + u * nthr;   // blockDim = rpc * T: exactly E elements per thread
            const int kk = e & (G - 1);
            const int rr = (e >> lg_G) & (rpc - 1);
            const int kg = e >> (lg_G + lg_rpc);
            const int k2 = (kg << lg_G) + kk;
            out[(((size_t)kg * a.M + m0 + rr) << lg_G) + kk] = split(rr, k2);
        }
    }
}

// Column element m of local spectrum column k2l (group kg = k2l / G, lane cc = k2l % G) lives at
//   b * bstride + (m >> lg_seg) * seg_stride + ((kg * 2^lg_seg + m % 2^lg_seg) * G + cc)
// i.e. the column is split into segments of 2^lg_seg rows (the slabs' row blocks after the
// all-to-all; one segment = the whole column for a single-GPU image).
struct FftColArgs {
    int H;          // N/2: global spectrum columns (cN[H] is the k2 = N/2 symbol term)
    int lg_G;       // layout interleave (columns per group)
    int lg_cpc;     // columns per CTA (a multiple of G)
    int SC;         // float2 per shared row, padded
    float taumu;    // tau * mu
    float scale;    // 1 / (M H), global M
    int lg_seg;     // log2 rows per segment (power of two)
    long long seg_stride;  // complex elements between segments
    long long bstride;     // complex elements between images
    int k2_off;     // global index of local column 0 (slab: rank * H / P)
    const float* sym;   // [H + 1][M] table of scale / symbol(k1, k2), fp64-computed and rounded once
                        // (L2-resident, shared by the batch); null: sym_scale
};

// scale / symbol(k1, k2).  SYMT: from the table (staged into shared memory at the kernel start by
// sym_stage, so its L2 latency hides behind the forward FFT); else the correctly rounded reciprocal of
// the fp32 symbol.
template <bool SYMT>
__device__ __forceinline__ float sym_at(const FftColArgs& a, const float* __restrict__ cM, const float* st, int k1,
                                        float ck) {
    if constexpr (SYMT) return st[k1];
    else return sym_scale(a.scale, a.taumu, __ldg(&cM[k1]), ck);
}
// cp.async (4-byte, L1-bypassing where possible) of this thread's E table entries of column k2 into st
template <int E, int T>
__device__ __forceinline__ void sym_stage(const FftColArgs& a, int M, int k2, int t, float* st) {
#pragma unroll
    for (int u = 0; u < E; u++) {
        const int k1 = t + u * T;
        SRSB_CHK(st + k1, 4);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(st + k1)),
                     "l"(a.sym + (size_t)k2 * M + k1) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void sym_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Column pass: forward FFT, divide by the symbol, inverse FFT, in place.  Threads of one column
// are consecutive (t fastest), so a warp works inside one transform.
// CONTIG: whole-image layout with G = 1 (one segment, each column M contiguous complex): element m
// is col[m], so the E loads and stores use immediate offsets from one base pointer.
template <int LOGM, int LOGE, bool CONTIG, bool SYMT>
__global__ void __maxnreg__(LOGM >= 12 ? SRSB_COLS_MAXNREG_BIG : SRSB_COLS_MAXNREG) k_cols_solve(float2* __restrict__ spec, const float2* __restrict__ twM,
                                                       const float* __restrict__ cM, const float* __restrict__ cN,
                                                       FftColArgs a) {
    constexpr int M = 1 << LOGM, E = 1 << LOGE, T = M / E;
    extern __shared__ float2 smem2[];
    const int G = 1 << a.lg_G;
    const int tid = threadIdx.x;
    const int t = tid % T, cl = tid / T;                 // cl: column within the CTA
    const int k2l = (blockIdx.x << a.lg_cpc) + cl;        // local spectrum column
    const int k2 = a.k2_off + k2l;                         // global spectrum column
    const int b = blockIdx.y;
    const int kg = k2l >> a.lg_G, cc = k2l & (G - 1);
    float2* base = spec + b * a.bstride + cc;
    float2* sm = smem2 + cl * a.SC;
    // SYMT: this column's scale / symbol entries, staged behind the exchange rows of the CTA's columns
    float* st = reinterpret_cast<float*>(smem2 + (blockDim.x / T) * a.SC) + cl * M;
    if constexpr (SYMT) sym_stage<E, T>(a, M, k2, t, st);
    // element m of the column (recomputed at the store: holding E 64-bit addresses across both FFTs
    // cost 32 registers)
    auto addr = [&](int m) -> long long {
        const int s = m >> a.lg_seg, mr = m & ((1 << a.lg_seg) - 1);
        return s * a.seg_stride + ((long long)((kg << a.lg_seg) + mr) << a.lg_G);
    };
    float2* col = spec + b * a.bstride + ((long long)k2l << LOGM);   // CONTIG only
    if (CONTIG && (SRSB_FFT_PF & 2) && tid == 0) {
        int bx, by;
        if (block_ahead_2d(SRSB_COLS_PF_DIST, bx, by))
            bulk_prefetch_l2(spec + by * a.bstride + ((long long)(bx << a.lg_cpc) << LOGM),
                             (uint32_t)((M << a.lg_cpc) * sizeof(float2)));
    }
    float2 v[E];
#pragma unroll
    for (int u = 0; u < E; u++) v[u] = CONTIG ? col[t + u * T] : base[addr(t + u * T)];
    fft_stages<LOGM, LOGE, 0, false>(v, sm, t, twM);
    if constexpr (SYMT) sym_wait();
    if (blockIdx.x == 0 && a.k2_off == 0) {  // CTA-uniform: slot 0 packs the real columns k2 = 0, N/2
#pragma unroll
        for (int u = 0; u < E; u++) sm[pad16(t + u * T)] = v[u];
        __syncthreads();
        if (k2 == 0) {
            const float c0 = __ldg(&cN[0]), ch = __ldg(&cN[a.H]);
#pragma unroll
            for (int u = 0; u < E; u++) {
                const int k1 = t + u * T;
                const float2 C = v[u];
                const float2 Cc = conjf2(sm[pad16((M - k1) & (M - 1))]);
                const float s0 = sym_at<SYMT>(a, cM, st, k1, c0);
                const float sh = SYMT ? __ldg(&a.sym[(size_t)a.H * M + k1]) : sym_at<false>(a, cM, st, k1, ch);
                const float p = 0.5f * (s0 + sh), m = 0.5f * (s0 - sh);
                v[u] = make_float2(p * C.x + m * Cc.x, p * C.y + m * Cc.y);
            }
        } else {
            const float ck = __ldg(&cN[k2]);
#pragma unroll
            for (int u = 0; u < E; u++) {
                const float s = sym_at<SYMT>(a, cM, st, t + u * T, ck);
                v[u] = make_float2(v[u].x * s, v[u].y * s);
            }
        }
        __syncthreads();
    } else {
        const float ck = SYMT ? 0.f : __ldg(&cN[k2]);
#pragma unroll
        for (int u = 0; u < E; u++) {
            const float s = sym_at<SYMT>(a, cM, st, t + u * T, ck);
            v[u] = make_float2(v[u].x * s, v[u].y * s);
        }
    }
    fft_stages<LOGM, LOGE, 0, true>(v, sm, t, twM);
#pragma unroll
    for (int u = 0; u < E; u++) {
        if (CONTIG) col[t + u * T] = v[u];
        else base[addr(t + u * T)] = v[u];
    }
}

// Persistent column solve for long contiguous columns (M >= 4096, G = 1, whole-image contexts):
// such a column needs a 256 / 512-thread CTA and only one fits per SM without spilling, so
// nothing overlaps its load with its transforms.  Here each CTA strides over the columns and one
// elected thread fetches the next column into a second shared buffer with a bulk async copy
// (cp.async.bulk on an mbarrier) while the current one is transformed.  Same arithmetic as
// k_cols_solve.
template <int LOGM, int LOGE, bool SYMT>
__global__ void __launch_bounds__(512, 1) k_cols_solve_p(float2* __restrict__ spec, const float2* __restrict__ twM,
                                                         const float* __restrict__ cM, const float* __restrict__ cN,
                                                         FftColArgs a, int ncols, int lg_hl) {
    constexpr int M = 1 << LOGM, E = 1 << LOGE, T = M / E;
    constexpr uint32_t BYTES = M * sizeof(float2);
    extern __shared__ float4 smem_cp[];
    float2* buf = reinterpret_cast<float2*>(smem_cp);      // [M] prefetch buffer (dense)
    float2* sm = buf + M;                                   // padded exchange row (SC)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + a.SC);
    const int t = threadIdx.x;
    const int hl = 1 << lg_hl;
    auto col_ptr = [&](int c) { return spec + (long long)(c >> lg_hl) * a.bstride + (long long)(c & (hl - 1)) * M; };
    int c = blockIdx.x;
    if (t == 0) mbar_init(bar, 1);
    __syncthreads();
    if (t == 0 && c < ncols) {
        mbar_expect_tx(bar, BYTES);
        bulk_load(buf, col_ptr(c), BYTES, bar);
    }
    for (int it = 0; c < ncols; c += gridDim.x, it++) {
        mbar_wait(bar, it & 1);
        float2 v[E];
#pragma unroll
        for (int u = 0; u < E; u++) v[u] = buf[t + u * T];
        __syncthreads();   // buf consumed: prefetch the next column while this one is transformed
        if (t == 0 && c + (int)gridDim.x < ncols) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, BYTES);
            bulk_load(buf, col_ptr(c + gridDim.x), BYTES, bar);
        }
        fft_stages<LOGM, LOGE, 0, false>(v, sm, t, twM);
        const int k2 = c & (hl - 1);
        if (k2 == 0) {   // slot 0 packs the real columns k2 = 0 and N/2 (iteration-uniform)
#pragma unroll
            for (int u = 0; u < E; u++) sm[pad16(t + u * T)] = v[u];
            __syncthreads();
            const float c0 = __ldg(&cN[0]), ch = __ldg(&cN[a.H]);
#pragma unroll
            for (int u = 0; u < E; u++) {
                const int k1 = t + u * T;
                const float2 C = v[u];
                const float2 Cc = conjf2(sm[pad16((M - k1) & (M - 1))]);
                const float s0 = SYMT ? __ldg(&a.sym[k1]) : sym_at<false>(a, cM, nullptr, k1, c0);
                const float sh = SYMT ? __ldg(&a.sym[(size_t)a.H * M + k1]) : sym_at<false>(a, cM, nullptr, k1, ch);
                const float pp = 0.5f * (s0 + sh), mm = 0.5f * (s0 - sh);
                v[u] = make_float2(pp * C.x + mm * Cc.x, pp * C.y + mm * Cc.y);
            }
            __syncthreads();
        } else {
            const float ck = __ldg(&cN[k2]);
#pragma unroll
            for (int u = 0; u < E; u++) {
                const float sc = SYMT ? __ldg(&a.sym[(size_t)k2 * M + t + u * T]) : sym_at<false>(a, cM, nullptr, t + u * T, ck);
                v[u] = make_float2(v[u].x * sc, v[u].y * sc);
            }
        }
        fft_stages<LOGM, LOGE, 0, true>(v, sm, t, twM);
        float2* out = col_ptr(c);
#pragma unroll
        for (int u = 0; u < E; u++) out[t + u * T] = v[u];
        __syncthreads();   // the exchange row is free for the next column
    }
}

// Batched in-place complex FFT of contiguous lines of M = 2^LOGM values (3-D solve: the i axis of every
// (k2, z) line of the transposed spectrum, sr_vol.cuh).  grid = lines / cpc, block cpc * M / E threads,
// dynamic shared memory cpc * SC float2; unnormalised, forward exp(-i) / inverse exp(+i).
template <int LOGM, int LOGE, bool INV>
__global__ void __launch_bounds__(512) k_lines_fft(float2* __restrict__ data, const float2* __restrict__ twM, int lg_cpc, int SC) {
    constexpr int M = 1 << LOGM, E = 1 << LOGE, T = M / E;
    extern __shared__ float2 smem2[];
    const int t = threadIdx.x % T, cl = threadIdx.x / T;
    float2* line = data + ((size_t)((blockIdx.x << lg_cpc) + cl) << LOGM);
    float2* sm = smem2 + cl * SC;
    float2 v[E];
#pragma unroll
    for (int u = 0; u < E; u++) v[u] = line[t + u * T];
    fft_stages<LOGM, LOGE, 0, INV>(v, sm, t, twM);
#pragma unroll
    for (int u = 0; u < E; u++) line[t + u * T] = v[u];
}

// NEXT-1 monitor partials of the c2r pass, out of line so the (untaken, monitor-off) branch costs the hot
// row transform no registers
static __device__ __noinline__ void c2r_partials(float dsum, float osum, double* dst) {
    const float pv[2] = {dsum, osum};
    block_partials<2>(pv, dst);
}

#define H_OF(L) (1 << (L))
// Row pass 2: transposed half spectrum -> inverse real FFT -> phi rows (accumulated, clamped).
#ifndef SRSB_C2R_MINB
#define SRSB_C2R_MINB (SRSB_C2R_OLD_SMEM ? 3 : 2)   // resident CTAs per SM asked of ptxas for the <= 256-thread
                                                   // launch-shape instances (2 caps them at 128 registers: without
                                                   // a cap the monitor reduction let ptxas take 153)
#endif
#ifndef SRSB_C2R_MINB_BIG
#define SRSB_C2R_MINB_BIG 1 // the same for the 512-thread instances (H = 4096: C5)
#endif
#ifndef SRSB_C2R_LATE_OLD
#define SRSB_C2R_LATE_OLD 0 // 1: fetch the accumulation source after the FFT (fewer live registers)
#endif
#ifndef SRSB_C2R_OLD_SMEM
#define SRSB_C2R_OLD_SMEM 0 // 1: the launch-shape instances stage the accumulation source (psi) into shared memory
                            // with cp.async at their start instead of holding it in 32 registers through the FFT
                            // (the host then adds rpc * 2H floats of dynamic shared memory to the c2r launch).
                            // Measured on C3: 0.258 ms per launch (78 registers, 3 CTAs / SM) against 0.189 ms
                            // with psi in registers (128 registers, 2 CTAs / SM): off
#endif
#ifndef SRSB_C2R_SHFL
#define SRSB_C2R_SHFL 1     // the row-major H = 512 instances (one warp per row) load their row straight into registers and
                            // get the mirrored bins by warp shuffles (no shared-memory gather): C3 c2r 0.146 -> 0.139 ms,
                            // bitwise equal to the gather (tools/solve_hash.py)
#endif
#ifndef SRSB_C2R_SHFL_LATE
#define SRSB_C2R_SHFL_LATE 0   // 1: the warp-shuffle c2r instances load the accumulation source after the FFT, L2-prefetched at
                               // their start (the combination measured faster on C3 and slower on C5 before the shuffle split)
#endif
#ifndef SRSB_C2R_OWN_PF
#define SRSB_C2R_OWN_PF 0   // 1: L2 bulk prefetch of the CTA's own psi rows at its start (with SRSB_C2R_LATE_OLD=1: the
                            // accumulation source is then loaded after the FFT, 32 registers fewer across it)
#endif
template <int LOGH, int LOGE, int LRPC = -1, int LG = -1>
__global__ void __launch_bounds__(LRPC >= 0 ? ((H_OF(LOGH) / (1 << LOGE)) << (LRPC >= 0 ? LRPC : 0)) : 512,
                                  (LRPC >= 0 && ((H_OF(LOGH) / (1 << LOGE)) << (LRPC >= 0 ? LRPC : 0)) <= 256) ? SRSB_C2R_MINB
                                  : (LRPC >= 0 ? SRSB_C2R_MINB_BIG : 1))
k_rows_c2r(const float2* __restrict__ spec, float* __restrict__ phi,
                                                   const float2* __restrict__ twH,
                                                   const float2* __restrict__ twR, FftRowArgs a) {
    constexpr int H = 1 << LOGH, E = 1 << LOGE, T = H / E;
    extern __shared__ float2 smem2[];
    const int tid = threadIdx.x;
    const int grp = tid / T, t = tid % T;
    // LRPC / LG >= 0: rows per CTA and column interleave fixed at compile time (the launch shapes of the
    // measured configs), so the transposed addressing folds into immediate offsets
    const int lg_rpc = LRPC >= 0 ? LRPC : a.lg_rpc, lg_G = LG >= 0 ? LG : a.lg_G;
    const int rpc = 1 << lg_rpc, G = 1 << lg_G;
    const int nthr = LRPC >= 0 ? (T << LRPC) : (int)blockDim.x;   // = blockDim.x
    const int b = blockIdx.y, m0 = blockIdx.x * rpc;
    const float2* in = spec + (size_t)b * H * a.M;
    float2* out = reinterpret_cast<float2*>(phi + b * a.plane + (long long)(m0 + grp) * (2 * H));
    if ((SRSB_FFT_PF & 4) && a.accum && tid == 0) {
        int bx, by;
        if (block_ahead_2d(SRSB_C2R_PF_DIST, bx, by))
            bulk_prefetch_l2(phi + by * a.plane + (long long)(bx * rpc) * (2 * H), (uint32_t)(rpc * 2 * H * 4));
    }
    // the warp-shuffle instances may take the late + prefetched accumulation source on their own (SRSB_C2R_SHFL_LATE)
    constexpr bool SHFLI = SRSB_C2R_SHFL && LG == LOGH && LRPC >= 0 && H_OF(LOGH) / (1 << LOGE) == 32 && (1 << LOGE) == 16;
    constexpr bool LATE = SRSB_C2R_LATE_OLD || (SRSB_C2R_SHFL_LATE && SHFLI);
    constexpr bool OWNPF = SRSB_C2R_OWN_PF || (SRSB_C2R_SHFL_LATE && SHFLI);
    if (OWNPF && a.accum && t == 0) bulk_prefetch_l2(out, (uint32_t)(2 * H * 4));
    // accumulation source (phi of the previous sweep), fetched first: its latency hides behind the FFT.
    // OSM: into shared memory by cp.async (no registers held across the FFT), else into registers
    constexpr bool OSM = SRSB_C2R_OLD_SMEM && LRPC >= 0 && !LATE;
    float2* old_sm = smem2 + (size_t)rpc * a.SR + (size_t)grp * H;
    float2 old[E];
    if (OSM && a.accum) {
#pragma unroll
        for (int u = 0; u < E; u++)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(old_sm + t + u * T)),
                         "l"(out + t + u * T) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    } else if (!LATE && a.accum) {
#pragma unroll
        for (int u = 0; u < E; u++) old[u] = out[t + u * T];
    }
    float2* sm = smem2 + grp * a.SR;
    float2 v[E];
    if constexpr (SRSB_C2R_SHFL && LG == LOGH && LRPC >= 0 && H_OF(LOGH) / (1 << LOGE) == 32 && (1 << LOGE) == 16) {
        // row-major spectrum, one warp per row (H = 512): thread t loads X[t + 32 u] (coalesced) and gets the partner
        // X[H - k] of k = t + 32 u from lane (32 - t) % 32, index 15 - u (lane 0: its own index 16 - u) by warp
        // shuffles: no shared-memory staging, no barrier before the FFT.  Same operands and operations: bitwise equal.
        const float2* xr = in + (size_t)(m0 + grp) * H;
        float2 x[E];
#pragma unroll
        for (int u = 0; u < E; u++) x[u] = __ldcs(xr + t + 32 * u);
        const int src = (32 - t) & 31;
#pragma unroll
        for (int u = 0; u < E; u++) {
            const float2 mine = x[15 - u];
            float2 part = make_float2(__shfl_sync(0xffffffffu, mine.x, src), __shfl_sync(0xffffffffu, mine.y, src));
            if (t == 0) part = x[(16 - u) & 15];
            const float2 X = x[u];
            if (u == 0 && t == 0) {
                v[u] = make_float2(0.5f * (X.x + X.y), 0.5f * (X.x - X.y));
            } else {
                const float2 Xc = conjf2(part);
                const float2 Ev = make_float2(0.5f * (X.x + Xc.x), 0.5f * (X.y + Xc.y));
                const float2 D = make_float2(0.5f * (X.x - Xc.x), 0.5f * (X.y - Xc.y));
                const float2 O = cmul(conjf2(__ldg(&twR[t + 32 * u])), D);  // W^{-k} D
                v[u] = make_float2(Ev.x - O.y, Ev.y + O.x);                 // E + i O
            }
        }
    } else {
    // transposed gather: blockDim = rpc * T threads, rpc * H elements -> exactly E per thread;
    // all E loads are issued before the shared stores
    if constexpr (LG == LOGH && LRPC >= 0 && E >= 2 && LOGH >= 1) {
        // row-major spectrum (G = H): row m0 + rr is H contiguous complex -> 16-byte loads of two adjacent bins
        constexpr int LHH = LOGH - 1;
        float4 tmp[E / 2];
        int sidx[E / 2];
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            const int e = tid + u * nthr;
            const int k2 = 2 * (e & ((1 << LHH) - 1)), rr = e >> LHH;
            tmp[u] = __ldcs(reinterpret_cast<const float4*>(in + (size_t)(m0 + rr) * H + k2));
            sidx[u] = rr * a.SR + pad16(k2);
        }
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            SRSB_CHK(&smem2[sidx[u] + 1], 8);
            smem2[sidx[u]] = make_float2(tmp[u].x, tmp[u].y);
            smem2[sidx[u] + 1] = make_float2(tmp[u].z, tmp[u].w);
        }
    } else if constexpr (LG == 0 && LRPC >= 1) {
        // contiguous columns: rows 2 rp, 2 rp + 1 of bin k2 are adjacent -> one 16-byte load per pair
        constexpr int LRP = LRPC - 1;
        float4 tmp[E / 2];
        int sidx[E / 2];
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            const int e = tid + u * nthr;
            const int rp = e & ((1 << LRP) - 1), k2 = e >> LRP;
            tmp[u] = __ldcs(reinterpret_cast<const float4*>(in + (size_t)k2 * a.M + m0 + 2 * rp));
            sidx[u] = 2 * rp * a.SR + pad16(k2);
        }
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            SRSB_CHK(&smem2[sidx[u] + a.SR], 8);
            smem2[sidx[u]] = make_float2(tmp[u].x, tmp[u].y);
            smem2[sidx[u] + a.SR] = make_float2(tmp[u].z, tmp[u].w);
        }
    } else {
        float2 tmp[E];
        int sidx[E];
#pragma unroll
        for (int u = 0; u < E; u++) {
            const int e = tid + u * nthr;
            const int kk = e & (G - 1);
            const int rr = (e >> lg_G) & (rpc - 1);
            const int kg = e >> (lg_G + lg_rpc);
            const int k2 = (kg << lg_G) + kk;
            tmp[u] = __ldcs(in + (((size_t)kg * a.M + m0 + rr) << lg_G) + kk);
            sidx[u] = rr * a.SR + pad16(k2);
        }
#pragma unroll
        for (int u = 0; u < E; u++) {
            SRSB_CHK(&smem2[sidx[u]], 8);
            smem2[sidx[u]] = tmp[u];
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < E; u++) {
        const int k = t + u * T;
        SRSB_CHK(&sm[pad16(k)], 8);
        if (k != 0) SRSB_CHK(&sm[pad16(H - k)], 8);
        const float2 X = sm[pad16(k)];
        if (k == 0) {
            // X.x = X[0], X.y = X[N/2]: Z[0] = E[0] + i O[0], E = (X0 + Xh)/2, O = (X0 - Xh)/2
            v[u] = make_float2(0.5f * (X.x + X.y), 0.5f * (X.x - X.y));
        } else {
            const float2 Xc = conjf2(sm[pad16(H - k)]);
            const float2 Ev = make_float2(0.5f * (X.x + Xc.x), 0.5f * (X.y + Xc.y));
            const float2 D = make_float2(0.5f * (X.x - Xc.x), 0.5f * (X.y - Xc.y));
            const float2 O = cmul(conjf2(__ldg(&twR[k])), D);  // W^{-k} D
            v[u] = make_float2(Ev.x - O.y, Ev.y + O.x);        // E + i O
        }
    }
    __syncthreads();
    }
    fft_stages<LOGH, LOGE, 0, true>(v, sm, t, twH);
    if (LATE && a.accum) {
#pragma unroll
        for (int u = 0; u < E; u++) old[u] = out[t + u * T];
    }
    if (OSM && a.accum) {   // each thread reads back exactly the values it copied
        asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
        for (int u = 0; u < E; u++) old[u] = old_sm[t + u * T];
    }
    float dsum = 0.f, osum = 0.f;
#pragma unroll
    for (int u = 0; u < E; u++) {
        float2 z = v[u];
        if (a.accum) {
            z.x += old[u].x;
            z.y += old[u].y;
        }
        if (a.clip > 0.f) {
            z.x = fminf(fmaxf(z.x, -a.clip), a.clip);
            z.y = fminf(fmaxf(z.y, -a.clip), a.clip);
        }
        out[t + u * T] = z;
        if (a.stats && a.accum) {   // NEXT-1: ||phi^{s+1} - phi^s||^2 and ||phi^s||^2
            const float dx = z.x - old[u].x, dy = z.y - old[u].y;
            dsum += dx * dx + dy * dy;
            osum += old[u].x * old[u].x + old[u].y * old[u].y;
        }
    }
#ifdef SRSB_C2R_STATS_ATOMIC   // A/B reference only (nondeterministic sums)
    if (a.stats && a.accum) {
        atomicAdd(a.stats, (double)dsum);
        atomicAdd(a.stats + 1, (double)osum);
    }
#else
    if (a.stats && a.accum)   // this CTA's partial sums -> its slot (image-major), reduced in a fixed order
        c2r_partials(dsum, osum, a.stats + ((long long)b * gridDim.x + blockIdx.x) * 2);
#endif
}

}  // namespace srsb
