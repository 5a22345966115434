// sr_stencil.cuh -- halo-tiled stencil kernels of the Split Bregman SR iteration (sm_100a).
//
//   k_rhs   : F = Eq. (37) RHS, with the non-local vector v of P:368
//             computed from u = h_eps(phi) w over a disc (or square) window.
//   k_wb    : w/b update: B of Eq. (41), generalized shrink Eq. (42), projection
//             Eq. (40) (BALL / SPHERE / NONE, Q1), Bregman Eq. (23);
//             or one fixed-point sweep of Eq. (38)-(39).
//   k_blur_rows / k_blur_cols / k_edge_g : edge indicator Eq. (1) (one-time).
//   k_init_w: w = grad phi0 (Alg. 1 (1)), b = 0.
//
// Tiling: a CTA of 32 x BY threads owns a tile of (BY*RT) rows x (32*CT) columns;
// the R-halo of u = h(phi) w is staged in shared memory as float2 (out-of-image
// taps are 0: reading Q5).  Each thread accumulates v for an RT x CT block in
// registers from separable partial sums: v(x) = sum_p e_p S_{L_p}(x + (p, 0)),
// S_L(y) = sum_{|q| <= L} e_q u(y + (0, q)), e_q = exp(-q^2/d^2), L_p = the disc's
// row half-width -- an exact regrouping of the window sum (different rounding order).
#pragma once
#include <cuda_runtime.h>
#include "sr_f32x2.cuh"
#include "sr_tma.cuh"
#include "sr_reduce.cuh"

namespace srsb {

constexpr float kPi = 3.14159265358979323846f;


// ------------------------------------------------------------------ regularizers (Eq. 5, 6, 11, 28, 29)
// All of H(x +- l), delta(x +- l), delta(x), delta'(x) from ONE sincospif(x / eps): the arguments
// (x +- l)/eps differ by the constant l/eps, so sin/cos follow by angle addition with
// (sinpi(l/eps), cospi(l/eps)) precomputed in double on the host.  Branch conditions use x +- l.
struct Reg {
    float eps, inv_eps, l;
    float sl, cl;          // sinpi(l / eps), cospi(l / eps)
    int l_eq_eps;          // l == eps (the default reading Q22): closed forms below
};

// With l = eps and a = x / eps, Eq. (5), (6), (11), (28), (29) reduce on |a| < 2 to
//   h  = (2 - |a| + sinpi(|a|)/pi) / 2,           h' = -sign(a) (1 - cospi(a)) / (2 eps),
//   delta = (1 + cospi(a)) / (2 eps) [|a| <= 1],  delta' = -(pi / (2 eps^2)) sinpi(a) [|a| <= 1],
// and all four vanish for |a| >= 2 (only one of H(x +- l) is inside its band at a time).
__device__ __forceinline__ float H_of(float y, float s, const Reg& r) {   // Eq. (5), s = sinpi(y/eps)
    if (y > r.eps) return 1.f;
    if (y < -r.eps) return 0.f;
    return 0.5f * (1.f + y * r.inv_eps + s * (1.f / kPi));
}
__device__ __forceinline__ float d_of(float y, float c, const Reg& r) {   // Eq. (6), c = cospi(y/eps)
    return fabsf(y) > r.eps ? 0.f : (1.f + c) * (0.5f * r.inv_eps);
}

struct RegVals {
    float h, hp, d, dp;    // h(x) Eq. (11), h'(x) Eq. (28), delta(x) Eq. (6), delta'(x) Eq. (29)
};

template <bool LEQ>
__device__ __forceinline__ RegVals reg_all(float x, const Reg& r) {
    RegVals v;
    if constexpr (LEQ) {
        const float a = x * r.inv_eps, aa = fabsf(a);
        if (aa >= 2.f) {
            v.h = v.hp = v.d = v.dp = 0.f;
            return v;
        }
        float s, c;
        sincospif(a, &s, &c);
        const float sg = copysignf(1.f, a);
        v.h = 0.5f * (2.f - aa + sg * s * (1.f / kPi));
        v.hp = -sg * (1.f - c) * (0.5f * r.inv_eps);
        const bool in = aa <= 1.f;
        v.d = in ? (1.f + c) * (0.5f * r.inv_eps) : 0.f;
        v.dp = in ? -(0.5f * kPi) * r.inv_eps * r.inv_eps * s : 0.f;
        return v;
    }
    if (fabsf(x) >= r.l + r.eps && fabsf(x) > r.eps) {   // outside every band: all four vanish
        v.h = v.hp = v.d = v.dp = 0.f;
        return v;
    }
    float s, c;
    sincospif(x * r.inv_eps, &s, &c);
    const float sp = s * r.cl + c * r.sl, cp = c * r.cl - s * r.sl;   // at x + l
    const float sm = s * r.cl - c * r.sl, cm = c * r.cl + s * r.sl;   // at x - l
    const float yp = x + r.l, ym = x - r.l;
    const float Hp = H_of(yp, sp, r), Hm = H_of(ym, sm, r);
    const float dpl = d_of(yp, cp, r), dmi = d_of(ym, cm, r);
    v.h = Hp * (1.f - Hm);
    v.hp = dpl * (1.f - Hm) - Hp * dmi;
    const bool in = fabsf(x) <= r.eps;
    v.d = in ? (1.f + c) * (0.5f * r.inv_eps) : 0.f;
    v.dp = in ? -(0.5f * kPi) * r.inv_eps * r.inv_eps * s : 0.f;
    return v;
}

template <bool LEQ>
__device__ __forceinline__ float reg_h(float x, const Reg& r) {
    if constexpr (LEQ) {
        const float aa = fabsf(x * r.inv_eps);
        return aa >= 2.f ? 0.f : 0.5f * (2.f - aa + sinpif(aa) * (1.f / kPi));
    }
    // fast exits: h = 0 when |x| >= l + eps (both factors saturate)
    if (fabsf(x) >= r.l + r.eps) return 0.f;
    float s, c;
    sincospif(x * r.inv_eps, &s, &c);
    const float sp = s * r.cl + c * r.sl;
    const float sm = s * r.cl - c * r.sl;
    return H_of(x + r.l, sp, r) * (1.f - H_of(x - r.l, sm, r));
}

// h(x) and delta(x) from one sincospif (w/b update)
template <bool LEQ>
__device__ __forceinline__ void reg_hd(float x, const Reg& r, float& h, float& d) {
    if constexpr (LEQ) {
        const float a = x * r.inv_eps, aa = fabsf(a);
        if (aa >= 2.f) {
            h = d = 0.f;
            return;
        }
        float s, c;
        sincospif(aa, &s, &c);
        h = 0.5f * (2.f - aa + s * (1.f / kPi));
        d = aa <= 1.f ? (1.f + c) * (0.5f * r.inv_eps) : 0.f;
        return;
    }
    if (fabsf(x) >= r.l + r.eps && fabsf(x) > r.eps) {
        h = d = 0.f;
        return;
    }
    float s, c;
    sincospif(x * r.inv_eps, &s, &c);
    const float sp = s * r.cl + c * r.sl;
    const float sm = s * r.cl - c * r.sl;
    h = H_of(x + r.l, sp, r) * (1.f - H_of(x - r.l, sm, r));
    d = fabsf(x) <= r.eps ? (1.f + c) * (0.5f * r.inv_eps) : 0.f;
}

// Two adjacent pixels at once (f32x2 arithmetic around the per-lane sincospif), branch-free.
// h(x) for the u staging:
template <bool LEQ>
__device__ __forceinline__ float2 reg_h2(float2 x, const Reg& r) {
    if constexpr (LEQ) {
        const float2 a = mul2(x, f2(r.inv_eps));
        const float2 aa = make_float2(fabsf(a.x), fabsf(a.y));
        if (aa.x >= 2.f && aa.y >= 2.f) return f2(0.f);   // outside the band (most pixels: skip the sines)
        const float2 sv = make_float2(sinpif(aa.x), sinpif(aa.y));
        const float2 h = mul2(fma2(sv, f2(1.f / kPi), sub2(f2(2.f), aa)), f2(0.5f));
        return make_float2(aa.x >= 2.f ? 0.f : h.x, aa.y >= 2.f ? 0.f : h.y);
    }
    return make_float2(reg_h<false>(x.x, r), reg_h<false>(x.y, r));
}
// h'(x), delta(x), delta'(x) for the RHS:
template <bool LEQ>
__device__ __forceinline__ void reg_rhs2(float2 x, const Reg& r, float2& hp, float2& d, float2& dp) {
    if constexpr (LEQ) {
        const float2 a = mul2(x, f2(r.inv_eps));
        if (fabsf(a.x) >= 2.f && fabsf(a.y) >= 2.f) {   // outside the band: all three vanish
            hp = d = dp = f2(0.f);
            return;
        }
        float2 sv, cv;
        sincospif(a.x, &sv.x, &cv.x);
        sincospif(a.y, &sv.y, &cv.y);
        const float k = 0.5f * r.inv_eps;
        const float2 hpm = mul2(sub2(f2(1.f), cv), f2(k));          // (1 - cospi a) k >= 0
        const float2 dm = fma2(cv, f2(k), f2(k));                    // (1 + cospi a) k
        const float2 dpm = mul2(sv, f2(-(0.5f * kPi) * r.inv_eps * r.inv_eps));
        const float ax = fabsf(a.x), ay = fabsf(a.y);
        hp = make_float2(ax >= 2.f ? 0.f : copysignf(hpm.x, -a.x), ay >= 2.f ? 0.f : copysignf(hpm.y, -a.y));
        d = make_float2(ax <= 1.f ? dm.x : 0.f, ay <= 1.f ? dm.y : 0.f);
        dp = make_float2(ax <= 1.f ? dpm.x : 0.f, ay <= 1.f ? dpm.y : 0.f);
        return;
    }
    const RegVals v0 = reg_all<false>(x.x, r), v1 = reg_all<false>(x.y, r);
    hp = make_float2(v0.hp, v1.hp);
    d = make_float2(v0.d, v1.d);
    dp = make_float2(v0.dp, v1.dp);
}

__host__ __device__ constexpr int isqrt_c(int v) {
    int r = 0;
    while ((r + 1) * (r + 1) <= v) r++;
    return r;
}
// Row half-width of the window at row offset p: disc floor(sqrt(R^2 - p^2)), square R.
template <int R, int SHAPE>
__host__ __device__ constexpr int half_width(int p) {
    return SHAPE == 0 ? isqrt_c(R * R - p * p) : R;
}

// Field layout (all kernels): pointers address local row 0 of image 0; image b, local row i
// (-gh <= i < M + gh: gh ghost rows above and below, filled by the slab halo exchange) is at
// p + b * plane + i * N.  M = local rows; Mg = global rows; row_off = global index of local row 0.
// slab = 0: the whole image is local (M = Mg), periodic neighbours wrap in-kernel; slab = 1: the
// neighbours of rows 0 and M-1 live in the ghost rows (the periodic wrap rows at ranks 0 and P-1).
struct StencilArgs {
    int M, N;
    int Mg, row_off, slab;
    long long plane;
    Reg reg;
    float e[9];        // e_q = exp(-q^2/d^2), q = 0..8
    float tau, gamma, alpha, beta, mu;
    float beta2_mu;    // 2 beta / mu
    float gamma_mu;    // gamma / mu
    int w_proj;        // 0 ball, 1 sphere, 2 none
    float b_max;
    int tiles_x, tiles_y, ntiles;   // tiles per row, per column, total (x batch)
    int gh;            // ghost rows above each plane (TMA coordinates address the allocation rows)
    int aos;           // 1: emit the full RHS F (AOS phi solver, NEXT-4); 0: the increment D = F - A psi
    int band_skip;     // 1: window sums only in the narrow band (exact, needs_v); 0: everywhere (SRSB_BAND_SKIP=0)
    double* stats;     // NEXT-1 monitor: per image [E_g, E_a, E_r, E_pen, ...] accumulated by k_wb; null = off
    int stats_stride;  // doubles per image in stats
};

// NEXT-1 monitor: this CTA's Eq. (22) partial sums -> its slot of the partials buffer a.stats
// (grid = tiles_x x tiles_y x batch; slot = image-major tile index, 4 doubles), summed per image in a
// fixed order by k_reduce_partials (sr_reduce.cuh): deterministic, no atomics.
__device__ __forceinline__ void monitor_partials(const StencilArgs& a, float e_g, float e_a, float e_r, float e_pen) {
    const float v[4] = {e_g, e_a, e_r, e_pen};
    const long long slot = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    block_partials<4>(v, a.stats + slot * 4);
}

#ifndef SRSB_ST_RT
#define SRSB_ST_RT 8
#endif
#ifndef SRSB_ST_BY
#define SRSB_ST_BY 8
#endif
constexpr int ST_CT = 2;            // columns per thread
constexpr int ST_RT = SRSB_ST_RT;   // rows per thread
constexpr int ST_BY = SRSB_ST_BY;   // thread rows per CTA
#ifndef SRSB_ST_MINB
#define SRSB_ST_MINB (32 / SRSB_ST_BY)
#endif
constexpr int ST_MINB = SRSB_ST_MINB;  // resident CTAs per SM the register budget targets (4: <= 64 regs)
constexpr int ST_TW = 32 * ST_CT;
constexpr int ST_TH = ST_BY * ST_RT;

template <int R>
struct TileGeom {
    static constexpr int RA = (R + 1) & ~1;              // halo rounded up to a 2-pixel chunk
    static constexpr int W = ST_TW + 2 * RA;             // staged columns [col0 - RA, col0 + TW + RA)
    static constexpr int CH = W / 2;                     // 16-byte chunks (2 px x 2 channels) per row
    static constexpr int LDC = (CH + 7) & ~7;            // chunk stride per row (multiple of 8)
    static constexpr int ROWS = ST_TH + 2 * R;
    static constexpr int BYTES = LDC * ROWS * 16;
};

// CT-wide vector loads / stores (CT = 2: float2, CT = 4: float4); p must be CT*4-byte aligned.
template <int CT>
__device__ __forceinline__ void ldv(const float* __restrict__ p, float (&o)[CT]) {
    if constexpr (CT == 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = q.x; o[1] = q.y; o[2] = q.z; o[3] = q.w;
    } else if constexpr (CT == 2) {
        const float2 q = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = q.x; o[1] = q.y;
    } else {
#pragma unroll
        for (int c = 0; c < CT; c++) o[c] = __ldg(p + c);
    }
}
template <int CT>
__device__ __forceinline__ void ldv_rw(const float* p, float (&o)[CT]) {   // coherent load (in-place fields)
    if constexpr (CT == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        o[0] = q.x; o[1] = q.y; o[2] = q.z; o[3] = q.w;
    } else if constexpr (CT == 2) {
        const float2 q = *reinterpret_cast<const float2*>(p);
        o[0] = q.x; o[1] = q.y;
    } else {
#pragma unroll
        for (int c = 0; c < CT; c++) o[c] = p[c];
    }
}
template <int CT>
__device__ __forceinline__ void stv(float* p, const float (&o)[CT]) {
    if constexpr (CT == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
    } else if constexpr (CT == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
    } else {
#pragma unroll
        for (int c = 0; c < CT; c++) p[c] = o[c];
    }
}

// bank-conflict-free chunk swizzle for CT = 4 (stride-2 chunk reads): 8 consecutive even (or odd)
// chunks map to 8 distinct bank quads.  CT = 2 reads consecutive chunks: identity.
__device__ __forceinline__ int swz(int c) { return ST_CT == 4 ? c ^ ((c >> 3) & 1) : c; }

// Stage u = h(phi) * w (two channels) over the tile + halo; zero outside the image (reading Q5).
// One 2-pixel chunk per thread and step: float2 global loads, one float4 shared store.
template <int R, bool LEQ>
__device__ __forceinline__ void stage_u(float4* __restrict__ U, const float* __restrict__ phi,
                                        const float* __restrict__ w1, const float* __restrict__ w2,
                                        int Mg, int row_off, int N, int row0, int col0, const Reg& reg) {
    using TG = TileGeom<R>;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    constexpr int NTH = 32 * ST_BY;
    // each thread owns one chunk column f for rows r = tid / CH, + RPP, + 2 RPP, ...: the column
    // bounds test and the column part of the address are computed once, rows advance by pointer
    // increments (no per-element division)
    constexpr int RPP = NTH / TG::CH;                    // rows covered per pass
    static_assert(RPP >= 1, "tile too wide for the CTA");
    const int f = tid % TG::CH, r_first = tid / TG::CH;
    if (r_first >= RPP) return;                          // the NTH % CH leftover threads
    const int gj = col0 - TG::RA + 2 * f;
    const bool col_in = gj >= 0 && gj < N;
    int gi = row0 - R + r_first;
    long long o = (long long)gi * N + gj;                // gi may address a ghost row
    float4* dst = U + r_first * TG::LDC + swz(f);
#pragma unroll 2
    for (int r = r_first; r < TG::ROWS; r += RPP) {
        float4 A = make_float4(0.f, 0.f, 0.f, 0.f);
        if (col_in && gi + row_off >= 0 && gi + row_off < Mg) {
            const float2 P = __ldg(reinterpret_cast<const float2*>(phi + o));
            const float2 X = __ldg(reinterpret_cast<const float2*>(w1 + o));
            const float2 Y = __ldg(reinterpret_cast<const float2*>(w2 + o));
            const float h0 = reg_h<LEQ>(P.x, reg), h1 = reg_h<LEQ>(P.y, reg);
            A = make_float4(h0 * X.x, h0 * Y.x, h1 * X.y, h1 * Y.y);
        }
        *dst = A;
        gi += RPP;
        o += (long long)RPP * N;
        dst += RPP * TG::LDC;
    }
}

// v for the thread's RT x CT block (tile-local rows r0.., cols c0..) from the staged u, in packed
// f32x2 arithmetic (both channels per instruction); conflict-free LDS.128 row reads.
template <int R, int SHAPE, int RT = ST_RT, int LDC = TileGeom<R>::LDC>
__device__ __forceinline__ void window_block(const float4* __restrict__ U, int r0, int c0, const float* e,
                                             float2 (&v)[RT][ST_CT]) {
    using TG = TileGeom<R>;
    constexpr int OFF = (TG::RA - R) & 1;                 // first needed float2 is odd -> load one earlier
    constexpr int NA = ST_CT + 2 * R + OFF;               // float2 values loaded per halo row
    constexpr int NC = (NA + 1) / 2;                      // chunks loaded per halo row
#pragma unroll
    for (int i = 0; i < RT; i++)
#pragma unroll
        for (int c = 0; c < ST_CT; c++) v[i][c] = make_float2(0.f, 0.f);
    float2 ew[R + 1];
#pragma unroll
    for (int q = 0; q <= R; q++) ew[q] = make_float2(e[q], e[q]);
    const int chunk0 = (c0 + TG::RA - R - OFF) >> 1;
#pragma unroll
    for (int rr = 0; rr < RT + 2 * R; rr++) {
        float2 a[2 * NC];
        const float4* row = U + (r0 + rr) * LDC;
        SRSB_CHK(row + swz(chunk0), 16);
        SRSB_CHK(row + swz(chunk0 + NC - 1), 16);
#pragma unroll
        for (int k = 0; k < NC; k++) {
            const float4 q4 = row[swz(chunk0 + k)];
            a[2 * k] = make_float2(q4.x, q4.y);
            a[2 * k + 1] = make_float2(q4.z, q4.w);
        }
        // S[L][c] = sum_{|q| <= L} e_q a[OFF + c + R + q]
        float2 S[R + 1][ST_CT];
#pragma unroll
        for (int c = 0; c < ST_CT; c++) {
            const int m = OFF + c + R;
            float2 acc = a[m];   // e_0 = exp(0) = 1 exactly: 1 * u is u (no multiply)
            S[0][c] = acc;
#pragma unroll
            for (int q = 1; q <= R; q++) {
                acc = fma2(ew[q], add2(a[m - q], a[m + q]), acc);
                S[q][c] = acc;
            }
        }
#pragma unroll
        for (int i = 0; i < RT; i++) {
            const int p = rr - R - i;   // row offset of this halo row w.r.t. output row i
            if (p >= -R && p <= R) {
                const int ap = p < 0 ? -p : p;
                const int L = half_width<R, SHAPE>(ap);
#pragma unroll
                for (int c = 0; c < ST_CT; c++)   // fma(1, S, v) = S + v with one rounding: the same as add
                    v[i][c] = ap == 0 ? add2(S[L][c], v[i][c]) : fma2(ew[ap], S[L][c], v[i][c]);
            }
        }
    }
}

// Increment form of Eq. (37):  D = F - A psi, A = 1 - tau mu Delta_per, i.e.
//   D = tau [ -gamma g |w| delta'(psi) + alpha g delta(psi) + 2 beta h'(psi) w.v + mu div(b - w)
//             + mu Delta_per psi ],
// so that phi^{s+1} = psi + A^{-1} D (= A^{-1} F, Eq. 33) and the FFT round-off scales with the
// increment instead of with |psi| ~ 1 on the plateaus.  Delta_per is the periodic 5-point
// Laplacian of Eq. (35) whose symbol is Eq. (32).
template <int R, int SHAPE, bool LEQ>
__device__ __forceinline__ void rhs_tile(float4* __restrict__ U, const float* __restrict__ phi,
                                         const float* __restrict__ w, const float* __restrict__ bv,
                                         const float* __restrict__ g, float* __restrict__ D, const StencilArgs& a,
                                         int img, int by, int bx) {
    const int M = a.M, N = a.N;
    const long long plane = a.plane;
    const float* ph = phi + img * plane;
    const float* w1 = w + img * 2 * plane;
    const float* w2 = w1 + plane;
    const float* b1 = bv + img * 2 * plane;
    const float* b2 = b1 + plane;
    const float* gg = g + img * plane;
    float* Do = D + img * plane;
    const int row0 = by * ST_TH, col0 = bx * ST_TW;
    stage_u<R, LEQ>(U, ph, w1, w2, a.Mg, a.row_off, N, row0, col0, a.reg);
    __syncthreads();
    const int r0 = threadIdx.y * ST_RT, c0 = threadIdx.x * ST_CT;
    const int gj = col0 + c0;
    if (gj >= N || row0 + r0 >= M) return;
    float2 v[ST_RT][ST_CT];
    window_block<R, SHAPE>(U, r0, c0, a.e, v);
    const int jl = (gj - 1) & (N - 1), jr = (gj + ST_CT) & (N - 1);   // periodic neighbours
    constexpr int CT = ST_CT;
    // periodic row neighbour: wrapped in-kernel for a whole image, a ghost row in slab mode
    auto prow = [&](int x) { return a.slab ? x : (x + M) & (M - 1); };
    // c1 = (b1 - w1) and psi of the row above the first output row
    float c1p[CT], Pu[CT], P[CT];
    {
        const int gi = row0 + r0 - 1;
#pragma unroll
        for (int c = 0; c < CT; c++) c1p[c] = 0.f;
        if (gi + a.row_off >= 0) {
            float bb[CT], ww[CT];
            ldv<CT>(b1 + (long long)gi * N + gj, bb);
            ldv<CT>(w1 + (long long)gi * N + gj, ww);
#pragma unroll
            for (int c = 0; c < CT; c++) c1p[c] = bb[c] - ww[c];
        }
        ldv<CT>(ph + (long long)prow(gi) * N + gj, Pu);
    }
    ldv<CT>(ph + (long long)(row0 + r0) * N + gj, P);
#pragma unroll
    for (int i = 0; i < ST_RT; i++) {
        const int gi = row0 + r0 + i;
        if (gi >= M) break;
        const int gig = gi + a.row_off;   // global row
        const long long o = (long long)gi * N + gj;
        float Pd[CT], w1_[CT], w2_[CT], b1_[CT], b2_[CT], g_[CT];
        ldv<CT>(ph + (long long)prow(gi + 1) * N + gj, Pd);
        const float pl = __ldg(ph + o - gj + jl), pr = __ldg(ph + o - gj + jr);
        ldv<CT>(w1 + o, w1_);
        ldv<CT>(w2 + o, w2_);
        ldv<CT>(b1 + o, b1_);
        ldv<CT>(b2 + o, b2_);
        ldv<CT>(gg + o, g_);
        float c2l = 0.f;   // (b2 - w2) at column gj - 1 (non-periodic divergence, Eq. 36 / Q6)
        if (gj > 0) c2l = __ldg(b2 + o - 1) - __ldg(w2 + o - 1);
        float out[CT];
#pragma unroll
        for (int c = 0; c < CT; c++) {
            const int j = gj + c;
            const float c1 = b1_[c] - w1_[c];
            const float c2 = b2_[c] - w2_[c];
            float dv = 0.f;
            if (gig < a.Mg - 1) dv += c1;
            if (gig > 0) dv -= c1p[c];
            if (j < N - 1) dv += c2;
            if (j > 0) dv -= c2l;
            c2l = c2;
            c1p[c] = c1;
            const float ps = P[c];
            const float left = c > 0 ? P[c > 0 ? c - 1 : 0] : pl;
            const float right = c < CT - 1 ? P[c < CT - 1 ? c + 1 : 0] : pr;
            // neighbour differences first: exact (Sterbenz) for nearby values, so the O(1) level of
            // psi does not enter the rounding of the Laplacian
            const float lap = ((Pu[c] - ps) + (Pd[c] - ps)) + ((left - ps) + (right - ps));
            const float wv = w1_[c] * v[i][c].x + w2_[c] * v[i][c].y;
            const RegVals rv = reg_all<LEQ>(ps, a.reg);
            // |w| (IEEE sqrt, Q20) only where delta' != 0: elsewhere its product with delta' is 0
            const float wn = rv.dp != 0.f ? sqrtf(w1_[c] * w1_[c] + w2_[c] * w2_[c]) : 0.f;
            const float t = -a.gamma * g_[c] * wn * rv.dp + a.alpha * g_[c] * rv.d + 2.f * a.beta * rv.hp * wv +
                            a.mu * dv;
            out[c] = a.aos ? ps + a.tau * t : a.tau * (t + a.mu * lap);
        }
        stv<CT>(Do + o, out);
#pragma unroll
        for (int c = 0; c < CT; c++) {
            Pu[c] = P[c];
            P[c] = Pd[c];
        }
    }
}

__device__ __forceinline__ void project_w(int mode, float& x, float& y) {
    const float n2 = x * x + y * y;
    if ((mode == 0 && n2 > 1.f) || (mode == 1 && n2 > 1e-8f)) {   // BALL: |w| > 1; SPHERE: |w| > 1e-4
        const float n = sqrtf(n2);                                // IEEE sqrt and divides (Q20)
        x = x / n;
        y = y / n;
    }
}

// One pixel of the w/b update.  ps, pn, pr: phi at (i, j), (i+1, j), (i, j+1); has_dn / has_rt: the
// forward differences exist (not the last global row / column, Eq. 35).  wa, wb2: w^k at the pixel
// (monitor only).  Outputs w^{k+1} = (x, y) and b^{k+1} = (nb1, nb2).
template <int MODE, bool UPDATE_B, bool LEQ, bool MON>
__device__ __forceinline__ void wb_pixel(const StencilArgs& a, float ps, float pn, float pr, bool has_dn, bool has_rt,
                                         float b1, float b2, float g, float2 v, float wa, float wb2, float& x,
                                         float& y, float& nb1, float& nb2, bool& bad, float& e_g, float& e_a,
                                         float& e_r, float& e_pen) {
    const float gp1 = has_dn ? pn - ps : 0.f;
    const float gp2 = has_rt ? pr - ps : 0.f;
    float hh, dd;
    reg_hd<LEQ>(ps, a.reg, hh, dd);
    if (MON) {   // energy of Eq. (22) at (phi^{k+1}, w^k, b^k), the state entering the update
        const float aa = ps * a.reg.inv_eps;
        const float H = aa > 1.f ? 1.f : (aa < -1.f ? 0.f : 0.5f * (1.f + aa + sinpif(aa) * (1.f / kPi)));
        e_g += g * sqrtf(wa * wa + wb2 * wb2) * dd;
        e_a += g * (1.f - H);
        e_r -= hh * (wa * v.x + wb2 * v.y);
        const float r1 = wa - gp1 - b1, r2 = wb2 - gp2 - b2;
        e_pen += 0.5f * a.mu * (r1 * r1 + r2 * r2);
    }
    if (MODE == 0) {
        const float Bx = gp1 + b1 + a.beta2_mu * hh * v.x;
        const float By = gp2 + b2 + a.beta2_mu * hh * v.y;
        const float t = a.gamma_mu * g * dd;
        const float nb2v = Bx * Bx + By * By;
        if (t == 0.f) {                                  // off the band (delta = 0): the shrink is the
            x = Bx;                                      // identity, exactly what the IEEE form below
            y = By;                                      // gives there ((|B| - 0)/|B| = 1)
        } else if (nb2v > 0.f) {
            const float nb = sqrtf(nb2v);                // |B|, IEEE (Q20)
            const float m = fmaxf(nb - t, 0.f) / nb;     // max(|B| - t, 0)/|B|, IEEE divide
            x = m * Bx;
            y = m * By;
        } else {
            x = 0.f;
            y = 0.f;
        }
    } else {
        const float den = a.gamma * g * dd + a.mu;
        x = (a.mu * gp1 + a.mu * b1 + 2.f * a.beta * hh * v.x) / den;
        y = (a.mu * gp2 + a.mu * b2 + 2.f * a.beta * hh * v.y) / den;
    }
    project_w(a.w_proj, x, y);
    nb1 = b1 + gp1 - x;
    nb2 = b2 + gp2 - y;
    if (UPDATE_B) {
        bad |= !(fabsf(nb1) <= a.b_max && fabsf(nb2) <= a.b_max) && a.b_max > 0.f;
        bad |= !isfinite(nb1) || !isfinite(nb2);
    }
}

// MODE 0: threshold (Eq. 41-42); MODE 1: fixed-point sweep (Eq. 38-39).  UPDATE_B: last pass,
// b += grad phi - w_new (Eq. 23) and the non-finite guard.  w_in is read for v (the halo) only in
// mode 1 beyond the pixel; in mode 0 w_in = w^k.  b is updated in place (pixel-local).
template <int R, int SHAPE, int MODE, bool UPDATE_B, bool LEQ, bool MON>
__device__ __forceinline__ void wb_tile(float4* __restrict__ U, const float* __restrict__ phi,
                                        const float* __restrict__ w_in, float* __restrict__ w_out,
                                        float* __restrict__ bv, const float* __restrict__ g,
                                        int* __restrict__ flag, const StencilArgs& a, int img, int by, int bx) {
    const int M = a.M, N = a.N;
    const long long plane = a.plane;
    const float* ph = phi + img * plane;
    const float* w1 = w_in + img * 2 * plane;
    const float* w2 = w1 + plane;
    float* o1 = w_out + img * 2 * plane;
    float* o2 = o1 + plane;
    float* b1 = bv + img * 2 * plane;
    float* b2 = b1 + plane;
    const float* gg = g + img * plane;
    const int row0 = by * ST_TH, col0 = bx * ST_TW;
    stage_u<R, LEQ>(U, ph, w1, w2, a.Mg, a.row_off, N, row0, col0, a.reg);
    __syncthreads();
    const int r0 = threadIdx.y * ST_RT, c0 = threadIdx.x * ST_CT;
    const int gj = col0 + c0;
    const bool active = gj < N && row0 + r0 < M;
    if (!MON && !active) return;   // the monitor variant keeps every thread for its CTA reduction
    float2 v[ST_RT][ST_CT];
    if (active) window_block<R, SHAPE>(U, r0, c0, a.e, v);
    bool bad = false;
    constexpr int CT = ST_CT;
    float e_g = 0.f, e_a = 0.f, e_r = 0.f, e_pen = 0.f;   // monitor partial sums (Eq. 22 terms)
#pragma unroll
    for (int i = 0; i < ST_RT; i++) {
        const int gi = row0 + r0 + i;
        if (!active || gi >= M) break;
        const int gig = gi + a.row_off;   // global row
        const long long o = (long long)gi * N + gj;
        float p_[CT + 1], pn_[CT], b1_[CT], b2_[CT], g_[CT];
        {
            float P[CT];
            ldv<CT>(ph + o, P);
#pragma unroll
            for (int c = 0; c < CT; c++) p_[c] = P[c];
        }
        if (gig < a.Mg - 1) ldv<CT>(ph + o + N, pn_);   // next row (a ghost row at the slab edge;
                                                         // grad component 1 is 0 on the last image row)
        else {
#pragma unroll
            for (int c = 0; c < CT; c++) pn_[c] = p_[c];
        }
        p_[CT] = (gj + CT < N) ? __ldg(ph + o + CT) : 0.f;
        ldv_rw<CT>(b1 + o, b1_);
        ldv_rw<CT>(b2 + o, b2_);
        ldv<CT>(gg + o, g_);
        float n1[CT], n2[CT], nb1[CT], nb2[CT];
#pragma unroll
        for (int c = 0; c < CT; c++) {
            const int j = gj + c;
            float wa = 0.f, wb2 = 0.f;
            if (MON) {
                wa = __ldg(w1 + o + c);
                wb2 = __ldg(w2 + o + c);
            }
            wb_pixel<MODE, UPDATE_B, LEQ, MON>(a, p_[c], pn_[c], p_[c + 1], gig < a.Mg - 1, j < N - 1, b1_[c], b2_[c],
                                               g_[c], v[i][c], wa, wb2, n1[c], n2[c], nb1[c], nb2[c], bad, e_g, e_a,
                                               e_r, e_pen);
        }
        stv<CT>(o1 + o, n1);
        stv<CT>(o2 + o, n2);
        if (UPDATE_B) {
            stv<CT>(b1 + o, nb1);
            stv<CT>(b2 + o, nb2);
        }
    }
    if (UPDATE_B && bad) atomicOr(flag, 1);
    if (MON) monitor_partials(a, e_g, e_a, e_r, e_pen);
}

// One CTA per tile (grid = tiles_x x tiles_y x batch).  A persistent variant with one-tile-ahead L2
// bulk prefetch measured slower: the loop raised register pressure.
template <int R, int SHAPE, bool LEQ>
__global__ void __launch_bounds__(32 * ST_BY, ST_MINB) k_rhs(const float* __restrict__ phi, const float* __restrict__ w,
                                                    const float* __restrict__ bv, const float* __restrict__ g,
                                                    float* __restrict__ D, StencilArgs a) {
    extern __shared__ float4 U[];
    rhs_tile<R, SHAPE, LEQ>(U, phi, w, bv, g, D, a, blockIdx.z, blockIdx.y, blockIdx.x);
}

// ------------------------------------------------------------------ TMA-staged RHS (k_rhs_tma)
// Same arithmetic as rhs_tile, different data movement.  One elected thread issues TMA box loads
// completing on mbarriers, so a CTA has a whole box set in flight at once instead of a few loads
// per thread:
//   group 1 (bar[0]): phi, w1, w2 over the tile + window halo -> u = h(phi) w staged as chunks;
//   group 2 (bar[1]): b1, b2 (one-row / one-column divergence halo) and g, loaded into the u
//                     region once the window sums are in registers (u is dead by then).
// Reusing the u region keeps the CTA at ~62 KB of shared memory (3 CTAs per SM) while the other
// resident CTAs cover each CTA's two load waits.  Boxes address the allocation rows (ghost rows
// included); rows outside the image are masked in the u staging exactly as in stage_u, columns
// outside are zero-filled by the TMA unit (w = 0 -> u = 0, reading Q5).
struct RhsMaps {
    CUtensorMap phi, w, b, g;   // phi / w: box PW x PH; b: BW x BH; g: TW x TH (TmaGeom)
    CUtensorMap bt;             // b, box TW x TH (the w/b update reads b at the tile only)
};

#ifndef SRSB_TMA_TH
#define SRSB_TMA_TH 32      // tile rows of the TMA kernels (a multiple of 8: 8 thread rows x TH/8 rows)
#endif
#ifndef SRSB_TMA_MINB
#define SRSB_TMA_MINB 3     // resident CTAs per SM asked of ptxas (shared memory allows 3 at TH = 32)
#endif
constexpr int TMA_TH = SRSB_TMA_TH;
constexpr int tma_hr(int R) { return R > 1 ? R : 1; }                 // box row halo (the Laplacian needs 1)
// box column halo: >= the u halo RA and >= 1 (Laplacian), rounded to 4 columns so every box row is a
// multiple of 32 bytes (box rows of 272 / 304 bytes faulted with an illegal instruction on B200)
constexpr int tma_ca(int R) { return ((((R + 1) & ~1) > 1 ? ((R + 1) & ~1) : 1) + 3) & ~3; }
constexpr int tma_pw(int R) { return ST_TW + 2 * tma_ca(R); }          // phi / w box width
constexpr int tma_ph(int R) { return TMA_TH + 2 * tma_hr(R); }         // phi / w box height
constexpr int TMA_BW = ST_TW + 8, TMA_BH = TMA_TH + 1;                 // b box: columns col0-4.., rows row0-1..

template <int R>
struct TmaGeom {
    static constexpr int TH = TMA_TH, TW = ST_TW, RT = TMA_TH / 8;   // 8 thread rows x RT rows, 32 x 2 columns
    static constexpr int RA = TileGeom<R>::RA;           // u halo columns (even)
    static constexpr int HR = tma_hr(R), CA = tma_ca(R);
    static constexpr int PW = tma_pw(R), PH = tma_ph(R);
    static constexpr int BW = TMA_BW, BH = TMA_BH;
    static constexpr int UROWS = TH + 2 * R, UCH = TileGeom<R>::CH, LDC = UCH;   // warps read one row: no pad
    static constexpr int al(int x) { return (x + 127) & ~127; }
    static constexpr int S_P = al(PW * PH * 4), S_B = al(BW * BH * 4), S_G = al(TW * TH * 4);
    static constexpr int S_U = al(LDC * UROWS * 16), S_BG = 2 * S_B + S_G;
    static constexpr int O_P = 0, O_W1 = S_P, O_W2 = 2 * S_P, O_U = 3 * S_P;
    static constexpr int O_B1 = O_U, O_B2 = O_U + S_B, O_G = O_U + 2 * S_B;   // group 2 reuses the u region
    static constexpr int O_BAR = O_U + (S_U > S_BG ? S_U : S_BG);
    static constexpr int BYTES = O_BAR + 16 + 128;       // + alignment slack of the dynamic base
    static constexpr uint32_t TX1 = (uint32_t)(3 * PW * PH) * 4, TX2 = (uint32_t)(2 * BW * BH + TW * TH) * 4;
};

// Narrow band (Eq. 11 and 28).  Every use of the window sum v is multiplied by
// h(psi) (w/b update, Eq. 41) or h'(psi) (RHS, Eq. 37), which are EXACTLY zero where the regularizer
// functions take their early exit: |psi| / eps >= 2 (l = eps) or |psi| >= l + eps and |psi| > eps.
// needs_v is the negation of that exit test (same fp32 expressions), so skipping the window sums (and
// the u staging of a tile none of whose pixels needs v) changes no result: the skipped terms are
// 0 * finite.  Out of the band -- most pixels, since the band follows the contour -- a stencil tile is
// then the pointwise part and its loads only.
template <bool LEQ>
__device__ __forceinline__ bool needs_v(float x, const Reg& r) {
    if constexpr (LEQ) return !(fabsf(x * r.inv_eps) >= 2.f);
    else return !(fabsf(x) >= r.l + r.eps && fabsf(x) > r.eps);
}
// any of the thread's RT x 2 tile pixels (rows inside the image) in the band; Ps = the phi box
template <bool LEQ, class G>
__device__ __forceinline__ bool block_needs_v(const float* Ps, int r0, int c0, int row0, int M, const Reg& r) {
    bool need = false;
#pragma unroll
    for (int i = 0; i < G::RT; i++) {
        if (row0 + r0 + i >= M) break;
        const float2 P = *reinterpret_cast<const float2*>(Ps + (G::HR + r0 + i) * G::PW + G::CA + c0);
        need |= needs_v<LEQ>(P.x, r) || needs_v<LEQ>(P.y, r);
    }
    return need;
}
template <int RT>
__device__ __forceinline__ void zero_v(float2 (&v)[RT][ST_CT]) {
#pragma unroll
    for (int i = 0; i < RT; i++)
#pragma unroll
        for (int c = 0; c < ST_CT; c++) v[i][c] = make_float2(0.f, 0.f);
}

// u = h(phi) w over the tile + R halo from the group-1 boxes, as 16-byte chunks (2 px x 2 channels)
// in TileGeom's layout; rows outside the image give u = 0 (reading Q5).  Branch-free, f32x2.
#ifndef SRSB_STAGE_U_OLD
#define SRSB_STAGE_U_OLD 0   // 1: the strided loop with a division per chunk (A/B reference)
#endif
template <int R, bool LEQ, class G>
__device__ __forceinline__ void stage_u_tma(float4* __restrict__ U, const float* Ps, const float* W1s,
                                            const float* W2s, int row0, int tid, const StencilArgs& a) {
#if SRSB_STAGE_U_OLD
    for (int k = tid; k < G::UROWS * G::UCH; k += 256) {
        const int r = k / G::UCH, f = k - r * G::UCH;
#else
    // fixed trip count, (r, f) stepped incrementally (256 = DR rows + DF chunks)
    constexpr int TOT = G::UROWS * G::UCH, NIT = (TOT + 255) / 256, DR = 256 / G::UCH, DF = 256 % G::UCH;
    int r = tid / G::UCH, f = tid - (tid / G::UCH) * G::UCH;
#pragma unroll
    for (int it = 0; it < NIT; it++, r += DR, f += DF) {
        if (f >= G::UCH) {
            f -= G::UCH;
            r++;
        }
        if (it == NIT - 1 && tid + it * 256 >= TOT) break;
#endif
        const int gr = row0 - R + r + a.row_off;   // global row
        const int o = (r + G::HR - R) * G::PW + (G::CA - G::RA) + 2 * f;
        const float2 P = *reinterpret_cast<const float2*>(Ps + o);
        const float2 X = *reinterpret_cast<const float2*>(W1s + o);
        const float2 Y = *reinterpret_cast<const float2*>(W2s + o);
        const float2 h = reg_h2<LEQ>(P, a.reg);
        const float2 hx = mul2(h, X), hy = mul2(h, Y);
        const bool in = gr >= 0 && gr < a.Mg;
        SRSB_CHK(Ps + o, 8);
        SRSB_CHK(W2s + o, 8);
        SRSB_CHK(&U[r * G::LDC + swz(f)], 16);
        U[r * G::LDC + swz(f)] = in ? make_float4(hx.x, hy.x, hx.y, hy.y) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// The pointwise part of Eq. (37) (increment form) for the thread's RT x 2 block,
// both pixels of a row in f32x2.  EDGE = false: the tile touches no image boundary (no masks, no
// periodic wrap loads, no ragged rows).
// TOREG: the results go to res[i] (k_rhs_r2c keeps the tile of D on chip) instead of D in global memory.
template <int R, bool LEQ, bool EDGE, class G, bool TOREG = false>
__device__ __forceinline__ void rhs_points_tma(const float* Ps, const float* W1s, const float* W2s, const float* B1s,
                                               const float* B2s, const float* Gs, const float* __restrict__ phi,
                                               float* __restrict__ D, const float2 (&v)[G::RT][ST_CT], int img,
                                               int row0, int r0, int c0, int col0, const StencilArgs& a,
                                               float2* res = nullptr) {
    const int M = a.M, N = a.N, gj = col0 + c0;
    const float* ph = phi + img * a.plane;
    float* Do = D + img * a.plane;
    // values of row i - 1 carried in registers: psi (the Laplacian's upper neighbour) and b1 - w1
    // (the divergence's upper term); psi of row i is the previous row's lower neighbour
    float2 P = *reinterpret_cast<const float2*>(Ps + (G::HR + r0) * G::PW + G::CA + c0);
    float2 Pc = *reinterpret_cast<const float2*>(Ps + (G::HR + r0 - 1) * G::PW + G::CA + c0);
    float2 c1c = sub2(*reinterpret_cast<const float2*>(B1s + r0 * G::BW + 4 + c0),
                      *reinterpret_cast<const float2*>(W1s + (G::HR + r0 - 1) * G::PW + G::CA + c0));
#pragma unroll
    for (int i = 0; i < G::RT; i++) {
        const int tr = r0 + i, gi = row0 + tr;
        if (EDGE && gi >= M) break;
        const float* prow = Ps + (G::HR + tr) * G::PW + G::CA + c0;
        const float* w1r = W1s + (G::HR + tr) * G::PW + G::CA + c0;
        const float* w2r = W2s + (G::HR + tr) * G::PW + G::CA + c0;
        const float* b1r = B1s + (1 + tr) * G::BW + 4 + c0;
        SRSB_CHK(prow - 1, 4 * (ST_CT + 2));
        SRSB_CHK(prow + G::PW, 8);
        SRSB_CHK(W2s + (G::HR + tr) * G::PW + G::CA + c0 - 1, 12);
        SRSB_CHK(b1r - G::BW, 8);
        SRSB_CHK(B2s + (1 + tr) * G::BW + 4 + c0 - 1, 12);
        SRSB_CHK(Gs + tr * G::TW + c0, 8);
        const float* b2r = B2s + (1 + tr) * G::BW + 4 + c0;
        const float2 Pn = *reinterpret_cast<const float2*>(prow + G::PW);
        float2 Pu = Pc, Pd = Pn;
        float pl = prow[-1], pr = prow[ST_CT];
        const float2 W1 = *reinterpret_cast<const float2*>(w1r), W2 = *reinterpret_cast<const float2*>(w2r);
        const float2 B1 = *reinterpret_cast<const float2*>(b1r), B2 = *reinterpret_cast<const float2*>(b2r);
        const float2 Gv = *reinterpret_cast<const float2*>(Gs + tr * G::TW + c0);
        const float2 c1n = sub2(B1, W1);
        float2 c1 = c1n, c1u = c1c, c2 = sub2(B2, W2);
        float2 c2l = make_float2(b2r[-1] - w2r[-1], c2.x);   // (b2 - w2) at columns gj - 1, gj
        if (EDGE) {
            const int gig = gi + a.row_off;
            if (!a.slab) {   // periodic rows of Eq. (32) wrap in-kernel for a whole image
                if (gi == 0) Pu = __ldg(reinterpret_cast<const float2*>(ph + (long long)(M - 1) * N + gj));
                if (gi == M - 1) Pd = __ldg(reinterpret_cast<const float2*>(ph + gj));
            }
            if (gj == 0) pl = __ldg(ph + (long long)gi * N + N - 1);
            if (gj + ST_CT == N) pr = __ldg(ph + (long long)gi * N);
            // Eq. (36) / Q6: terms outside the image are dropped (x + 0 and x - 0 are exact)
            if (gig >= a.Mg - 1) c1 = f2(0.f);
            if (gig <= 0) c1u = f2(0.f);
            if (gj + 1 >= N - 1) c2.y = 0.f;
            if (gj == 0) c2l.x = 0.f;
        }
        const float2 lap = add2(add2(sub2(Pu, P), sub2(Pd, P)),
                                add2(sub2(make_float2(pl, P.x), P), sub2(make_float2(P.y, pr), P)));
        const float2 dv = sub2(add2(sub2(c1, c1u), c2), c2l);
        const float2 wv = fma2(W1, make_float2(v[i][0].x, v[i][1].x), mul2(W2, make_float2(v[i][0].y, v[i][1].y)));
        float2 hp, dd, dp;
        reg_rhs2<LEQ>(P, a.reg, hp, dd, dp);
        // |w| (IEEE sqrt, Q20) only where delta' != 0 (the band): elsewhere its product with delta' is 0
        float2 wn = f2(0.f);
        if (dp.x != 0.f) wn.x = sqrtf(fmaf(W1.x, W1.x, W2.x * W2.x));
        if (dp.y != 0.f) wn.y = sqrtf(fmaf(W1.y, W1.y, W2.y * W2.y));
        // t = g (alpha delta - gamma |w| delta') + 2 beta h' w.v + mu div(b - w)
        float2 t = mul2(Gv, fma2(f2(a.alpha), dd, mul2(f2(-a.gamma), mul2(wn, dp))));
        t = fma2(f2(2.f * a.beta), mul2(hp, wv), t);
        t = fma2(f2(a.mu), dv, t);
        const float2 out = a.aos ? fma2(f2(a.tau), t, P) : mul2(f2(a.tau), fma2(f2(a.mu), lap, t));
        if constexpr (TOREG) res[i] = out;
        else *reinterpret_cast<float2*>(Do + (long long)gi * N + gj) = out;
        Pc = P;
        P = Pn;
        c1c = c1n;
    }
}

// L2 prefetch in the TMA stencils (k_rhs_tma: SRSB_RHS_PF, k_wb_tma: SRSB_WB_PF):
//   bit 0: the CTA's own group 2 at its start (its later TMA load then hits L2);
//   bit 1: both groups of the CTA SRSB_*_PF_DIST launches ahead (scheduled later on a freed slot).
// Measured on C3 (whole step, 2 steps each): none 21.05k, rhs bit 1 + wb bit 1 21.36k, rhs 2 + wb 1 21.24k /
// 21.20k Mpx-iter/s (rhs 0.447 -> 0.422 ms, wb 0.519 -> 0.488 ms in isolation; under the sustained step the
// extra traffic meets the power cap, so the step gains ~1 %); rhs 2 at distance 888: 20.27k.
#ifndef SRSB_RHS_PF
#define SRSB_RHS_PF 2
#endif
#ifndef SRSB_WB_PF
#define SRSB_WB_PF 1
#endif
#ifndef SRSB_RHS_PF_DIST
#define SRSB_RHS_PF_DIST (148 * SRSB_TMA_MINB) // one wave of resident CTAs
#endif
#ifndef SRSB_WB_PF_DIST
#define SRSB_WB_PF_DIST (148 * SRSB_TMA_MINB)
#endif
// tile coordinates of the CTA `ahead` launches after this one (blockIdx.x fastest); false past the grid
__device__ __forceinline__ bool tile_ahead(int ahead, int& bx, int& by, int& bz) {
    const long long lin = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z) + ahead;
    if (lin >= (long long)gridDim.x * gridDim.y * gridDim.z) return false;
    bx = (int)(lin % gridDim.x);
    by = (int)((lin / gridDim.x) % gridDim.y);
    bz = (int)(lin / ((long long)gridDim.x * gridDim.y));
    return true;
}

template <int R, int SHAPE, bool LEQ>
__global__ void __launch_bounds__(256, SRSB_TMA_MINB) k_rhs_tma(const __grid_constant__ RhsMaps maps,
                                                    const float* __restrict__ phi, float* __restrict__ D,
                                                    StencilArgs a) {
    using G = TmaGeom<R>;
    extern __shared__ unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((128 - (smem_u32(sm_raw) & 127)) & 127);
    float* Ps = reinterpret_cast<float*>(sm + G::O_P);
    float* W1s = reinterpret_cast<float*>(sm + G::O_W1);
    float* W2s = reinterpret_cast<float*>(sm + G::O_W2);
    float* B1s = reinterpret_cast<float*>(sm + G::O_B1);
    float* B2s = reinterpret_cast<float*>(sm + G::O_B2);
    float* Gs = reinterpret_cast<float*>(sm + G::O_G);
    float4* U = reinterpret_cast<float4*>(sm + G::O_U);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + G::O_BAR);
    const int img = blockIdx.z, row0 = blockIdx.y * G::TH, col0 = blockIdx.x * G::TW;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int ar = a.gh + row0;   // allocation row of local row row0
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bar[0], G::TX1);
        tma_load_3d(Ps, &maps.phi, &bar[0], col0 - G::CA, ar - G::HR, img);
        tma_load_3d(W1s, &maps.w, &bar[0], col0 - G::CA, ar - G::HR, 2 * img);
        tma_load_3d(W2s, &maps.w, &bar[0], col0 - G::CA, ar - G::HR, 2 * img + 1);
        if (SRSB_RHS_PF & 1) {
            tma_prefetch_3d(&maps.b, col0 - 4, ar - 1, 2 * img);
            tma_prefetch_3d(&maps.b, col0 - 4, ar - 1, 2 * img + 1);
            tma_prefetch_3d(&maps.g, col0, ar, img);
        }
        int bx, by, bz;
        if ((SRSB_RHS_PF & 2) && tile_ahead(SRSB_RHS_PF_DIST, bx, by, bz)) {
            const int c = bx * G::TW, r = a.gh + by * G::TH;
            tma_prefetch_3d(&maps.phi, c - G::CA, r - G::HR, bz);
            tma_prefetch_3d(&maps.w, c - G::CA, r - G::HR, 2 * bz);
            tma_prefetch_3d(&maps.w, c - G::CA, r - G::HR, 2 * bz + 1);
            tma_prefetch_3d(&maps.b, c - 4, r - 1, 2 * bz);
            tma_prefetch_3d(&maps.b, c - 4, r - 1, 2 * bz + 1);
            tma_prefetch_3d(&maps.g, c, r, bz);
        }
    }
    mbar_wait(&bar[0], 0);
    const int r0 = threadIdx.y * G::RT, c0 = threadIdx.x * ST_CT;
    const int M = a.M, N = a.N, gj = col0 + c0;
    const bool active = gj < N && row0 + r0 < M;
    // narrow band: v only where h'(psi) != 0; u staged only if some pixel of the tile needs v
    const bool own = !a.band_skip || (active && block_needs_v<LEQ, G>(Ps, r0, c0, row0, M, a.reg));
    float2 v[G::RT][ST_CT];
    zero_v<G::RT>(v);
    if (__syncthreads_or(own)) {
        // u = h(phi) w over the tile + R halo, as 16-byte chunks (2 px x 2 channels) in TileGeom's layout
        stage_u_tma<R, LEQ, G>(U, Ps, W1s, W2s, row0, tid, a);
        __syncthreads();
        if (active && own) window_block<R, SHAPE, G::RT, G::LDC>(U, r0, c0, a.e, v);
    }
    __syncthreads();   // u is dead: group 2 lands in its place
    if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads of u before async writes
        mbar_expect_tx(&bar[1], G::TX2);
        tma_load_3d(B1s, &maps.b, &bar[1], col0 - 4, ar - 1, 2 * img);
        tma_load_3d(B2s, &maps.b, &bar[1], col0 - 4, ar - 1, 2 * img + 1);
        tma_load_3d(Gs, &maps.g, &bar[1], col0, ar, img);
    }
    if (!active) return;
    mbar_wait(&bar[1], 0);
    // interior tiles (no image boundary, no ragged rows) take the check-free path
    const bool edge = row0 + a.row_off == 0 || row0 + G::TH + a.row_off >= a.Mg || row0 + G::TH > M || col0 == 0 ||
                      col0 + G::TW >= N;
    if (edge)
        rhs_points_tma<R, LEQ, true, G>(Ps, W1s, W2s, B1s, B2s, Gs, phi, D, v, img, row0, r0, c0, col0, a);
    else
        rhs_points_tma<R, LEQ, false, G>(Ps, W1s, W2s, B1s, B2s, Gs, phi, D, v, img, row0, r0, c0, col0, a);
}

// ------------------------------------------------------------------ TMA-staged w/b update (k_wb_tma)
// Data movement of k_rhs_tma for the w/b update: group 1 = phi, w^k (tile + window halo; the box's
// row / column halo also holds the forward neighbours of Eq. 35), group 2 = b1, b2, g at the tile,
// landing in the dead u region after the window sums.  The per-pixel arithmetic is wb_pixel, shared
// with wb_tile.  b is updated in place (pixel-local), w^{k+1} goes to the other ping-pong buffer.
template <int R>
struct WbGeom {
    using T = TmaGeom<R>;
    static constexpr int TH = T::TH, TW = T::TW, RT = T::RT, HR = T::HR, CA = T::CA, PW = T::PW, PH = T::PH;
    static constexpr int UROWS = T::UROWS, UCH = T::UCH, LDC = T::LDC, RA = T::RA;
    static constexpr int S_T = T::al(TW * TH * 4);       // one tile-sized field (b1, b2, g)
    static constexpr int O_P = 0, O_W1 = T::S_P, O_W2 = 2 * T::S_P, O_U = 3 * T::S_P;
    static constexpr int O_B1 = O_U, O_B2 = O_U + S_T, O_G = O_U + 2 * S_T;
    static constexpr int O_BAR = O_U + (T::S_U > 3 * S_T ? T::S_U : 3 * S_T);
    static constexpr int BYTES = O_BAR + 16 + 128;
    static constexpr uint32_t TX1 = T::TX1, TX2 = (uint32_t)(3 * TW * TH) * 4;
};

template <int R, int SHAPE, int MODE, bool UPDATE_B, bool LEQ, bool MON = false>
__global__ void __launch_bounds__(256, SRSB_TMA_MINB) k_wb_tma(const __grid_constant__ RhsMaps maps, float* __restrict__ w_out,
                                                   float* __restrict__ bv, int* __restrict__ flag, StencilArgs a) {
    using G = WbGeom<R>;
    extern __shared__ unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((128 - (smem_u32(sm_raw) & 127)) & 127);
    float* Ps = reinterpret_cast<float*>(sm + G::O_P);
    float* W1s = reinterpret_cast<float*>(sm + G::O_W1);
    float* W2s = reinterpret_cast<float*>(sm + G::O_W2);
    float* B1s = reinterpret_cast<float*>(sm + G::O_B1);
    float* B2s = reinterpret_cast<float*>(sm + G::O_B2);
    float* Gs = reinterpret_cast<float*>(sm + G::O_G);
    float4* U = reinterpret_cast<float4*>(sm + G::O_U);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + G::O_BAR);
    const int img = blockIdx.z, row0 = blockIdx.y * G::TH, col0 = blockIdx.x * G::TW;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int ar = a.gh + row0;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bar[0], G::TX1);
        tma_load_3d(Ps, &maps.phi, &bar[0], col0 - G::CA, ar - G::HR, img);
        tma_load_3d(W1s, &maps.w, &bar[0], col0 - G::CA, ar - G::HR, 2 * img);
        tma_load_3d(W2s, &maps.w, &bar[0], col0 - G::CA, ar - G::HR, 2 * img + 1);
        if (SRSB_WB_PF & 1) {
            tma_prefetch_3d(&maps.bt, col0, ar, 2 * img);
            tma_prefetch_3d(&maps.bt, col0, ar, 2 * img + 1);
            tma_prefetch_3d(&maps.g, col0, ar, img);
        }
        int bx, by, bz;
        if ((SRSB_WB_PF & 2) && tile_ahead(SRSB_WB_PF_DIST, bx, by, bz)) {
            const int c = bx * G::TW, r = a.gh + by * G::TH;
            tma_prefetch_3d(&maps.phi, c - G::CA, r - G::HR, bz);
            tma_prefetch_3d(&maps.w, c - G::CA, r - G::HR, 2 * bz);
            tma_prefetch_3d(&maps.w, c - G::CA, r - G::HR, 2 * bz + 1);
            tma_prefetch_3d(&maps.bt, c, r, 2 * bz);
            tma_prefetch_3d(&maps.bt, c, r, 2 * bz + 1);
            tma_prefetch_3d(&maps.g, c, r, bz);
        }
    }
    mbar_wait(&bar[0], 0);
    const int r0 = threadIdx.y * G::RT, c0 = threadIdx.x * ST_CT;
    const int M = a.M, N = a.N, gj = col0 + c0;
    const bool active = gj < N && row0 + r0 < M;
    // narrow band: v' only where h(phi^{k+1}) != 0 (Eq. 41; the monitor's E_r carries the same factor)
    const bool own = !a.band_skip || (active && block_needs_v<LEQ, G>(Ps, r0, c0, row0, M, a.reg));
    float2 v[G::RT][ST_CT];
    zero_v<G::RT>(v);
    if (__syncthreads_or(own)) {
        stage_u_tma<R, LEQ, G>(U, Ps, W1s, W2s, row0, tid, a);
        __syncthreads();
        if (active && own) window_block<R, SHAPE, G::RT, G::LDC>(U, r0, c0, a.e, v);
    }
    __syncthreads();   // u is dead: group 2 lands in its place
    if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[1], G::TX2);
        tma_load_3d(B1s, &maps.bt, &bar[1], col0, ar, 2 * img);
        tma_load_3d(B2s, &maps.bt, &bar[1], col0, ar, 2 * img + 1);
        tma_load_3d(Gs, &maps.g, &bar[1], col0, ar, img);
    }
    if (!MON && !active) return;   // the monitor variant keeps every thread for its CTA reduction
    if (active) mbar_wait(&bar[1], 0);
    constexpr int CT = ST_CT;
    bool bad = false;
    float e_g = 0.f, e_a = 0.f, e_r = 0.f, e_pen = 0.f;
    float* o1 = w_out + img * 2 * a.plane;
    float* o2 = o1 + a.plane;
    float* b1g = bv + img * 2 * a.plane;
    float* b2g = b1g + a.plane;
#pragma unroll
    for (int i = 0; i < G::RT; i++) {
        const int tr = r0 + i, gi = row0 + tr;
        if (!active || gi >= M) break;
        const int gig = gi + a.row_off;
        const float* prow = Ps + (G::HR + tr) * G::PW + G::CA + c0;
        const float2 P = *reinterpret_cast<const float2*>(prow);
        const float2 Pn = *reinterpret_cast<const float2*>(prow + G::PW);
        const float p_[CT + 1] = {P.x, P.y, prow[CT]}, pn_[CT] = {Pn.x, Pn.y};
        SRSB_CHK(prow, 4 * (CT + 1));
        SRSB_CHK(prow + G::PW, 8);
        SRSB_CHK(B1s + tr * G::TW + c0, 8);
        SRSB_CHK(Gs + tr * G::TW + c0, 8);
        const float2 B1 = *reinterpret_cast<const float2*>(B1s + tr * G::TW + c0);
        const float2 B2 = *reinterpret_cast<const float2*>(B2s + tr * G::TW + c0);
        const float2 Gv = *reinterpret_cast<const float2*>(Gs + tr * G::TW + c0);
        const float b1_[CT] = {B1.x, B1.y}, b2_[CT] = {B2.x, B2.y}, g_[CT] = {Gv.x, Gv.y};
        float wa_[CT] = {0.f, 0.f}, wb_[CT] = {0.f, 0.f};
        if (MON) {
            const float2 W1 = *reinterpret_cast<const float2*>(W1s + (G::HR + tr) * G::PW + G::CA + c0);
            const float2 W2 = *reinterpret_cast<const float2*>(W2s + (G::HR + tr) * G::PW + G::CA + c0);
            wa_[0] = W1.x; wa_[1] = W1.y; wb_[0] = W2.x; wb_[1] = W2.y;
        }
        float n1[CT], n2[CT], nb1[CT], nb2[CT];
#pragma unroll
        for (int c = 0; c < CT; c++)
            wb_pixel<MODE, UPDATE_B, LEQ, MON>(a, p_[c], pn_[c], p_[c + 1], gig < a.Mg - 1, gj + c < N - 1, b1_[c],
                                               b2_[c], g_[c], v[i][c], wa_[c], wb_[c], n1[c], n2[c], nb1[c], nb2[c],
                                               bad, e_g, e_a, e_r, e_pen);
        const long long o = (long long)gi * N + gj;
        stv<CT>(o1 + o, n1);
        stv<CT>(o2 + o, n2);
        if (UPDATE_B) {
            stv<CT>(b1g + o, nb1);
            stv<CT>(b2g + o, nb2);
        }
    }
    if (UPDATE_B && bad) atomicOr(flag, 1);
    if (MON) monitor_partials(a, e_g, e_a, e_r, e_pen);
}

// MON: the NEXT-1 monitor variant (Eq. 22 energy partial sums), used only when monitoring is on
template <int R, int SHAPE, int MODE, bool UPDATE_B, bool LEQ, bool MON = false>
__global__ void __launch_bounds__(32 * ST_BY, ST_MINB) k_wb(const float* __restrict__ phi, const float* __restrict__ w_in,
                                                   float* __restrict__ w_out, float* __restrict__ bv,
                                                   const float* __restrict__ g, int* __restrict__ flag,
                                                   StencilArgs a) {
    extern __shared__ float4 U[];
    wb_tile<R, SHAPE, MODE, UPDATE_B, LEQ, MON>(U, phi, w_in, w_out, bv, g, flag, a, blockIdx.z, blockIdx.y,
                                                blockIdx.x);
}

}  // namespace srsb
