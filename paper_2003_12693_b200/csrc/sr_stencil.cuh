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

namespace srsb {

constexpr float kPi = 3.14159265358979323846f;

struct Reg {  // regularizer constants (Eq. 5, 6, 11, 28, 29)
    float eps, inv_eps, l;
};

__device__ __forceinline__ float Heps(float x, const Reg& r) {
    if (x > r.eps) return 1.f;
    if (x < -r.eps) return 0.f;
    const float a = x * r.inv_eps;
    return 0.5f * (1.f + a + sinpif(a) * (1.f / kPi));
}
__device__ __forceinline__ float deps(float x, const Reg& r) {
    if (fabsf(x) > r.eps) return 0.f;
    return (1.f + cospif(x * r.inv_eps)) * (0.5f * r.inv_eps);
}
__device__ __forceinline__ float dpeps(float x, const Reg& r) {
    if (fabsf(x) > r.eps) return 0.f;
    return -(0.5f * kPi) * r.inv_eps * r.inv_eps * sinpif(x * r.inv_eps);
}
__device__ __forceinline__ float hband(float x, const Reg& r) {
    return Heps(x + r.l, r) * (1.f - Heps(x - r.l, r));
}
__device__ __forceinline__ float hpband(float x, const Reg& r) {
    return deps(x + r.l, r) * (1.f - Heps(x - r.l, r)) - Heps(x + r.l, r) * deps(x - r.l, r);
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

struct StencilArgs {
    int M, N;
    Reg reg;
    float e[9];        // e_q = exp(-q^2/d^2), q = 0..8
    float tau, gamma, alpha, beta, mu;
    float beta2_mu;    // 2 beta / mu
    float gamma_mu;    // gamma / mu
    int w_proj;        // 0 ball, 1 sphere, 2 none
    float b_max;
};

constexpr int ST_CT = 4;   // columns per thread
constexpr int ST_RT = 8;   // rows per thread
constexpr int ST_BY = 4;   // thread rows per CTA
constexpr int ST_TW = 32 * ST_CT;
constexpr int ST_TH = ST_BY * ST_RT;

template <int R>
struct TileGeom {
    static constexpr int LD = ST_TW + 2 * R + 1;   // float2 per smem row (odd: spreads banks)
    static constexpr int ROWS = ST_TH + 2 * R;
    static constexpr int BYTES = LD * ROWS * 8;
};

// Stage u = h(phi) * w (two channels) over the tile + R halo; zero outside the image.
template <int R>
__device__ __forceinline__ void stage_u(float2* __restrict__ U, const float* __restrict__ phi,
                                        const float* __restrict__ w1, const float* __restrict__ w2,
                                        int M, int N, int row0, int col0, const Reg& reg) {
    using TG = TileGeom<R>;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int nth = 32 * ST_BY;
    constexpr int W = ST_TW + 2 * R;
    for (int e = tid; e < TG::ROWS * W; e += nth) {
        const int r = e / W, c = e - r * W;
        const int gi = row0 - R + r, gj = col0 - R + c;
        float2 u = make_float2(0.f, 0.f);
        if (gi >= 0 && gi < M && gj >= 0 && gj < N) {
            const size_t o = (size_t)gi * N + gj;
            const float hh = hband(__ldg(phi + o), reg);
            u = make_float2(hh * __ldg(w1 + o), hh * __ldg(w2 + o));
        }
        U[r * TG::LD + c] = u;
    }
}

// v for the thread's RT x CT block (tile-local rows r0.., cols c0..) from the staged u.
template <int R, int SHAPE>
__device__ __forceinline__ void window_block(const float2* __restrict__ U, int r0, int c0, const float* e,
                                             float2 (&v)[ST_RT][ST_CT]) {
    using TG = TileGeom<R>;
#pragma unroll
    for (int i = 0; i < ST_RT; i++)
#pragma unroll
        for (int c = 0; c < ST_CT; c++) v[i][c] = make_float2(0.f, 0.f);
#pragma unroll
    for (int rr = 0; rr < ST_RT + 2 * R; rr++) {
        float2 a[ST_CT + 2 * R];
#pragma unroll
        for (int x = 0; x < ST_CT + 2 * R; x++) a[x] = U[(r0 + rr) * TG::LD + c0 + x];
        // S[L][c] = sum_{|q| <= L} e_q a[c + R + q]
        float2 S[R + 1][ST_CT];
#pragma unroll
        for (int c = 0; c < ST_CT; c++) {
            float2 acc = make_float2(e[0] * a[c + R].x, e[0] * a[c + R].y);
            S[0][c] = acc;
#pragma unroll
            for (int q = 1; q <= R; q++) {
                acc.x = fmaf(e[q], a[c + R - q].x + a[c + R + q].x, acc.x);
                acc.y = fmaf(e[q], a[c + R - q].y + a[c + R + q].y, acc.y);
                S[q][c] = acc;
            }
        }
#pragma unroll
        for (int i = 0; i < ST_RT; i++) {
            const int p = rr - R - i;   // row offset of this halo row w.r.t. output row i
            if (p >= -R && p <= R) {
                const int ap = p < 0 ? -p : p;
                const int L = half_width<R, SHAPE>(ap);
                const float ep = e[ap];
#pragma unroll
                for (int c = 0; c < ST_CT; c++) {
                    v[i][c].x = fmaf(ep, S[L][c].x, v[i][c].x);
                    v[i][c].y = fmaf(ep, S[L][c].y, v[i][c].y);
                }
            }
        }
    }
}

// F = psi + tau [ -gamma g |w| delta'(psi) + alpha g delta(psi) + 2 beta h'(psi) w.v + mu div(b - w) ]
template <int R, int SHAPE>
__global__ void __launch_bounds__(32 * ST_BY) k_rhs(const float* __restrict__ phi, const float* __restrict__ w,
                                                    const float* __restrict__ bv, const float* __restrict__ g,
                                                    float* __restrict__ F, StencilArgs a) {
    extern __shared__ float2 U[];
    const int M = a.M, N = a.N;
    const size_t plane = (size_t)M * N;
    const int img = blockIdx.z;
    const float* ph = phi + img * plane;
    const float* w1 = w + img * 2 * plane;
    const float* w2 = w1 + plane;
    const float* b1 = bv + img * 2 * plane;
    const float* b2 = b1 + plane;
    const float* gg = g + img * plane;
    float* Fo = F + img * plane;
    const int row0 = blockIdx.y * ST_TH, col0 = blockIdx.x * ST_TW;
    stage_u<R>(U, ph, w1, w2, M, N, row0, col0, a.reg);
    __syncthreads();
    const int r0 = threadIdx.y * ST_RT, c0 = threadIdx.x * ST_CT;
    const int gj = col0 + c0;
    if (gj >= N) return;
    float2 v[ST_RT][ST_CT];
    window_block<R, SHAPE>(U, r0, c0, a.e, v);
    // c1 = (b1 - w1) of the row above the first output row
    float c1p[ST_CT];
    {
        const int gi = row0 + r0 - 1;
#pragma unroll
        for (int c = 0; c < ST_CT; c++) c1p[c] = 0.f;
        if (gi >= 0 && gi < M) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(b1 + (size_t)gi * N + gj));
            const float4 ww = __ldg(reinterpret_cast<const float4*>(w1 + (size_t)gi * N + gj));
            c1p[0] = bb.x - ww.x; c1p[1] = bb.y - ww.y; c1p[2] = bb.z - ww.z; c1p[3] = bb.w - ww.w;
        }
    }
#pragma unroll
    for (int i = 0; i < ST_RT; i++) {
        const int gi = row0 + r0 + i;
        if (gi >= M) break;
        const size_t o = (size_t)gi * N + gj;
        const float4 P4 = __ldg(reinterpret_cast<const float4*>(ph + o));
        const float4 W1 = __ldg(reinterpret_cast<const float4*>(w1 + o));
        const float4 W2 = __ldg(reinterpret_cast<const float4*>(w2 + o));
        const float4 B1 = __ldg(reinterpret_cast<const float4*>(b1 + o));
        const float4 B2 = __ldg(reinterpret_cast<const float4*>(b2 + o));
        const float4 G4 = __ldg(reinterpret_cast<const float4*>(gg + o));
        const float p_[4] = {P4.x, P4.y, P4.z, P4.w};
        const float w1_[4] = {W1.x, W1.y, W1.z, W1.w};
        const float w2_[4] = {W2.x, W2.y, W2.z, W2.w};
        const float b1_[4] = {B1.x, B1.y, B1.z, B1.w};
        const float b2_[4] = {B2.x, B2.y, B2.z, B2.w};
        const float g_[4] = {G4.x, G4.y, G4.z, G4.w};
        float c2l = 0.f;   // (b2 - w2) at column gj - 1
        if (gj > 0) c2l = __ldg(b2 + o - 1) - __ldg(w2 + o - 1);
        float out[4];
#pragma unroll
        for (int c = 0; c < ST_CT; c++) {
            const int j = gj + c;
            const float c1 = b1_[c] - w1_[c];
            const float c2 = b2_[c] - w2_[c];
            float dv = 0.f;
            if (gi < M - 1) dv += c1;
            if (gi > 0) dv -= c1p[c];
            if (j < N - 1) dv += c2;
            if (j > 0) dv -= c2l;
            c2l = c2;
            c1p[c] = c1;
            const float ps = p_[c];
            const float wn = sqrtf(w1_[c] * w1_[c] + w2_[c] * w2_[c]);
            const float wv = w1_[c] * v[i][c].x + w2_[c] * v[i][c].y;
            const float t = -a.gamma * g_[c] * wn * dpeps(ps, a.reg) + a.alpha * g_[c] * deps(ps, a.reg) +
                            2.f * a.beta * hpband(ps, a.reg) * wv + a.mu * dv;
            out[c] = ps + a.tau * t;
        }
        *reinterpret_cast<float4*>(Fo + o) = make_float4(out[0], out[1], out[2], out[3]);
    }
}

__device__ __forceinline__ void project_w(int mode, float& x, float& y) {
    const float n = sqrtf(x * x + y * y);
    if (mode == 0) {
        if (n > 1.f) { x /= n; y /= n; }
    } else if (mode == 1) {
        if (n > 1e-4f) { x /= n; y /= n; }
    }
}

// MODE 0: threshold (Eq. 41-42); MODE 1: fixed-point sweep (Eq. 38-39).  UPDATE_B: last pass,
// b += grad phi - w_new (Eq. 23) and the non-finite guard.  w_in is read for v (the halo) only in
// mode 1 beyond the pixel; in mode 0 w_in = w^k.  b is updated in place (pixel-local).
template <int R, int SHAPE, int MODE, bool UPDATE_B>
__global__ void __launch_bounds__(32 * ST_BY) k_wb(const float* __restrict__ phi, const float* __restrict__ w_in,
                                                   float* __restrict__ w_out, float* __restrict__ bv,
                                                   const float* __restrict__ g, int* __restrict__ flag,
                                                   StencilArgs a) {
    extern __shared__ float2 U[];
    const int M = a.M, N = a.N;
    const size_t plane = (size_t)M * N;
    const int img = blockIdx.z;
    const float* ph = phi + img * plane;
    const float* w1 = w_in + img * 2 * plane;
    const float* w2 = w1 + plane;
    float* o1 = w_out + img * 2 * plane;
    float* o2 = o1 + plane;
    float* b1 = bv + img * 2 * plane;
    float* b2 = b1 + plane;
    const float* gg = g + img * plane;
    const int row0 = blockIdx.y * ST_TH, col0 = blockIdx.x * ST_TW;
    stage_u<R>(U, ph, w1, w2, M, N, row0, col0, a.reg);
    __syncthreads();
    const int r0 = threadIdx.y * ST_RT, c0 = threadIdx.x * ST_CT;
    const int gj = col0 + c0;
    if (gj >= N) return;
    float2 v[ST_RT][ST_CT];
    window_block<R, SHAPE>(U, r0, c0, a.e, v);
    bool bad = false;
#pragma unroll
    for (int i = 0; i < ST_RT; i++) {
        const int gi = row0 + r0 + i;
        if (gi >= M) break;
        const size_t o = (size_t)gi * N + gj;
        const float4 P4 = __ldg(reinterpret_cast<const float4*>(ph + o));
        float4 Pn = P4;   // next row (grad component 1 is 0 on the last row)
        if (gi < M - 1) Pn = __ldg(reinterpret_cast<const float4*>(ph + o + N));
        const float pr = (gj + ST_CT < N) ? __ldg(ph + o + ST_CT) : 0.f;
        const float4 B1 = *reinterpret_cast<const float4*>(b1 + o);
        const float4 B2 = *reinterpret_cast<const float4*>(b2 + o);
        const float4 G4 = __ldg(reinterpret_cast<const float4*>(gg + o));
        const float p_[5] = {P4.x, P4.y, P4.z, P4.w, pr};
        const float pn_[4] = {Pn.x, Pn.y, Pn.z, Pn.w};
        const float b1_[4] = {B1.x, B1.y, B1.z, B1.w};
        const float b2_[4] = {B2.x, B2.y, B2.z, B2.w};
        const float g_[4] = {G4.x, G4.y, G4.z, G4.w};
        float n1[4], n2[4], nb1[4], nb2[4];
#pragma unroll
        for (int c = 0; c < ST_CT; c++) {
            const int j = gj + c;
            const float ps = p_[c];
            const float gp1 = (gi < M - 1) ? pn_[c] - ps : 0.f;
            const float gp2 = (j < N - 1) ? p_[c + 1] - ps : 0.f;
            const float hh = hband(ps, a.reg);
            float x, y;
            if (MODE == 0) {
                const float Bx = gp1 + b1_[c] + a.beta2_mu * hh * v[i][c].x;
                const float By = gp2 + b2_[c] + a.beta2_mu * hh * v[i][c].y;
                const float t = a.gamma_mu * g_[c] * deps(ps, a.reg);
                const float nb = sqrtf(Bx * Bx + By * By);
                if (nb > 0.f) {
                    const float m = fmaxf(nb - t, 0.f) / nb;
                    x = m * Bx;
                    y = m * By;
                } else {
                    x = 0.f;
                    y = 0.f;
                }
            } else {
                const float den = a.gamma * g_[c] * deps(ps, a.reg) + a.mu;
                x = (a.mu * gp1 + a.mu * b1_[c] + 2.f * a.beta * hh * v[i][c].x) / den;
                y = (a.mu * gp2 + a.mu * b2_[c] + 2.f * a.beta * hh * v[i][c].y) / den;
            }
            project_w(a.w_proj, x, y);
            n1[c] = x;
            n2[c] = y;
            nb1[c] = b1_[c] + gp1 - x;
            nb2[c] = b2_[c] + gp2 - y;
            if (UPDATE_B) {
                bad |= !(fabsf(nb1[c]) <= a.b_max && fabsf(nb2[c]) <= a.b_max) && a.b_max > 0.f;
                bad |= !isfinite(nb1[c]) || !isfinite(nb2[c]);
            }
        }
        *reinterpret_cast<float4*>(o1 + o) = make_float4(n1[0], n1[1], n1[2], n1[3]);
        *reinterpret_cast<float4*>(o2 + o) = make_float4(n2[0], n2[1], n2[2], n2[3]);
        if (UPDATE_B) {
            *reinterpret_cast<float4*>(b1 + o) = make_float4(nb1[0], nb1[1], nb1[2], nb1[3]);
            *reinterpret_cast<float4*>(b2 + o) = make_float4(nb2[0], nb2[1], nb2[2], nb2[3]);
        }
    }
    if (UPDATE_B && bad) atomicOr(flag, 1);
}

}  // namespace srsb
