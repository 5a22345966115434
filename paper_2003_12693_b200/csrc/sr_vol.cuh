// sr_vol.cuh -- 3-D extension of the SB-SR iteration ("The algorithm can
// also be extended to 3D", Fig. 6; reading Q26 of DESIGN.md: every operator gains the depth
// axis z).  Volumes are [D][M][N] fp32, one volume per context; vector fields are stored as three
// planes (components along rows i, columns j, depth z).
//
//   phi solve (Eq. 31-33 in 3-D, symbol 1 + tau mu (6 - 2cos z1 - 2cos z2 - 2cos z3)):
//     k_rows_r2c over the D*M rows (sr_fft.cuh) -> k3_planes_solve: per spectrum column k2 the
//     whole D x M plane in shared memory, 2-D FFT (radix-2, bit-reversed load), divide by the
//     symbol (the packed k2 = 0 / N/2 slot unpacked with its (-k3, -k1) partner in the same
//     plane), inverse 2-D FFT -> k_rows_c2r over the D*M rows (increment form, clamp).
//   RHS (Eq. 37) and w/b update (Eq. 41-42 / 38-39, 40, 23): 4 x 8 x 32 voxel tiles, u = h(phi) w
//     staged in shared memory (three SoA planes with the R halo), the ball window summed per
//     (z, i) row with partial sums S_L built incrementally in L (exact regrouping).
//   Edge indicator (Eq. 1 in 3-D): separable Gaussian along j, i, z (replicate padding), central
//     differences; init w = grad phi0, b = 0.
#pragma once
#include <cuda_runtime.h>

#include "sr_stencil.cuh"

namespace srsb {

struct VolArgs {
    int D, M, N;
    long long vol;     // D * M * N
    Reg reg;
    float e[9];        // exp(-q^2/d^2)
    float tau, gamma, alpha, beta, mu, beta2_mu, gamma_mu;
    int w_proj;
    float b_max;
    int aos;           // unused in 3-D (FFT solver only); kept 0
    int band_skip;     // 1: ball sums only in the narrow band (exact; SRSB_BAND_SKIP=0 turns it off)
};

// ------------------------------------------------------------------ 2-D FFT of one spectrum plane
__device__ __forceinline__ int brev_bits(int v, int bits) { return bits ? (int)(__brev((unsigned)v) >> (32 - bits)) : 0; }

// padded plane index: row z of M complex + one pad slot per row (strided D-axis access)
__device__ __forceinline__ int pidx(int z, int i, int M) { return z * (M + 1) + i; }

// In-place radix-2 DIT stages along one axis of the plane (input already bit-reversed along it).
// AXIS 0: lines along i (length M = 2^lgM, D lines); AXIS 1: lines along z (length D = 2^lgD, M
// lines).  tw: the axis' twiddles exp(-2 pi i m / L), m < L/2, staged in shared memory.
template <int AXIS, bool INV>
__device__ __forceinline__ void plane_stages(float2* P, int lgD, int lgM, const float2* tw) {
    const int M = 1 << lgM;
    const int lgL = AXIS == 0 ? lgM : lgD, lgl = AXIS == 0 ? lgD : lgM;
    const int nb = 1 << (lgL - 1 + lgl);            // butterflies per stage
    for (int s = 0; s < lgL; s++) {
        const int h = 1 << s;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int line = b >> (lgL - 1), bb = b & ((1 << (lgL - 1)) - 1);
            const int k = bb & (h - 1), i0 = ((bb >> s) << (s + 1)) + k, i1 = i0 + h;
            const int a0 = AXIS == 0 ? pidx(line, i0, M) : pidx(i0, line, M);
            const int a1 = AXIS == 0 ? pidx(line, i1, M) : pidx(i1, line, M);
            float2 w = tw[k << (lgL - 1 - s)];
            if (INV) w.y = -w.y;
            const float2 x0 = P[a0], x1 = P[a1];
            const float2 t = make_float2(w.x * x1.x - w.y * x1.y, w.x * x1.y + w.y * x1.x);
            P[a0] = make_float2(x0.x + t.x, x0.y + t.y);
            P[a1] = make_float2(x0.x - t.x, x0.y - t.y);
        }
        __syncthreads();
    }
}

// bit-reverse permutation along one axis, in place
template <int AXIS>
__device__ __forceinline__ void plane_brev(float2* P, int lgD, int lgM) {
    const int M = 1 << lgM;
    const int lgL = AXIS == 0 ? lgM : lgD, lgl = AXIS == 0 ? lgD : lgM;
    if (lgL == 0) return;
    for (int e = threadIdx.x; e < (1 << (lgL + lgl)); e += blockDim.x) {
        const int line = e >> lgL, x = e & ((1 << lgL) - 1), y = brev_bits(x, lgL);
        if (x < y) {
            const int a = AXIS == 0 ? pidx(line, x, M) : pidx(x, line, M);
            const int c = AXIS == 0 ? pidx(line, y, M) : pidx(y, line, M);
            const float2 t = P[a];
            P[a] = P[c];
            P[c] = t;
        }
    }
    __syncthreads();
}

struct PlaneArgs {
    int D, M, H;
    float taumu, scale;   // scale = 1 / (D M H)
};

// ------------------------------------------------------------------ stencils
constexpr int V_TZ = 4, V_TY = 8, V_TX = 32;   // voxel tile; CTA = 32 x 8 threads, 4 z per thread

template <int R>
struct VolGeom {
    static constexpr int SZ = V_TZ + 2 * R, SY = V_TY + 2 * R, SX = V_TX + 2 * R;
    static constexpr int PLANE = SZ * SY * SX;       // floats per staged channel
    static constexpr int BYTES = 3 * PLANE * 4;
};

// ball row half-width for (r, p): floor(sqrt(R^2 - r^2 - p^2)), -1 if outside; cube: R
template <int R, int SHAPE>
__host__ __device__ constexpr int ball_half(int r, int p) {
    return SHAPE == 1 ? R : (r * r + p * p > R * R ? -1 : isqrt_c(R * R - r * r - p * p));
}

// Stage u = h(phi) w (three channels) over the tile + R halo; zero outside the volume (Q5).
template <int R, bool LEQ>
__device__ __forceinline__ void vol_stage_u(float* __restrict__ U, const float* __restrict__ phi,
                                            const float* __restrict__ w, const VolArgs& a, int z0, int y0, int x0) {
    using G = VolGeom<R>;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int k = tid; k < G::PLANE; k += 256) {
        const int zs = k / (G::SY * G::SX), rem = k - zs * (G::SY * G::SX), ys = rem / G::SX, xs = rem - ys * G::SX;
        const int z = z0 - R + zs, y = y0 - R + ys, x = x0 - R + xs;
        float u1 = 0.f, u2 = 0.f, u3 = 0.f;
        if (z >= 0 && z < a.D && y >= 0 && y < a.M && x >= 0 && x < a.N) {
            const long long o = ((long long)z * a.M + y) * a.N + x;
            const float h = reg_h<LEQ>(__ldg(phi + o), a.reg);
            u1 = h * __ldg(w + o);
            u2 = h * __ldg(w + a.vol + o);
            u3 = h * __ldg(w + 2 * a.vol + o);
        }
        U[k] = u1;
        U[G::PLANE + k] = u2;
        U[2 * G::PLANE + k] = u3;
    }
}

// v for the thread's 4 voxels (z0 + 0..3, y, x): ball sum by rows with incremental partial sums
template <int R, int SHAPE>
__device__ __forceinline__ void vol_window(const float* __restrict__ U, const float* e, float (&v)[V_TZ][3]) {
    using G = VolGeom<R>;
    const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
    for (int zz = 0; zz < V_TZ; zz++) v[zz][0] = v[zz][1] = v[zz][2] = 0.f;
#pragma unroll
    for (int zs = 0; zs < G::SZ; zs++) {
#pragma unroll
        for (int p = -R; p <= R; p++) {
            const int row = (zs * G::SY + ty + R + p) * G::SX + tx + R;
            float S[3][R + 1];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const float* Uc = U + c * G::PLANE + row;
                float acc = e[0] * Uc[0];
                S[c][0] = acc;
#pragma unroll
                for (int q = 1; q <= R; q++) {
                    acc = fmaf(e[q], Uc[-q] + Uc[q], acc);
                    S[c][q] = acc;
                }
            }
#pragma unroll
            for (int zz = 0; zz < V_TZ; zz++) {
                const int r = zs - R - zz;
                if (r < -R || r > R) continue;
                const int L = ball_half<R, SHAPE>(r < 0 ? -r : r, p < 0 ? -p : p);
                if (L < 0) continue;
                const float wgt = e[r < 0 ? -r : r] * e[p < 0 ? -p : p];
#pragma unroll
                for (int c = 0; c < 3; c++) v[zz][c] = fmaf(wgt, S[c][L], v[zz][c]);
            }
        }
    }
}

// Narrow band in 3-D (as needs_v in sr_stencil.cuh): the thread's V_TZ voxels (z0 + 0..3, y, x) that
// lie in the volume need v only where h / h' != 0; a tile none of whose voxels does skips the staging.
template <bool LEQ>
__device__ __forceinline__ bool vol_needs_v(const float* __restrict__ phi, const VolArgs& a, int z0, int y, int x) {
    if (x >= a.N || y >= a.M) return false;
    bool need = false;
#pragma unroll
    for (int zz = 0; zz < V_TZ; zz++) {
        const int z = z0 + zz;
        if (z >= a.D) break;
        need |= needs_v<LEQ>(__ldg(phi + ((long long)z * a.M + y) * a.N + x), a.reg);
    }
    return need;
}
template <int R, int SHAPE, bool LEQ>
__device__ __forceinline__ void vol_v(float* U, const float* __restrict__ phi, const float* __restrict__ w,
                                      const VolArgs& a, int z0, int y0, int x0, float (&v)[V_TZ][3]) {
#pragma unroll
    for (int zz = 0; zz < V_TZ; zz++) v[zz][0] = v[zz][1] = v[zz][2] = 0.f;
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    const bool own = !a.band_skip || vol_needs_v<LEQ>(phi, a, z0, y, x);
    if (__syncthreads_or(own)) {
        vol_stage_u<R, LEQ>(U, phi, w, a, z0, y0, x0);
        __syncthreads();
        if (own && x < a.N && y < a.M) vol_window<R, SHAPE>(U, a.e, v);
    }
}

// Eq. (37) in 3-D, increment form: D = tau [ -gamma g |w| delta' + alpha g delta
//   + 2 beta h' w.v + mu div(b - w) + mu Delta_per psi ].
template <int R, int SHAPE, bool LEQ>
__global__ void __launch_bounds__(256) k3_rhs(const float* __restrict__ phi, const float* __restrict__ w,
                                              const float* __restrict__ b, const float* __restrict__ g,
                                              float* __restrict__ Dout, VolArgs a) {
    extern __shared__ float4 smem_v4[];
    float* U = reinterpret_cast<float*>(smem_v4);
    const int x0 = blockIdx.x * V_TX, y0 = blockIdx.y * V_TY, z0 = blockIdx.z * V_TZ;
    float v[V_TZ][3];
    vol_v<R, SHAPE, LEQ>(U, phi, w, a, z0, y0, x0, v);
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= a.N || y >= a.M) return;
    const int D = a.D, M = a.M, N = a.N;
    const long long V = a.vol;
#pragma unroll
    for (int zz = 0; zz < V_TZ; zz++) {
        const int z = z0 + zz;
        if (z >= D) break;
        const long long o = ((long long)z * M + y) * N + x;
        const float ps = __ldg(phi + o);
        // periodic 7-point Laplacian (Eq. 32's operator), neighbour differences first
        const int zp = (z + 1) & (D - 1), zm = (z - 1) & (D - 1), yp = (y + 1) & (M - 1), ym = (y - 1) & (M - 1);
        const int xp = (x + 1) & (N - 1), xm = (x - 1) & (N - 1);
        const float lap = ((__ldg(phi + ((long long)z * M + yp) * N + x) - ps) + (__ldg(phi + ((long long)z * M + ym) * N + x) - ps)) +
                          ((__ldg(phi + ((long long)z * M + y) * N + xp) - ps) + (__ldg(phi + ((long long)z * M + y) * N + xm) - ps)) +
                          ((__ldg(phi + ((long long)zp * M + y) * N + x) - ps) + (__ldg(phi + ((long long)zm * M + y) * N + x) - ps));
        // div(b - w), Eq. (36) per axis (Neumann adjoint, Q6)
        const float w1 = __ldg(w + o), w2 = __ldg(w + V + o), w3 = __ldg(w + 2 * V + o);
        float dv = 0.f;
        if (y < M - 1) dv += __ldg(b + o) - w1;
        if (y > 0) dv -= __ldg(b + o - N) - __ldg(w + o - N);
        if (x < N - 1) dv += __ldg(b + V + o) - w2;
        if (x > 0) dv -= __ldg(b + V + o - 1) - __ldg(w + V + o - 1);
        if (z < D - 1) dv += __ldg(b + 2 * V + o) - w3;
        if (z > 0) dv -= __ldg(b + 2 * V + o - (long long)M * N) - __ldg(w + 2 * V + o - (long long)M * N);
        const float gg = __ldg(g + o);
        const float wn = sqrtf(w1 * w1 + w2 * w2 + w3 * w3);
        const float wv = w1 * v[zz][0] + w2 * v[zz][1] + w3 * v[zz][2];
        const RegVals rv = reg_all<LEQ>(ps, a.reg);
        const float t = -a.gamma * gg * wn * rv.dp + a.alpha * gg * rv.d + 2.f * a.beta * rv.hp * wv + a.mu * dv;
        Dout[o] = a.tau * (t + a.mu * lap);
    }
}

__device__ __forceinline__ void project3(int mode, float& x, float& y, float& z) {
    const float n2 = x * x + y * y + z * z;
    if ((mode == 0 && n2 > 1.f) || (mode == 1 && n2 > 1e-8f)) {
        const float n = sqrtf(n2);   // IEEE sqrt and divides (Q20)
        x = x / n;
        y = y / n;
        z = z / n;
    }
}

// w/b update in 3-D.  MODE 0: Eq. (41)-(42); MODE 1: one fixed-point pass of Eq. (38)-(39).
template <int R, int SHAPE, int MODE, bool UPDATE_B, bool LEQ>
__global__ void __launch_bounds__(256) k3_wb(const float* __restrict__ phi, const float* __restrict__ w_in,
                                             float* __restrict__ w_out, float* __restrict__ b,
                                             const float* __restrict__ g, int* __restrict__ flag, VolArgs a) {
    extern __shared__ float4 smem_v4[];
    float* U = reinterpret_cast<float*>(smem_v4);
    const int x0 = blockIdx.x * V_TX, y0 = blockIdx.y * V_TY, z0 = blockIdx.z * V_TZ;
    float v[V_TZ][3];
    vol_v<R, SHAPE, LEQ>(U, phi, w_in, a, z0, y0, x0, v);
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= a.N || y >= a.M) return;
    const int D = a.D, M = a.M, N = a.N;
    const long long V = a.vol;
    bool bad = false;
#pragma unroll
    for (int zz = 0; zz < V_TZ; zz++) {
        const int z = z0 + zz;
        if (z >= D) break;
        const long long o = ((long long)z * M + y) * N + x;
        const float ps = __ldg(phi + o);
        const float gp1 = y < M - 1 ? __ldg(phi + o + N) - ps : 0.f;
        const float gp2 = x < N - 1 ? __ldg(phi + o + 1) - ps : 0.f;
        const float gp3 = z < D - 1 ? __ldg(phi + o + (long long)M * N) - ps : 0.f;
        const float b1 = b[o], b2 = b[V + o], b3 = b[2 * V + o];
        const float gg = __ldg(g + o);
        float hh, dd;
        reg_hd<LEQ>(ps, a.reg, hh, dd);
        float n1, n2, n3;
        if (MODE == 0) {
            const float B1 = gp1 + b1 + a.beta2_mu * hh * v[zz][0];
            const float B2 = gp2 + b2 + a.beta2_mu * hh * v[zz][1];
            const float B3 = gp3 + b3 + a.beta2_mu * hh * v[zz][2];
            const float t = a.gamma_mu * gg * dd;
            const float nb = B1 * B1 + B2 * B2 + B3 * B3;
            if (nb > 0.f) {
                const float sn = sqrtf(nb);
                const float m = fmaxf(sn - t, 0.f) / sn;   // IEEE (Q20)
                n1 = m * B1;
                n2 = m * B2;
                n3 = m * B3;
            } else {
                n1 = n2 = n3 = 0.f;
            }
        } else {
            const float den = a.gamma * gg * dd + a.mu;
            n1 = (a.mu * gp1 + a.mu * b1 + 2.f * a.beta * hh * v[zz][0]) / den;
            n2 = (a.mu * gp2 + a.mu * b2 + 2.f * a.beta * hh * v[zz][1]) / den;
            n3 = (a.mu * gp3 + a.mu * b3 + 2.f * a.beta * hh * v[zz][2]) / den;
        }
        project3(a.w_proj, n1, n2, n3);
        w_out[o] = n1;
        w_out[V + o] = n2;
        w_out[2 * V + o] = n3;
        if (UPDATE_B) {
            const float c1 = b1 + gp1 - n1, c2 = b2 + gp2 - n2, c3 = b3 + gp3 - n3;
            b[o] = c1;
            b[V + o] = c2;
            b[2 * V + o] = c3;
            bad |= !(fabsf(c1) <= a.b_max && fabsf(c2) <= a.b_max && fabsf(c3) <= a.b_max) && a.b_max > 0.f;
            bad |= !isfinite(c1) || !isfinite(c2) || !isfinite(c3);
        }
    }
    if (UPDATE_B && bad) atomicOr(flag, 1);
}

#ifdef SRSB_VOL_HOST_KERNELS   // non-template kernels: defined in srsb3.cu only
// grid = H (one spectrum column k2 per CTA), dynamic smem D (M + 1) + (M + D) / 2 float2.
// spec[k2][z * M + i] (the row pass's layout with G = 1 over the D*M rows).
__global__ void __launch_bounds__(1024) k3_planes_solve(float2* __restrict__ spec, const float2* __restrict__ twM,
                                                        const float2* __restrict__ twD, const float* __restrict__ cM,
                                                        const float* __restrict__ cD, const float* __restrict__ cN,
                                                        PlaneArgs a) {
    extern __shared__ float4 smem_v4[];
    float2* P = reinterpret_cast<float2*>(smem_v4);
    const int D = a.D, M = a.M, k2 = blockIdx.x;
    const int lgD = __ffs(D) - 1, lgM = __ffs(M) - 1;
    float2* tM = P + D * (M + 1);
    float2* tD = tM + M / 2;
    for (int m = threadIdx.x; m < M / 2; m += blockDim.x) tM[m] = __ldg(&twM[m]);
    for (int m = threadIdx.x; m < D / 2; m += blockDim.x) tD[m] = __ldg(&twD[m]);
    float2* col = spec + (long long)k2 * D * M;
    // load with the i-axis bit reversal folded in
    for (int e = threadIdx.x; e < D * M; e += blockDim.x) {
        const int z = e >> lgM, i = e & (M - 1);
        P[pidx(z, brev_bits(i, lgM), M)] = col[e];
    }
    __syncthreads();
    plane_stages<0, false>(P, lgD, lgM, tM);
    plane_brev<1>(P, lgD, lgM);
    plane_stages<1, false>(P, lgD, lgM, tD);
    // divide by the symbol (Eq. 32 in 3-D); k2 = 0 holds (X[.., 0], X[.., N/2]) packed as Z = A + iB
    const float cn = __ldg(&cN[k2]);
    if (k2 != 0) {
        for (int e = threadIdx.x; e < D * M; e += blockDim.x) {
            const int z = e >> lgM, i = e & (M - 1);
            const float s = a.scale / (1.f + a.taumu * (__ldg(&cD[z]) + __ldg(&cM[i]) + cn));
            float2& v = P[pidx(z, i, M)];
            v = make_float2(v.x * s, v.y * s);
        }
    } else {
        const float c0 = __ldg(&cN[0]), ch = __ldg(&cN[a.H]);
        for (int e = threadIdx.x; e < D * M; e += blockDim.x) {   // each (k, -k) pair once
            const int z = e >> lgM, i = e & (M - 1);
            const int zn = (D - z) & (D - 1), in = (M - i) & (M - 1);
            const int e2 = zn * M + in;
            if (e2 < e) continue;
            const float cc = __ldg(&cD[z]) + __ldg(&cM[i]);   // the same for the partner (even symbol)
            const float s0 = a.scale / (1.f + a.taumu * (cc + c0)), sh = a.scale / (1.f + a.taumu * (cc + ch));
            const float p = 0.5f * (s0 + sh), m = 0.5f * (s0 - sh);
            const float2 C = P[pidx(z, i, M)], C2 = P[pidx(zn, in, M)];
            // v(k) = p C(k) + m conj(C(-k)), v(-k) = p C(-k) + m conj(C(k))
            P[pidx(z, i, M)] = make_float2(p * C.x + m * C2.x, p * C.y - m * C2.y);
            if (e2 != e) P[pidx(zn, in, M)] = make_float2(p * C2.x + m * C.x, p * C2.y - m * C.y);
        }
    }
    __syncthreads();
    plane_brev<0>(P, lgD, lgM);
    plane_brev<1>(P, lgD, lgM);
    plane_stages<0, true>(P, lgD, lgM, tM);
    plane_stages<1, true>(P, lgD, lgM, tD);
    for (int e = threadIdx.x; e < D * M; e += blockDim.x) {
        const int z = e >> lgM, i = e & (M - 1);
        col[e] = P[pidx(z, i, M)];
    }
}

// ------------------------------------------------------------------ one-time kernels
// separable normalized Gaussian along AXIS (0: j, 1: i, 2: z) with replicate padding
__global__ void k3_blur(const float* __restrict__ in, float* __restrict__ out, int D, int M, int N, int axis, int r,
                        const float* __restrict__ k) {
    const long long n = (long long)D * M * N;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(q % N), y = (int)((q / N) % M), z = (int)(q / ((long long)M * N));
        float acc = 0.f;
        for (int t = -r; t <= r; t++) {
            int xx = x, yy = y, zz = z;
            if (axis == 0) xx = min(max(x + t, 0), N - 1);
            else if (axis == 1) yy = min(max(y + t, 0), M - 1);
            else zz = min(max(z + t, 0), D - 1);
            acc = fmaf(__ldg(&k[t + r]), __ldg(in + ((long long)zz * M + yy) * N + xx), acc);
        }
        out[q] = acc;
    }
}

// Eq. (1) step 2 in 3-D: central differences (replicate padding), g = 1 / (1 + rho |grad|^s)
__global__ void k3_edge_g(const float* __restrict__ fs, float* __restrict__ g, int D, int M, int N, float rho, int s) {
    const long long n = (long long)D * M * N;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(q % N), y = (int)((q / N) % M), z = (int)(q / ((long long)M * N));
        auto at = [&](int zz, int yy, int xx) { return __ldg(fs + ((long long)zz * M + yy) * N + xx); };
        const float gx = 0.5f * (at(z, min(y + 1, M - 1), x) - at(z, max(y - 1, 0), x));
        const float gy = 0.5f * (at(z, y, min(x + 1, N - 1)) - at(z, y, max(x - 1, 0)));
        const float gz = 0.5f * (at(min(z + 1, D - 1), y, x) - at(max(z - 1, 0), y, x));
        const float m2 = gx * gx + gy * gy + gz * gz;
        g[q] = 1.f / (1.f + rho * (s == 2 ? m2 : sqrtf(m2)));
    }
}

// Alg. 1 (1) in 3-D: w = grad phi0 (forward differences, 0 on the last index per axis), b = 0
__global__ void k3_init_w(const float* __restrict__ phi, float* __restrict__ w, float* __restrict__ b, int D, int M,
                          int N) {
    const long long n = (long long)D * M * N;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(q % N), y = (int)((q / N) % M), z = (int)(q / ((long long)M * N));
        const float c = phi[q];
        w[q] = y < M - 1 ? phi[q + N] - c : 0.f;
        w[n + q] = x < N - 1 ? phi[q + 1] - c : 0.f;
        w[2 * n + q] = z < D - 1 ? phi[q + (long long)M * N] - c : 0.f;
        b[q] = 0.f;
        b[n + q] = 0.f;
        b[2 * n + q] = 0.f;
    }
}

#endif  // SRSB_VOL_HOST_KERNELS

}  // namespace srsb
