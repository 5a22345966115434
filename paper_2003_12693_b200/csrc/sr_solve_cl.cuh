// sr_solve_cl.cuh -- the whole phi solve of Eq. (31)-(33) in ONE kernel for small images:
// the small-image latency path.  Three launches (k_rows_r2c, k_cols_tri, k_rows_c2r) and two
// round trips of the spectrum through L2 become one launch, with the spectrum never leaving the chip.
//
// A thread-block CLUSTER spans one image: CTA `rank` of NC owns RPC = M / NC consecutive rows.
//   1. row R2C of its rows (N/2-point complex Stockham FFT in registers + shared memory, real split) into
//      its own shared memory, row-major;
//   2. the column pass as the cyclic tridiagonal solve of sr_tri.cuh with chunk length L = RPC: one
//      thread per spectrum column runs the local recurrences over the CTA's rows and publishes the end
//      values Bf, Bb in shared memory;
//   3. cluster barrier; the carries Yin = sum_m rho^(m-1) Bf[rank - m], Zin = sum_m rho^(m-1) Bb[rank + m]
//      are read from the neighbouring CTAs through distributed shared memory (cyclic in the cluster);
//   4. forward / backward recurrences with the true carries, x in place;
//   5. inverse real FFT of its rows, phi = psi + z (increment form), clamp, store.
// Same arithmetic as the three-kernel path except the chunk length of the recurrences (RPC instead of 16),
// i.e. another rounding order of the same sums.
#pragma once
#include "sr_fft.cuh"
#include "sr_tri.cuh"

namespace srsb {

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ float2 ld_cl_f2(const float2* p, uint32_t rank) {   // p: local shared address
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(remote) : "memory");
    return v;
}

struct SolveClArgs {
    long long plane;   // floats per image plane of the real fields
    int SR;            // float2 per shared row (padded)
    float clip;        // > 0: clamp the output
    int accum;         // 1: out = out + z (increment form), 0: out = z
    int mmax;          // carry terms (<= NC)
};

// grid (NC, B), cluster (NC, 1, 1), block RPC * H / 16 threads (>= H);
// dynamic shared memory (RPC * SR + 2 H) float2.  tc: TriCol table built for chunk length RPC.
template <int LOGH, int LRPC>
__global__ void __launch_bounds__(((1 << LOGH) / 16) << LRPC) k_solve_cluster(const float* __restrict__ F, float* __restrict__ out,
                                                                             const float2* __restrict__ twH,
                                                                             const float2* __restrict__ twR,
                                                                             const TriCol* __restrict__ tc, SolveClArgs a) {
    constexpr int H = 1 << LOGH, LOGE = 4, E = 16, T = H / E, RPC = 1 << LRPC, NT = RPC * T;
    static_assert(NT >= H, "one recurrence thread per spectrum column");
    extern __shared__ float2 smem2[];
    float2* BfS = smem2 + RPC * a.SR;
    float2* BbS = BfS + H;
    const int tid = threadIdx.x, grp = tid / T, t = tid % T;
    const uint32_t rank = blockIdx.x, NC = gridDim.x;
    const int b = blockIdx.y, m0 = rank * RPC;
    float2* sm = smem2 + grp * a.SR;
    float2* orow = reinterpret_cast<float2*>(out + b * a.plane + (long long)(m0 + grp) * (2 * H));
    float2 old[E];
    if (a.accum) {
#pragma unroll
        for (int u = 0; u < E; u++) old[u] = orow[t + u * T];
    }
    {   // 1. row R2C
        const float2* x = reinterpret_cast<const float2*>(F + b * a.plane + (long long)(m0 + grp) * (2 * H));
        float2 v[E];
#pragma unroll
        for (int u = 0; u < E; u++) v[u] = __ldcs(x + t + u * T);
        fft_stages<LOGH, LOGE, 0, false>(v, sm, t, twH);
#pragma unroll
        for (int u = 0; u < E; u++) {
            SRSB_CHK(&sm[pad16(t + u * T)], 8);
            sm[pad16(t + u * T)] = v[u];
        }
    }
    __syncthreads();
    {   // real split in place: bins k2 and H - k2 of a row by one thread (slot 0 packs X[0], X[N/2])
        auto split2 = [&](float2 Za, float2 Zb, float2 tw) -> float2 {   // Zb = Z[H - k]
            const float2 Zc = conjf2(Zb);
            const float2 Ev = make_float2(0.5f * (Za.x + Zc.x), 0.5f * (Za.y + Zc.y));
            const float2 D = make_float2(0.5f * (Za.x - Zc.x), 0.5f * (Za.y - Zc.y));
            const float2 O = make_float2(D.y, -D.x);  // -i D
            const float2 wo = cmul(tw, O);
            return make_float2(Ev.x + wo.x, Ev.y + wo.y);
        };
#pragma unroll
        for (int u = 0; u < E / 2; u++) {
            const int e = tid + u * NT;
            const int k2 = e & (H / 2 - 1), rr = e >> (LOGH - 1);
            float2* row = smem2 + rr * a.SR;
            SRSB_CHK(&row[pad16(H - 1)], 8);
            if (k2 == 0) {
                const float2 A0 = row[0], B0 = row[pad16(H / 2)];
                row[0] = make_float2(A0.x + A0.y, A0.x - A0.y);
                row[pad16(H / 2)] = split2(B0, B0, __ldg(&twR[H / 2]));
            } else {
                const float2 A0 = row[pad16(k2)], B0 = row[pad16(H - k2)];
                row[pad16(k2)] = split2(A0, B0, __ldg(&twR[k2]));
                row[pad16(H - k2)] = split2(B0, A0, __ldg(&twR[H - k2]));
            }
        }
    }
    __syncthreads();
    // 2. local recurrences of column tid over the CTA's rows
    const bool colthr = tid < H;
    const TriCol* q = tc + (colthr ? tid : 0);
    const float2 r = make_float2(__ldg(&q->r[0]), __ldg(&q->r[1]));
    float2* colp = smem2 + pad16(colthr ? tid : 0);
    if (colthr) {
        float2 y = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
#pragma unroll 8
        for (int j = 0; j < RPC; j++) {
            const float2 df = colp[j * a.SR], db = colp[(RPC - 1 - j) * a.SR];
            y.x = fmaf(r.x, y.x, df.x);
            y.y = fmaf(r.y, y.y, df.y);
            z.x = fmaf(r.x, z.x, db.x);
            z.y = fmaf(r.y, z.y, db.y);
        }
        SRSB_CHK(&BbS[tid], 8);
        SRSB_CHK(&colp[(RPC - 1) * a.SR], 8);
        BfS[tid] = y;
        BbS[tid] = z;
    }
    // 3. the cluster's end values are complete
    cl_arrive();
    cl_wait();
    float2 y = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
    if (colthr) {
        const float2 rho = make_float2(__ldg(&q->rho[0]), __ldg(&q->rho[1]));
        float2 wgt = make_float2(1.f, 1.f);
        for (int m = 1; m <= a.mmax; m++) {
            const float2 f = ld_cl_f2(BfS + tid, (rank + NC - (uint32_t)m) % NC);
            const float2 bk = ld_cl_f2(BbS + tid, (rank + (uint32_t)m) % NC);
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
    cl_arrive();   // this CTA's remote reads are done (waited on before exit)
    if (colthr) {  // 4. recurrences with the true carries; y_j in registers, x_j = ks (y_j + r z_{j+1}) in place
        float2 yv[RPC];
#pragma unroll
        for (int j = 0; j < RPC; j++) {
            const float2 d = colp[j * a.SR];
            y.x = fmaf(r.x, y.x, d.x);
            y.y = fmaf(r.y, y.y, d.y);
            yv[j] = y;
        }
        const float2 ks = make_float2(__ldg(&q->ks[0]), __ldg(&q->ks[1]));
#pragma unroll
        for (int j = RPC - 1; j >= 0; j--) {
            const float2 d = colp[j * a.SR];
            colp[j * a.SR] = make_float2(ks.x * fmaf(r.x, z.x, yv[j].x), ks.y * fmaf(r.y, z.y, yv[j].y));
            z.x = fmaf(r.x, z.x, d.x);
            z.y = fmaf(r.y, z.y, d.y);
        }
    }
    __syncthreads();
    {   // 5. inverse real FFT of the CTA's rows (k_rows_c2r's arithmetic)
        float2 v[E];
#pragma unroll
        for (int u = 0; u < E; u++) {
            const int k = t + u * T;
            const float2 X = sm[pad16(k)];
            if (k == 0) {
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
        fft_stages<LOGH, LOGE, 0, true>(v, sm, t, twH);
#pragma unroll
        for (int u = 0; u < E; u++) {
            float2 zz = v[u];
            if (a.accum) {
                zz.x += old[u].x;
                zz.y += old[u].y;
            }
            if (a.clip > 0.f) {
                zz.x = fminf(fmaxf(zz.x, -a.clip), a.clip);
                zz.y = fminf(fmaxf(zz.y, -a.clip), a.clip);
            }
            orow[t + u * T] = zz;
        }
    }
    cl_wait();   // no CTA leaves while a peer may still read its end values
}

typedef void (*SolveClKernel)(const float*, float*, const float2*, const float2*, const TriCol*, SolveClArgs);
// solve_cl.cu: instance for N = 2^(log2_h + 1) and 2^lg_rpc rows per CTA, or null
SolveClKernel pick_solve_cluster(int log2_h, int lg_rpc);

}  // namespace srsb
