// sr_fused.cuh -- the RHS of Eq. (37) fused with the row R2C pass of the phi solve (sm_100a).
//
// k_rhs_r2c = k_rhs_tma's tile work (TMA-staged phi, w, b, g; u = h(phi) w; window sums of P:368;
// the pointwise increment form of Eq. (37)) + k_rows_r2c's row transform, with the
// increment D never leaving the chip (SURVEY §8(d)'s fused layout: 28 instead of 36 B/px per sweep).
//
// A thread-block CLUSTER spans one band of TH = 32 image rows: its N / 64 CTAs are the band's
// 32 x 64 tiles (cluster rank = tile column).  Each CTA computes D for its tile into registers,
// parks it in its own shared memory, and after a cluster barrier gathers its share of the band's
// rows -- 32 / (N/64) whole rows -- from the N / 64 tiles through distributed shared memory
// (ld.shared::cluster).  64 threads then run the N/2-point complex Stockham FFT of those rows
// (fft_stages, E = 16 values per thread, named barrier), the real-FFT split, and store the packed
// half spectrum transposed and contiguous per column (spec[b][k2][m], the G = 1 layout of
// k_rows_r2c), bitwise the values k_rhs_tma -> k_rows_r2c produce (same arithmetic, same order).
// Every thread arrives on a second cluster barrier after its remote reads and waits on it before
// exiting, so no CTA's shared memory disappears under a peer's gather.
#pragma once
#include <cooperative_groups.h>
#include "sr_fft.cuh"
#include "sr_stencil.cuh"

namespace srsb {

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// 8-byte load from the shared memory of CTA `rank` of the cluster at the same offset as local `p`
__device__ __forceinline__ float2 ld_dsmem_f2(const float* p, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(remote) : "memory");
    return v;
}

template <int R, int SHAPE, bool LEQ, int LOGH>
__global__ void __launch_bounds__(256, SRSB_TMA_MINB) k_rhs_r2c(const __grid_constant__ RhsMaps maps,
                                                                const float* __restrict__ phi,
                                                                float2* __restrict__ spec,
                                                                const float2* __restrict__ twH,
                                                                const float2* __restrict__ twR, StencilArgs a, int SR) {
    using G = TmaGeom<R>;
    constexpr int H = 1 << LOGH, E = H < 16 ? H : 16, LOGE = LOGH < 4 ? LOGH : 4, T = H / E;
    constexpr int NCT = (2 * H) / G::TW;          // CTAs per band = cluster size
    constexpr int RPC = G::TH / NCT;              // band rows transformed per CTA
    constexpr int NFT = RPC * T;                  // threads running the transforms
    static_assert(NCT >= 1 && G::TH % NCT == 0 && NFT % 32 == 0 && NFT <= 256, "fused shape");
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
    float* Dt = reinterpret_cast<float*>(sm + G::O_P);            // [TH][TW] tile of D (after the reads)
    float2* Fr = reinterpret_cast<float2*>(sm + G::O_W1);         // RPC padded FFT rows of SR float2
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
    const int M = a.M, N = a.N;
    const bool active = col0 + c0 < N && row0 + r0 < M;
    const bool own = !a.band_skip || (active && block_needs_v<LEQ, G>(Ps, r0, c0, row0, M, a.reg));
    float2 v[G::RT][ST_CT];
    zero_v<G::RT>(v);
    if (__syncthreads_or(own)) {
        stage_u_tma<R, LEQ, G>(U, Ps, W1s, W2s, row0, tid, a);
        __syncthreads();
        if (active && own) window_block<R, SHAPE, G::RT, G::LDC>(U, r0, c0, a.e, v);
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[1], G::TX2);
        tma_load_3d(B1s, &maps.b, &bar[1], col0 - 4, ar - 1, 2 * img);
        tma_load_3d(B2s, &maps.b, &bar[1], col0 - 4, ar - 1, 2 * img + 1);
        tma_load_3d(Gs, &maps.g, &bar[1], col0, ar, img);
    }
    float2 res[G::RT];
    if (active) {
        mbar_wait(&bar[1], 0);
        const bool edge = row0 + a.row_off == 0 || row0 + G::TH + a.row_off >= a.Mg || row0 + G::TH > M ||
                          col0 == 0 || col0 + G::TW >= N;
        if (edge)
            rhs_points_tma<R, LEQ, true, G, true>(Ps, W1s, W2s, B1s, B2s, Gs, phi, nullptr, v, img, row0, r0, c0,
                                                  col0, a, res);
        else
            rhs_points_tma<R, LEQ, false, G, true>(Ps, W1s, W2s, B1s, B2s, Gs, phi, nullptr, v, img, row0, r0, c0,
                                                   col0, a, res);
    }
    __syncthreads();   // every read of the staged boxes is done: the P region takes the tile of D
    if (active) {
#pragma unroll
        for (int i = 0; i < G::RT; i++)
            if (row0 + r0 + i < M) {
                SRSB_CHK(Dt + (r0 + i) * G::TW + c0, 8);
                *reinterpret_cast<float2*>(Dt + (r0 + i) * G::TW + c0) = res[i];
            }
    }
    // the band's tiles of D are complete in the cluster's shared memory
    cluster_arrive();
    cluster_wait();
    const uint32_t q = blockIdx.x;               // cluster rank (the cluster spans the band's tiles)
    if (tid < NFT) {
        const int grp = tid / T, t = tid - grp * T;
        const int br = q * RPC + grp;            // band row of this transform
        // gather: complex element k = t + u T is the real pair (2k, 2k + 1) of band row br, held by
        // tile (2k) / TW at local column (2k) % TW
        float2 x[E];
#pragma unroll
        for (int u = 0; u < E; u++) {
            const int k2 = 2 * (t + u * T);
            SRSB_CHK(Dt + br * G::TW + (k2 % G::TW), 8);
            x[u] = ld_dsmem_f2(Dt + br * G::TW + (k2 % G::TW), (uint32_t)(k2 / G::TW));
        }
        cluster_arrive();                        // this thread's remote reads are done
        float2* srow = Fr + grp * SR;
        SRSB_CHK(srow, SR * 8);
        fft_stages<LOGH, LOGE, 0, false, NFT>(x, srow, t, twH);
#pragma unroll
        for (int u = 0; u < E; u++) srow[pad16(t + u * T)] = x[u];
        fft_bar<NFT>();
        // real split and transposed store: bins k2 and H - k2 of rows 2 rp, 2 rp + 1 (16-byte stores),
        // the same formulas as k_rows_r2c's mirrored split
        float2* out = spec + (size_t)img * H * M;
        const int m0 = row0 + q * RPC;
        auto split2 = [&](float2 Za, float2 Zb, float2 tw) -> float2 {   // Zb = Z[H - k]
            const float2 Zc = conjf2(Zb);
            const float2 Ev = make_float2(0.5f * (Za.x + Zc.x), 0.5f * (Za.y + Zc.y));
            const float2 D = make_float2(0.5f * (Za.x - Zc.x), 0.5f * (Za.y - Zc.y));
            const float2 O = make_float2(D.y, -D.x);  // -i D
            const float2 wo = cmul(tw, O);
            return make_float2(Ev.x + wo.x, Ev.y + wo.y);
        };
        constexpr int NP = RPC / 2, TOT = NP * (H / 2);
        for (int e = tid; e < TOT; e += NFT) {
            const int rp = e % NP, k2 = e / NP;
            if (m0 + 2 * rp >= M) continue;
            const float2* ra = Fr + (2 * rp) * SR;
            const float2* rb = ra + SR;
            float2 X0, X1, Y0, Y1;
            if (k2 == 0) {
                const float2 A0 = ra[0], A1 = rb[0];
                X0 = make_float2(A0.x + A0.y, A0.x - A0.y);  // (X[0], X[N/2]) packed
                X1 = make_float2(A1.x + A1.y, A1.x - A1.y);
                const float2 th = __ldg(&twR[H / 2]);
                const float2 B0 = ra[pad16(H / 2)], B1 = rb[pad16(H / 2)];
                Y0 = split2(B0, B0, th);
                Y1 = split2(B1, B1, th);
            } else {
                const float2 t1 = __ldg(&twR[k2]), t2 = __ldg(&twR[H - k2]);
                const float2 A0 = ra[pad16(k2)], B0 = ra[pad16(H - k2)];
                const float2 A1 = rb[pad16(k2)], B1 = rb[pad16(H - k2)];
                X0 = split2(A0, B0, t1);
                X1 = split2(A1, B1, t1);
                Y0 = split2(B0, A0, t2);
                Y1 = split2(B1, A1, t2);
            }
            const int k2m = k2 == 0 ? H / 2 : H - k2;
            *reinterpret_cast<float4*>(out + (size_t)k2 * M + m0 + 2 * rp) = make_float4(X0.x, X0.y, X1.x, X1.y);
            *reinterpret_cast<float4*>(out + (size_t)k2m * M + m0 + 2 * rp) = make_float4(Y0.x, Y0.y, Y1.x, Y1.y);
        }
    } else {
        cluster_arrive();
    }
    cluster_wait();                              // no CTA leaves while a peer may still read its tile
}

}  // namespace srsb
