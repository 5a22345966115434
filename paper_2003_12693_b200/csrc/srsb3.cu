// srsb3.cu -- host side of the 3-D extension (include/srsb.h "3-D"): one
// D x M x N volume per context, the same parameters as the 2-D library (sr_sb_params; M, N the
// in-plane sizes, batch = 1), FFT phi solver only.
//
// Per outer iteration: S x (k3_rhs -> phi solve -> ) + k3_wb passes; the phi solve (Eq. 31-33 in 3-D) is
//   k_rows_r2c over the D*M rows (FFT along j) -> k_lines_fft (FFT along i of every (k2, z) line) -> k3_unpack0
//   (the packed k2 = 0 / N/2 plane split into two planes) -> k_cols_tri_rm along z (cyclic tridiagonal solve per
//   (k1, k2)) -> k3_repack0 -> k_lines_fft inverse -> k_rows_c2r: any D >= 16, M >= 32;
//   smaller volumes (or SRSB_VOL_SOLVE=plane) keep k3_planes_solve, one D x M plane in shared memory; captured once in a CUDA graph of 2 iterations (the w
// ping-pong parity), replayed by sr_sb3_iterate.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/srsb.h"
#include "sr_kernels.h"
#include "sr_tri.cuh"
#define SRSB_VOL_HOST_KERNELS
#include "sr_vol3.h"

using namespace srsb;

// Plane 0 of the transposed spectrum after the FFT along i: Z = FFT_i(X0 + i XH), X0 / XH the real k2 = 0 / N/2
// columns of the row pass's packed slot.  A = FFT_i(X0) = (Z[k] + conj Z[-k]) / 2 stays in plane 0,
// B = FFT_i(XH) = (Z[k] - conj Z[-k]) / (2i) goes to plane H, so the z solve sees H + 1 ordinary planes.
// One thread per (z, k <= M/2) pair (k, M - k); in place.
__global__ void k3_unpack0(float2* __restrict__ P0, float2* __restrict__ PH, int D, int M) {
    const int half = M / 2 + 1;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)D * half) return;
    const int z = (int)(e / half), k = (int)(e % half), kn = (M - k) & (M - 1);
    const long long ik = (long long)z * M + k, in = (long long)z * M + kn;
    const float2 Zk = P0[ik], Zn = P0[in];
    const float2 A = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
    const float2 B = make_float2(0.5f * (Zk.y + Zn.y), -0.5f * (Zk.x - Zn.x));
    P0[ik] = A;
    PH[ik] = B;
    if (kn != k) {
        P0[in] = make_float2(A.x, -A.y);
        PH[in] = make_float2(B.x, -B.y);
    }
}
// ... and back: Z = A + i B into plane 0
__global__ void k3_repack0(float2* __restrict__ P0, const float2* __restrict__ PH, long long n) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const float2 A = P0[e], B = PH[e];
    P0[e] = make_float2(A.x - B.y, A.y + B.x);
}

struct sr_sb3_ctx {
    sr_sb_params p;
    int D = 0, device = 0;
    cudaStream_t user = nullptr, s = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    long long vol = 0;
    float *phi = nullptr, *F = nullptr, *w[2] = {nullptr, nullptr}, *b = nullptr, *g = nullptr, *tmp = nullptr;
    float2* spec = nullptr;
    float2* spec2 = nullptr;           // lines path: (H + 1) planes, the z solve is out of place
    TriCol* tri_tab = nullptr;         // [(H + 1)][M] constants of the z recurrences
    bool lines = false;                // FFT along j and i + tridiagonal solve along z (any size); else the plane solve
    LinesFftKernel lfwd = nullptr, linv = nullptr;
    ColTriRmKernel tri = nullptr;
    int l_lg_cpc = 0, l_threads = 0, l_smem = 0, l_sc = 0, l_grid = 0;
    dim3 t_grid;
    int t_threads = 0, t_smem = 0, t_mmax = 0;
    float2 *twH = nullptr, *twR = nullptr, *twM = nullptr, *twD = nullptr;
    float *cM = nullptr, *cD = nullptr, *cN = nullptr, *blurk = nullptr;
    int* flag = nullptr;
    int wcur = 0, rblur = 0;
    long long k = 0;
    bool have_state = false;
    RowKernel rfwd = nullptr;
    RowInvKernel rinv = nullptr;
    VolRhsKernel rhs = nullptr;
    VolWbKernel wb[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    FftRowArgs ra{};
    PlaneArgs pa{};
    VolArgs va{};
    dim3 rgrid, rblock, vgrid, vblock;
    int rsmem = 0, psmem = 0, vsmem = 0, pthreads = 0;
    cudaGraphExec_t graph = nullptr;
    int graph_wcur = -1;
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_cls;
    std::string err;
};

namespace {

thread_local std::string g3_create_err;

sr_status fail3(sr_sb3_ctx* c, sr_status st, const std::string& m) {
    if (c) c->err = m;
    return st;
}

#define CK3(call)                                                                                \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail3(c, SR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
    } while (0)
#define RET3(x)                      \
    do {                             \
        sr_status r_ = (x);          \
        if (r_ != SR_OK) return r_;  \
    } while (0)

bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }
int lg2(int v) {
    int r = 0;
    while ((1 << r) < v) r++;
    return r;
}

struct Dev3 {
    int prev = -1;
    explicit Dev3(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~Dev3() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

sr_status validate3(const sr_sb_params* p, int D, std::string& m) {
    if (!p) { m = "params is NULL"; return SR_ERR_ARG; }
    if (!pow2(p->M) || !pow2(p->N) || !pow2(D) || p->M < 8 || p->N < 8 || p->N > 8192 || D > 1024) {
        m = "D, M, N must be powers of two (M, N >= 8, N <= 8192, D <= 1024)";
        return SR_ERR_SHAPE;
    }
    if (p->batch != 1) { m = "3-D contexts hold one volume (batch = 1)"; return SR_ERR_SHAPE; }
    if (!(p->tau >= 0.f) || !(p->mu > 0.f) || !(p->epsilon > 0.f) || !(p->d > 0.f) || !(p->sigma > 0.f) ||
        !(p->l >= 0.f) || !(p->rho >= 0.f)) {
        m = "need tau >= 0, mu > 0, epsilon > 0, d > 0, sigma > 0, l >= 0, rho >= 0";
        return SR_ERR_ARG;
    }
    if ((int)std::ceil(3.0 * p->sigma) > 8) { m = "sigma too large"; return SR_ERR_ARG; }
    if (p->window < 0 || p->window > kMaxWindow3) { m = "3-D window radius must be in [0, 4]"; return SR_ERR_ARG; }
    if (p->window_shape != SR_WIN_DISC && p->window_shape != SR_WIN_SQUARE) { m = "bad window_shape"; return SR_ERR_ARG; }
    if (p->S < 1) { m = "S must be >= 1"; return SR_ERR_ARG; }
    if (p->s != 1 && p->s != 2) { m = "s must be 1 or 2"; return SR_ERR_ARG; }
    if (p->w_proj < 0 || p->w_proj > 2) { m = "bad w_proj"; return SR_ERR_ARG; }
    if (p->w_mode != SR_W_THRESHOLD && p->w_mode != SR_W_FIXED_POINT) { m = "bad w_mode"; return SR_ERR_ARG; }
    if (p->w_mode == SR_W_FIXED_POINT && p->w_iters < 1) { m = "w_iters must be >= 1"; return SR_ERR_ARG; }
    if (p->phi_clip < 0.f) { m = "phi_clip must be >= 0"; return SR_ERR_ARG; }
    if (p->phi_solver != SR_PHI_FFT) { m = "3-D contexts use the FFT phi solver"; return SR_ERR_ARG; }
    return SR_OK;
}

sr_status configure3(sr_sb3_ctx* c) {
    const sr_sb_params& p = c->p;
    const int D = c->D, M = p.M, N = p.N, H = N / 2, rows = D * M;
    c->vol = (long long)D * M * N;
    c->rfwd = pick_row_fwd(lg2(H));
    c->rinv = pick_row_inv(lg2(H));
    if (!c->rfwd || !c->rinv) return fail3(c, SR_ERR_SHAPE, "no FFT kernel for this N");
    // row passes over the D*M rows, G = 1 (spectrum column k2 = one contiguous D x M plane)
    const int E_h = H < 16 ? H : 16, T_h = H / E_h;
    int rpc = 8;
    while (rpc * T_h < 64 && rpc < 32) rpc <<= 1;
    while ((rpc * T_h > 512 || rpc * (H + H / 16 + 32) * 8 > 72 * 1024) && rpc > 1) rpc >>= 1;
    if (rpc > rows) rpc = rows;
    int sr = H + (H >> 4);
    sr = ((sr + 15) & ~15) + 1;
    c->ra.plane = c->vol;
    c->ra.M = rows;
    c->ra.lg_rpc = lg2(rpc);
    c->ra.lg_G = 0;
    c->ra.SR = sr;
    c->ra.clip = 0.f;
    c->ra.accum = 0;
    c->ra.stats = nullptr;
    c->rgrid = dim3(rows / rpc, 1, 1);
    c->rblock = dim3(rpc * T_h, 1, 1);
    c->rsmem = rpc * sr * (int)sizeof(float2);
    CK3(cudaFuncSetAttribute((const void*)c->rfwd, cudaFuncAttributeMaxDynamicSharedMemorySize, c->rsmem));
    CK3(cudaFuncSetAttribute((const void*)c->rinv, cudaFuncAttributeMaxDynamicSharedMemorySize, c->rsmem));
    {   // solve path: lines (general) or plane (small volumes)
        const char* ev = std::getenv("SRSB_VOL_SOLVE");
        const int L = 1 << kTriLogL;
        c->lines = false;
        if (D >= L && M >= 32 && !(ev && ev[0] == 'p')) {
            const double a = (double)p.tau * (double)p.mu;
            const double r0 = tri_ratio(a, 1.0 + 2.0 * a, nullptr);   // (k1, k2) = (0, 0): the slowest decay
            const int mm = tri_carry_terms(std::pow(r0, L), D / L, nullptr);
            c->lfwd = pick_lines_fft(lg2(M), false);
            c->linv = pick_lines_fft(lg2(M), true);
            if (mm <= kTriRmMaxCarry && c->lfwd && c->linv) {
                c->lines = true;
                c->t_mmax = mm;
            }
        }
        const bool plane_fits = (long long)(D * (M + 1) + M / 2 + D / 2 + 1) * 8 <= 200 * 1024;
        if (!c->lines && !plane_fits)
            return fail3(c, SR_ERR_SHAPE, "3-D: this volume needs the lines solve (D >= 16, M >= 32, tau mu not extreme); "
                                          "the plane solve holds one D x M spectrum plane in shared memory (D (M + 1) <= 25600)");
    }
    if (c->lines) {
        const int L = 1 << kTriLogL, C = D / L;
        const int E_m = M < 16 ? M : 16, T_m = M / E_m;
        int cpc = 1;
        while (cpc * T_m < 64 && cpc * 2 <= H * D) cpc *= 2;
        int sc = M + (M >> 4);
        sc = ((sc + 15) & ~15) + 1;
        c->l_lg_cpc = lg2(cpc);
        c->l_threads = cpc * T_m;
        c->l_sc = sc;
        c->l_smem = cpc * sc * (int)sizeof(float2);
        c->l_grid = H * D / cpc;
        CK3(cudaFuncSetAttribute((const void*)c->lfwd, cudaFuncAttributeMaxDynamicSharedMemorySize, c->l_smem));
        CK3(cudaFuncSetAttribute((const void*)c->linv, cudaFuncAttributeMaxDynamicSharedMemorySize, c->l_smem));
        int W = 8;
        if (W > C) W = C;
        c->tri = pick_col_tri_rm();
        c->t_threads = 32 * W;
        c->t_smem = (W * L + 2 * (c->t_mmax + W)) * 32 * (int)sizeof(float2);
        c->t_grid = dim3(M / 32, C / W, H + 1);
        CK3(cudaFuncSetAttribute((const void*)c->tri, cudaFuncAttributeMaxDynamicSharedMemorySize, c->t_smem));
        const size_t nplane = (size_t)D * M;
        if (!c->spec2 && cudaMalloc((void**)&c->spec2, (size_t)(H + 1) * nplane * sizeof(float2)) != cudaSuccess)
            return fail3(c, SR_ERR_OOM, "spectrum allocation failed");
        if (!c->tri_tab && cudaMalloc((void**)&c->tri_tab, (size_t)(H + 1) * M * sizeof(TriCol)) != cudaSuccess)
            return fail3(c, SR_ERR_OOM, "tridiagonal table allocation failed");
        // constants of c x_z - a (x_{z-1} + x_{z+1}) = d_z per (plane k2, column k1), fp64 -> fp32:
        // c = 1 + tau mu (6 - 2 cos(2 pi k1 / M) - 2 cos(2 pi k2 / N)); plane H is k2 = N/2 (unpacked from slot 0)
        std::vector<TriCol> tab((size_t)(H + 1) * M);
        const double a = (double)p.tau * (double)p.mu, pi_ = 3.14159265358979323846;
        for (int k2 = 0; k2 <= H; k2++)
            for (int k1 = 0; k1 < M; k1++) {
                double sq = 1.0, clos = 1.0;
                const double cc = 1.0 + a * (6.0 - 2.0 * std::cos(2 * pi_ * k1 / M) - 2.0 * std::cos(2 * pi_ * k2 / N));
                const double r = tri_ratio(a, cc, &sq), rho = std::pow(r, L);
                const int mm = tri_carry_terms(rho, C, &clos);
                TriCol& t = tab[(size_t)k2 * M + k1];
                for (int q = 0; q < 2; q++) {
                    t.r[q] = (float)r;
                    t.ks[q] = (float)(1.0 / (sq * (double)H * (double)M));   // + the j and i FFT normalisations
                    t.rho[q] = (float)rho;
                    t.clos[q] = (float)clos;
                }
                t.mmax = mm;
                t.pad_[0] = t.pad_[1] = t.pad_[2] = 0;
            }
        CK3(cudaMemcpyAsync(c->tri_tab, tab.data(), tab.size() * sizeof(TriCol), cudaMemcpyHostToDevice, c->s));
        CK3(cudaStreamSynchronize(c->s));
    }
    // plane solve
    c->pa.D = D;
    c->pa.M = M;
    c->pa.H = H;
    c->pa.taumu = p.tau * p.mu;
    c->pa.scale = (float)(1.0 / ((double)D * (double)M * (double)H));
    c->psmem = (D * (M + 1) + M / 2 + D / 2 + 1) * (int)sizeof(float2);
    c->pthreads = 1024;
    if (!c->lines)
        CK3(cudaFuncSetAttribute((const void*)k3_planes_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, c->psmem));
    // stencils
    if (!pick_vol(p.window, p.window_shape, p.l == p.epsilon, c->rhs, c->wb, c->vsmem))
        return fail3(c, SR_ERR_ARG, "window radius not supported in 3-D");
    CK3(cudaFuncSetAttribute((const void*)c->rhs, cudaFuncAttributeMaxDynamicSharedMemorySize, c->vsmem));
    for (int m = 0; m < 2; m++)
        for (int u = 0; u < 2; u++)
            CK3(cudaFuncSetAttribute((const void*)c->wb[m][u], cudaFuncAttributeMaxDynamicSharedMemorySize, c->vsmem));
    c->vgrid = dim3((N + V_TX - 1) / V_TX, (M + V_TY - 1) / V_TY, (D + V_TZ - 1) / V_TZ);
    c->vblock = dim3(32, 8, 1);
    VolArgs& a = c->va;
    a.D = D;
    a.M = M;
    a.N = N;
    a.vol = c->vol;
    a.reg.eps = p.epsilon;
    a.reg.inv_eps = 1.f / p.epsilon;
    a.reg.l = p.l;
    a.reg.sl = (float)std::sin(3.14159265358979323846 * (double)p.l / (double)p.epsilon);
    a.reg.cl = (float)std::cos(3.14159265358979323846 * (double)p.l / (double)p.epsilon);
    a.reg.l_eq_eps = p.l == p.epsilon ? 1 : 0;
    for (int q = 0; q <= 8; q++) a.e[q] = (float)std::exp(-(double)(q * q) / ((double)p.d * p.d));
    a.tau = p.tau;
    a.gamma = p.gamma;
    a.alpha = p.alpha;
    a.beta = p.beta;
    a.mu = p.mu;
    a.beta2_mu = 2.f * p.beta / p.mu;
    a.gamma_mu = p.gamma / p.mu;
    a.w_proj = p.w_proj;
    a.b_max = p.b_max;
    a.aos = 0;
    {
        const char* e = getenv("SRSB_BAND_SKIP");
        a.band_skip = (e && e[0] == '0') ? 0 : 1;
    }
    // tables (fp64 -> fp32)
    const double pi = 3.14159265358979323846;
    std::vector<float2> twH(H), twR(H), twM(M), twD(D);
    std::vector<float> cM(M), cD(D), cN(H + 1);
    for (int m = 0; m < H; m++) twH[m] = make_float2((float)std::cos(-2 * pi * m / H), (float)std::sin(-2 * pi * m / H));
    for (int k = 0; k < H; k++) twR[k] = make_float2((float)std::cos(-2 * pi * k / N), (float)std::sin(-2 * pi * k / N));
    for (int m = 0; m < M; m++) twM[m] = make_float2((float)std::cos(-2 * pi * m / M), (float)std::sin(-2 * pi * m / M));
    for (int m = 0; m < D; m++) twD[m] = make_float2((float)std::cos(-2 * pi * m / D), (float)std::sin(-2 * pi * m / D));
    for (int k = 0; k < M; k++) cM[k] = (float)(2.0 - 2.0 * std::cos(2 * pi * k / M));
    for (int k = 0; k < D; k++) cD[k] = (float)(2.0 - 2.0 * std::cos(2 * pi * k / D));
    for (int k = 0; k <= H; k++) cN[k] = (float)(2.0 - 2.0 * std::cos(2 * pi * k / N));
    c->rblur = (int)std::ceil(3.0 * p.sigma);
    std::vector<float> kb(2 * c->rblur + 1);
    {
        double ks = 0.0;
        std::vector<double> kd(2 * c->rblur + 1);
        for (int t = -c->rblur; t <= c->rblur; t++) ks += kd[t + c->rblur] = std::exp(-(double)(t * t) / (2.0 * p.sigma * p.sigma));
        for (size_t t = 0; t < kd.size(); t++) kb[t] = (float)(kd[t] / ks);
    }
    CK3(cudaMemcpyAsync(c->twH, twH.data(), H * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->twR, twR.data(), H * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->twM, twM.data(), M * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->twD, twD.data(), D * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->cM, cM.data(), M * 4, cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->cD, cD.data(), D * 4, cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->cN, cN.data(), (H + 1) * 4, cudaMemcpyHostToDevice, c->s));
    CK3(cudaMemcpyAsync(c->blurk, kb.data(), kb.size() * 4, cudaMemcpyHostToDevice, c->s));
    CK3(cudaStreamSynchronize(c->s));
    return SR_OK;
}

void prof_b(sr_sb3_ctx* c) {
    if (!c->prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->s);
    c->ev_pool.push_back(e);
}
void prof_e(sr_sb3_ctx* c, int cls) {
    if (!c->prof) return;
    prof_b(c);
    c->ev_cls.push_back(cls);
}

void enq_rhs3(sr_sb3_ctx* c, float* out) {
    prof_b(c);
    c->rhs<<<c->vgrid, c->vblock, c->vsmem, c->s>>>(c->phi, c->w[c->wcur], c->b, c->g, out, c->va);
    prof_e(c, SR_K_RHS);
}
void enq_solve3(sr_sb3_ctx* c, const float* in, float* out, float clip, int accum) {
    prof_b(c);
    c->rfwd<<<c->rgrid, c->rblock, c->rsmem, c->s>>>(in, c->spec, c->twH, c->twR, c->ra);
    prof_e(c, SR_K_ROWS_R2C);
    prof_b(c);
    const float2* solved = c->spec;
    if (c->lines) {
        const int D = c->D, M = c->p.M, H = c->p.N / 2;
        const long long nplane = (long long)D * M;
        c->lfwd<<<c->l_grid, c->l_threads, c->l_smem, c->s>>>(c->spec, c->twM, c->l_lg_cpc, c->l_sc);
        // the packed plane 0 -> plane 0 (k2 = 0) and plane H (k2 = N/2); spec and spec2 hold H + 1 planes
        k3_unpack0<<<(int)((nplane / 2 + D + 255) / 256), 256, 0, c->s>>>(c->spec, c->spec + (size_t)H * nplane, D, M);
        c->tri<<<c->t_grid, c->t_threads, c->t_smem, c->s>>>(c->spec, c->spec2, c->tri_tab, lg2(D), lg2(M), M, c->t_mmax, M);
        k3_repack0<<<(int)((nplane + 255) / 256), 256, 0, c->s>>>(c->spec2, c->spec2 + (size_t)H * nplane, nplane);
        c->linv<<<c->l_grid, c->l_threads, c->l_smem, c->s>>>(c->spec2, c->twM, c->l_lg_cpc, c->l_sc);
        solved = c->spec2;
    } else {
        k3_planes_solve<<<c->p.N / 2, c->pthreads, c->psmem, c->s>>>(c->spec, c->twM, c->twD, c->cM, c->cD, c->cN, c->pa);
    }
    prof_e(c, SR_K_COLS_SOLVE);
    FftRowArgs ra = c->ra;
    ra.clip = clip;
    ra.accum = accum;
    prof_b(c);
    c->rinv<<<c->rgrid, c->rblock, c->rsmem, c->s>>>(solved, out, c->twH, c->twR, ra);
    prof_e(c, SR_K_ROWS_C2R);
}
void enq_wb3(sr_sb3_ctx* c, int last) {
    prof_b(c);
    c->wb[c->p.w_mode][last]<<<c->vgrid, c->vblock, c->vsmem, c->s>>>(c->phi, c->w[c->wcur], c->w[c->wcur ^ 1],
                                                                       c->b, c->g, c->flag, c->va);
    prof_e(c, SR_K_WB);
    c->wcur ^= 1;
}
void enq_iteration3(sr_sb3_ctx* c) {
    for (int s = 0; s < c->p.S; s++) {
        enq_rhs3(c, c->F);
        enq_solve3(c, c->F, c->phi, s == c->p.S - 1 ? c->p.phi_clip : 0.f, 1);
    }
    const int passes = c->p.w_mode == SR_W_FIXED_POINT ? c->p.w_iters : 1;
    for (int r = 0; r < passes; r++) enq_wb3(c, r == passes - 1);
}

sr_status begin3(sr_sb3_ctx* c) {
    CK3(cudaEventRecord(c->ev_in, c->user));
    CK3(cudaStreamWaitEvent(c->s, c->ev_in, 0));
    return SR_OK;
}
sr_status end3(sr_sb3_ctx* c) {
    CK3(cudaGetLastError());
    CK3(cudaEventRecord(c->ev_out, c->s));
    CK3(cudaStreamWaitEvent(c->user, c->ev_out, 0));
    return SR_OK;
}
sr_status copy3(sr_sb3_ctx* c, void* dst, const void* src, long long n) {
    CK3(cudaMemcpyAsync(dst, src, (size_t)n * 4, cudaMemcpyDefault, c->s));
    return SR_OK;
}

}  // namespace

extern "C" {

sr_status sr_sb3_create(const sr_sb_params* p, int D, int device, void* stream, sr_sb3_ctx** out) {
    if (!out) { g3_create_err = "out is NULL"; return SR_ERR_ARG; }
    *out = nullptr;
    std::string m;
    sr_status st = validate3(p, D, m);
    if (st != SR_OK) { g3_create_err = m; return st; }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        g3_create_err = "no such CUDA device";
        return SR_ERR_CUDA;
    }
    Dev3 dg(device);
    sr_sb3_ctx* c = new sr_sb3_ctx();
    c->p = *p;
    c->D = D;
    c->device = device;
    c->user = (cudaStream_t)stream;
    const long long V = (long long)D * p->M * p->N;
    const size_t nspec = (size_t)(p->N / 2 + 1) * D * p->M;   // + plane N/2 of the lines solve (unpacked from slot 0)
    bool ok = cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) == cudaSuccess;
    auto al = [&](void** ptr, size_t bytes) { return cudaMalloc(ptr, bytes) == cudaSuccess; };
    ok = ok && al((void**)&c->phi, V * 4) && al((void**)&c->F, V * 4) && al((void**)&c->w[0], 3 * V * 4) &&
         al((void**)&c->w[1], 3 * V * 4) && al((void**)&c->b, 3 * V * 4) && al((void**)&c->g, V * 4) &&
         al((void**)&c->tmp, V * 4) && al((void**)&c->spec, nspec * sizeof(float2)) &&
         al((void**)&c->twH, p->N / 2 * sizeof(float2)) && al((void**)&c->twR, p->N / 2 * sizeof(float2)) &&
         al((void**)&c->twM, p->M * sizeof(float2)) && al((void**)&c->twD, D * sizeof(float2)) &&
         al((void**)&c->cM, p->M * 4) && al((void**)&c->cD, D * 4) && al((void**)&c->cN, (p->N / 2 + 1) * 4) &&
         al((void**)&c->blurk, 17 * 4) && al((void**)&c->flag, sizeof(int));
    if (!ok) {
        cudaGetLastError();
        g3_create_err = "device allocation failed";
        sr_sb3_destroy(c);
        return SR_ERR_OOM;
    }
    cudaMemsetAsync(c->flag, 0, sizeof(int), c->s);
    st = configure3(c);
    if (st != SR_OK) {
        g3_create_err = c->err;
        sr_sb3_destroy(c);
        return st;
    }
    *out = c;
    return SR_OK;
}

sr_status sr_sb3_set_image(sr_sb3_ctx* c, const float* volume, const float* phi0) {
    if (!c) return SR_ERR_ARG;
    if (!volume || !phi0) return fail3(c, SR_ERR_ARG, "NULL pointer");
    Dev3 dg(c->device);
    RET3(begin3(c));
    const int D = c->D, M = c->p.M, N = c->p.N;
    RET3(copy3(c, c->F, volume, c->vol));
    RET3(copy3(c, c->phi, phi0, c->vol));
    const int thr = 256, blk = (int)std::min<long long>((c->vol + thr - 1) / thr, 148 * 16);
    // Eq. (1): G_sigma * f along j, i, z, then g
    k3_blur<<<blk, thr, 0, c->s>>>(c->F, c->tmp, D, M, N, 0, c->rblur, c->blurk);
    k3_blur<<<blk, thr, 0, c->s>>>(c->tmp, c->g, D, M, N, 1, c->rblur, c->blurk);
    k3_blur<<<blk, thr, 0, c->s>>>(c->g, c->tmp, D, M, N, 2, c->rblur, c->blurk);
    k3_edge_g<<<blk, thr, 0, c->s>>>(c->tmp, c->g, D, M, N, c->p.rho, c->p.s);
    k3_init_w<<<blk, thr, 0, c->s>>>(c->phi, c->w[0], c->b, D, M, N);
    c->wcur = 0;
    c->k = 0;
    c->have_state = true;
    RET3(end3(c));
    return SR_OK;
}

sr_status sr_sb3_iterate(sr_sb3_ctx* c, int K) {
    if (!c) return SR_ERR_ARG;
    if (K < 0) return fail3(c, SR_ERR_ARG, "K must be >= 0");
    if (!c->have_state) return fail3(c, SR_ERR_STATE, "iterate before set_image/set_state");
    Dev3 dg(c->device);
    RET3(begin3(c));
    int k = 0;
    if (K >= 2) {
        if (!c->graph || c->graph_wcur != c->wcur) {
            if (c->graph) cudaGraphExecDestroy(c->graph);
            c->graph = nullptr;
            const int w0 = c->wcur;
            cudaGraph_t gr;
            CK3(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
            enq_iteration3(c);
            enq_iteration3(c);
            CK3(cudaStreamEndCapture(c->s, &gr));
            cudaError_t e = cudaGraphInstantiate(&c->graph, gr, 0);
            cudaGraphDestroy(gr);
            if (e != cudaSuccess) return fail3(c, SR_ERR_CUDA, std::string("graph: ") + cudaGetErrorString(e));
            c->wcur = w0;
            c->graph_wcur = w0;
        }
        for (; k + 2 <= K; k += 2) CK3(cudaGraphLaunch(c->graph, c->s));   // 2 iterations: wcur unchanged
    }
    for (; k < K; k++) enq_iteration3(c);
    c->k += K;
    RET3(end3(c));
    return SR_OK;
}

sr_status sr_sb3_get_phi(sr_sb3_ctx* c, float* phi_out) {
    if (!c) return SR_ERR_ARG;
    if (!phi_out) return fail3(c, SR_ERR_ARG, "NULL pointer");
    Dev3 dg(c->device);
    RET3(begin3(c));
    RET3(copy3(c, phi_out, c->phi, c->vol));
    RET3(end3(c));
    return SR_OK;
}

sr_status sr_sb3_get_state(sr_sb3_ctx* c, float* phi, float* w, float* b, float* g) {
    if (!c) return SR_ERR_ARG;
    if (!c->have_state) return fail3(c, SR_ERR_STATE, "no state");
    Dev3 dg(c->device);
    RET3(begin3(c));
    if (phi) RET3(copy3(c, phi, c->phi, c->vol));
    if (w) RET3(copy3(c, w, c->w[c->wcur], 3 * c->vol));
    if (b) RET3(copy3(c, b, c->b, 3 * c->vol));
    if (g) RET3(copy3(c, g, c->g, c->vol));
    RET3(end3(c));
    CK3(cudaStreamSynchronize(c->user));
    return SR_OK;
}

sr_status sr_sb3_set_state(sr_sb3_ctx* c, const float* phi, const float* w, const float* b, const float* g) {
    if (!c) return SR_ERR_ARG;
    if (!phi || !w || !b || !g) return fail3(c, SR_ERR_ARG, "NULL pointer");
    Dev3 dg(c->device);
    RET3(begin3(c));
    c->wcur = 0;
    RET3(copy3(c, c->phi, phi, c->vol));
    RET3(copy3(c, c->w[0], w, 3 * c->vol));
    RET3(copy3(c, c->b, b, 3 * c->vol));
    RET3(copy3(c, c->g, g, c->vol));
    c->have_state = true;
    RET3(end3(c));
    return SR_OK;
}

sr_status sr_sb3_debug_solve(sr_sb3_ctx* c, const float* F, float* phi_out) {
    if (!c) return SR_ERR_ARG;
    if (!F || !phi_out) return fail3(c, SR_ERR_ARG, "NULL pointer");
    Dev3 dg(c->device);
    RET3(begin3(c));
    RET3(copy3(c, c->F, F, c->vol));
    enq_solve3(c, c->F, c->tmp, 0.f, 0);
    RET3(copy3(c, phi_out, c->tmp, c->vol));
    RET3(end3(c));
    return SR_OK;
}

sr_status sr_sb3_debug_rhs(sr_sb3_ctx* c, float* D_out) {
    if (!c) return SR_ERR_ARG;
    if (!D_out) return fail3(c, SR_ERR_ARG, "NULL pointer");
    if (!c->have_state) return fail3(c, SR_ERR_STATE, "no state");
    Dev3 dg(c->device);
    RET3(begin3(c));
    enq_rhs3(c, c->F);
    RET3(copy3(c, D_out, c->F, c->vol));
    RET3(end3(c));
    return SR_OK;
}

sr_status sr_sb3_profile(sr_sb3_ctx* c, int K, float* ms_out, int* launches_out) {
    if (!c) return SR_ERR_ARG;
    if (K < 1 || !ms_out || !launches_out) return fail3(c, SR_ERR_ARG, "K >= 1 and non-NULL outputs required");
    if (!c->have_state) return fail3(c, SR_ERR_STATE, "no state");
    Dev3 dg(c->device);
    RET3(begin3(c));
    c->prof = true;
    for (int i = 0; i < K; i++) enq_iteration3(c);
    c->prof = false;
    RET3(end3(c));
    CK3(cudaStreamSynchronize(c->s));
    for (int k = 0; k < SR_K_NCLASSES; k++) { ms_out[k] = 0.f; launches_out[k] = 0; }
    for (size_t i = 0; i < c->ev_cls.size(); i++) {
        float ms = 0.f;
        CK3(cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
        ms_out[c->ev_cls[i]] += ms;
        launches_out[c->ev_cls[i]] += 1;
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    c->ev_pool.clear();
    c->ev_cls.clear();
    c->k += K;
    return SR_OK;
}

sr_status sr_sb3_sync(sr_sb3_ctx* c) {
    if (!c) return SR_ERR_ARG;
    Dev3 dg(c->device);
    CK3(cudaStreamSynchronize(c->s));
    int flag = 0;
    CK3(cudaMemcpy(&flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) return fail3(c, SR_ERR_NONFINITE, "non-finite or |b| > b_max in the w/b update");
    return SR_OK;
}

void sr_sb3_destroy(sr_sb3_ctx* c) {
    if (!c) return;
    Dev3 dg(c->device);
    if (c->s) cudaStreamSynchronize(c->s);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    void* ptrs[] = {c->phi, c->F, c->w[0], c->w[1], c->b, c->g, c->tmp, c->spec, c->spec2, c->tri_tab, c->twH, c->twR,
                    c->twM, c->twD, c->cM, c->cD, c->cN, c->blurk, c->flag};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_out) cudaEventDestroy(c->ev_out);
    if (c->s) cudaStreamDestroy(c->s);
    delete c;
}

const char* sr_sb3_last_error(const sr_sb3_ctx* c) { return c ? c->err.c_str() : g3_create_err.c_str(); }

}  // extern "C"
