// srsb.cu -- context, launch configuration, CUDA graph and C ABI of libsrsb.so.
// See include/srsb.h for the contract and DESIGN.md for the design.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/srsb.h"
#include "sr_kernels.h"
#include "sr_setup.cuh"

using namespace srsb;

namespace {

constexpr int kMaxWindow = 8;
constexpr int kGraphIters = 2;   // iterations per captured graph (even: restores the w ping-pong parity)

int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) r++;
    return r;
}
bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

}  // namespace

struct sr_sb_ctx {
    sr_sb_params p;
    int device = 0;
    cudaStream_t user = nullptr;   // caller's stream
    cudaStream_t s = nullptr;      // private work stream (capturable)
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    size_t plane = 0;              // M * N
    float *phi = nullptr, *F = nullptr, *w[2] = {nullptr, nullptr}, *b = nullptr, *g = nullptr;
    float2* spec = nullptr;
    float2 *twH = nullptr, *twM = nullptr, *twR = nullptr;
    float *cM = nullptr, *cN = nullptr;
    int* flag = nullptr;
    int wcur = 0;
    long long k = 0;
    bool have_state = false;
    cudaGraphExec_t graph = nullptr;
    int graph_wcur = -1;
    std::string err;
    // launch configuration
    RowKernel rfwd = nullptr;
    RowInvKernel rinv = nullptr;
    ColKernel cols = nullptr;
    RhsKernel rhs = nullptr;
    WbKernel wb[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    FftRowArgs ra{};
    FftColArgs ca{};
    StencilArgs sa{};
    dim3 rgrid, rblock, cgrid, cblock, sgrid, sblock;
    int rsmem = 0, csmem = 0, ssmem = 0;
    // sr_sb_profile
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_cls;
    size_t ev_used = 0;
};

namespace {

sr_status fail(sr_sb_ctx* c, sr_status st, const std::string& msg) {
    if (c) c->err = msg;
    return st;
}

thread_local std::string g_create_err;

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(c, SR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

sr_status validate(const sr_sb_params* p, std::string& msg) {
    if (!p) { msg = "params is NULL"; return SR_ERR_ARG; }
    if (!is_pow2(p->M) || !is_pow2(p->N) || p->M < 8 || p->N < 8 || p->M > 8192 || p->N > 8192) {
        msg = "M and N must be powers of two in [8, 8192]";
        return SR_ERR_SHAPE;
    }
    if (p->batch < 1) { msg = "batch must be >= 1"; return SR_ERR_SHAPE; }
    if (!(p->tau >= 0.f) || !(p->mu > 0.f) || !(p->epsilon > 0.f) || !(p->d > 0.f) || !(p->sigma > 0.f) ||
        !(p->l >= 0.f) || !(p->rho >= 0.f)) {
        msg = "need tau >= 0, mu > 0, epsilon > 0, d > 0, sigma > 0, l >= 0, rho >= 0";
        return SR_ERR_ARG;
    }
    if ((int)std::ceil(3.0 * p->sigma) > 8) { msg = "sigma too large (radius ceil(3 sigma) must be <= 8)"; return SR_ERR_ARG; }
    if (p->window < 0 || p->window > kMaxWindow) { msg = "window radius must be in [0, 8]"; return SR_ERR_ARG; }
    if (p->window_shape != SR_WIN_DISC && p->window_shape != SR_WIN_SQUARE) { msg = "bad window_shape"; return SR_ERR_ARG; }
    if (p->S < 1) { msg = "S must be >= 1"; return SR_ERR_ARG; }
    if (p->s != 1 && p->s != 2) { msg = "s must be 1 or 2"; return SR_ERR_ARG; }
    if (p->w_proj < 0 || p->w_proj > 2) { msg = "bad w_proj"; return SR_ERR_ARG; }
    if (p->w_mode != SR_W_THRESHOLD && p->w_mode != SR_W_FIXED_POINT) { msg = "bad w_mode"; return SR_ERR_ARG; }
    if (p->w_mode == SR_W_FIXED_POINT && p->w_iters < 1) { msg = "w_iters must be >= 1"; return SR_ERR_ARG; }
    if (p->phi_clip < 0.f) { msg = "phi_clip must be >= 0"; return SR_ERR_ARG; }
    return SR_OK;
}

sr_status configure(sr_sb_ctx* c) {
    const sr_sb_params& p = c->p;
    const int M = p.M, N = p.N, H = N / 2, B = p.batch;
    const int lgH = ilog2(H), lgM = ilog2(M);
    c->rfwd = pick_row_fwd(lgH);
    c->rinv = pick_row_inv(lgH);
    c->cols = pick_col(lgM);
    if (!c->rfwd || !c->rinv || !c->cols) return fail(c, SR_ERR_SHAPE, "no FFT kernel for this size");
    // Launch shapes (measured on B200, C3: smaller CTAs overlap load and FFT phases better):
    //  rows: rpc rows per CTA, 64..512 threads, <= ~72 KB shared;  E = min(16, H) values per thread
    const int E_h = H < 16 ? H : 16, T_h = H / E_h;
    int rpc = 8;
    while (rpc * T_h < 64 && rpc < 32) rpc <<= 1;
    while ((rpc * T_h > 512 || rpc * (H + H / 16 + 32) * 8 > 72 * 1024) && rpc > 1) rpc >>= 1;
    if (rpc > M) rpc = M;
    if (const char* ev = std::getenv("SRSB_RPC")) {   // tuning knob (power of two)
        const int v = std::atoi(ev);
        if (v >= 1 && v <= M && v * T_h <= 512 && (v & (v - 1)) == 0) rpc = v;
    }
    //  column-group interleave of the transposed spectrum: rpc * G >= 8 complex = 64 B contiguous
    int G = 8 / rpc;
    if (G < 1) G = 1;
    if (G > H) G = H;
    if (const char* ev = std::getenv("SRSB_G")) {     // tuning knob (power of two)
        const int v = std::atoi(ev);
        if (v >= 1 && v <= H && (v & (v - 1)) == 0) G = v;
    }
    //  columns per CTA: a multiple of G, >= 64 threads, <= 512
    const int E_m = M < 16 ? M : 16, T_m = M / E_m;
    int cpc = G;
    while (cpc * T_m < 64 && cpc * 2 <= H) cpc *= 2;
    while (cpc * T_m > 512 && cpc > G) cpc >>= 1;
    if (const char* ev = std::getenv("SRSB_CPC")) {   // tuning knob (power of two, multiple of G)
        const int v = std::atoi(ev);
        if (v >= G && v <= H && v * T_m <= 512 && (v & (v - 1)) == 0) cpc = v;
    }
    if (cpc * T_m > 512) return fail(c, SR_ERR_SHAPE, "column FFT too large for one CTA");
    auto padded = [](int n, int extra) {   // float2 slots: one pad per 16, rounded to 16, + extra
        int sz = n + (n >> 4);
        sz = (sz + 15) & ~15;
        return sz + extra;
    };
    c->ra.M = M;
    c->ra.lg_rpc = ilog2(rpc);
    c->ra.lg_G = ilog2(G);
    c->ra.SR = padded(H, G < 16 ? G : 1);
    c->ra.clip = 0.f;
    c->ra.accum = 0;
    c->rgrid = dim3(M / rpc, B, 1);
    c->rblock = dim3(rpc * T_h, 1, 1);
    c->rsmem = rpc * c->ra.SR * (int)sizeof(float2);
    c->ca.H = H;
    c->ca.lg_G = ilog2(G);
    c->ca.lg_cpc = ilog2(cpc);
    c->ca.SC = padded(M, 1);
    c->ca.taumu = p.tau * p.mu;
    c->ca.scale = (float)(1.0 / ((double)M * (double)H));
    c->cgrid = dim3(H / cpc, B, 1);
    c->cblock = dim3(cpc * T_m, 1, 1);
    c->csmem = cpc * c->ca.SC * (int)sizeof(float2);
    // stencils
    int smem = 0;
    bool ok = pick_stencil(p.window, p.window_shape, p.l == p.epsilon, c->rhs, c->wb, smem);
    if (!ok) return fail(c, SR_ERR_ARG, "window radius not supported");
    c->ssmem = smem;
    c->sblock = dim3(32, ST_BY, 1);
    c->sa.tiles_x = (N + ST_TW - 1) / ST_TW;
    c->sa.tiles_y = (M + ST_TH - 1) / ST_TH;
    c->sa.ntiles = c->sa.tiles_x * c->sa.tiles_y * B;
    StencilArgs& a = c->sa;
    a.M = M;
    a.N = N;
    a.reg.eps = p.epsilon;
    a.reg.inv_eps = 1.f / p.epsilon;
    a.reg.l = p.l;
    a.reg.sl = (float)std::sin(3.14159265358979323846 * (double)p.l / (double)p.epsilon);
    a.reg.cl = (float)std::cos(3.14159265358979323846 * (double)p.l / (double)p.epsilon);
    a.reg.l_eq_eps = (p.l == p.epsilon) ? 1 : 0;
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
    // opt-in shared memory above 48 KB
    CK(cudaFuncSetAttribute((const void*)c->rfwd, cudaFuncAttributeMaxDynamicSharedMemorySize, c->rsmem));
    CK(cudaFuncSetAttribute((const void*)c->rinv, cudaFuncAttributeMaxDynamicSharedMemorySize, c->rsmem));
    CK(cudaFuncSetAttribute((const void*)c->cols, cudaFuncAttributeMaxDynamicSharedMemorySize, c->csmem));
    CK(cudaFuncSetAttribute((const void*)c->rhs, cudaFuncAttributeMaxDynamicSharedMemorySize, c->ssmem));
    for (int m = 0; m < 2; m++)
        for (int u = 0; u < 2; u++)
            CK(cudaFuncSetAttribute((const void*)c->wb[m][u], cudaFuncAttributeMaxDynamicSharedMemorySize, c->ssmem));
    c->sgrid = dim3(c->sa.tiles_x, c->sa.tiles_y, B);
    return SR_OK;
}

sr_status make_tables(sr_sb_ctx* c) {
    const int M = c->p.M, N = c->p.N, H = N / 2;
    const double pi = 3.14159265358979323846;
    std::vector<float2> twH(H), twM(M), twR(H);
    std::vector<float> cM(M), cN(H + 1);
    for (int m = 0; m < H; m++) twH[m] = make_float2((float)std::cos(-2 * pi * m / H), (float)std::sin(-2 * pi * m / H));
    for (int m = 0; m < M; m++) twM[m] = make_float2((float)std::cos(-2 * pi * m / M), (float)std::sin(-2 * pi * m / M));
    for (int k = 0; k < H; k++) twR[k] = make_float2((float)std::cos(-2 * pi * k / N), (float)std::sin(-2 * pi * k / N));
    for (int k = 0; k < M; k++) cM[k] = (float)(2.0 - 2.0 * std::cos(2 * pi * k / M));
    for (int k = 0; k <= H; k++) cN[k] = (float)(2.0 - 2.0 * std::cos(2 * pi * k / N));
    CK(cudaMemcpyAsync(c->twH, twH.data(), H * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK(cudaMemcpyAsync(c->twM, twM.data(), M * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK(cudaMemcpyAsync(c->twR, twR.data(), H * sizeof(float2), cudaMemcpyHostToDevice, c->s));
    CK(cudaMemcpyAsync(c->cM, cM.data(), M * sizeof(float), cudaMemcpyHostToDevice, c->s));
    CK(cudaMemcpyAsync(c->cN, cN.data(), (H + 1) * sizeof(float), cudaMemcpyHostToDevice, c->s));
    CK(cudaStreamSynchronize(c->s));
    return SR_OK;
}

// ------------------------------------------------------------------ enqueue helpers
// profiling hooks (sr_sb_profile): no-ops unless c->prof is set
void prof_begin(sr_sb_ctx* c) {
    if (!c->prof) return;
    if (c->ev_pool.size() < c->ev_used + 2) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        c->ev_pool.push_back(a);
        c->ev_pool.push_back(b);
    }
    cudaEventRecord(c->ev_pool[c->ev_used], c->s);
}
void prof_end(sr_sb_ctx* c, int cls) {
    if (!c->prof) return;
    cudaEventRecord(c->ev_pool[c->ev_used + 1], c->s);
    c->ev_cls.push_back(cls);
    c->ev_used += 2;
}

// phi_out = A^{-1} F (accum = 0) or phi_out += A^{-1} F (accum = 1, increment form), then clamp
sr_status enq_solve(sr_sb_ctx* c, const float* F, float* out, float clip, int accum) {
    FftRowArgs ra = c->ra;
    ra.accum = accum;
    prof_begin(c);
    c->rfwd<<<c->rgrid, c->rblock, c->rsmem, c->s>>>(F, c->spec, c->twH, c->twR, ra);
    prof_end(c, SR_K_ROWS_R2C);
    prof_begin(c);
    c->cols<<<c->cgrid, c->cblock, c->csmem, c->s>>>(c->spec, c->twM, c->cM, c->cN, c->ca);
    prof_end(c, SR_K_COLS_SOLVE);
    ra.clip = clip;
    prof_begin(c);
    c->rinv<<<c->rgrid, c->rblock, c->rsmem, c->s>>>(c->spec, out, c->twH, c->twR, ra);
    prof_end(c, SR_K_ROWS_C2R);
    return SR_OK;
}

sr_status enq_rhs(sr_sb_ctx* c, float* F) {
    prof_begin(c);
    c->rhs<<<c->sgrid, c->sblock, c->ssmem, c->s>>>(c->phi, c->w[c->wcur], c->b, c->g, F, c->sa);
    prof_end(c, SR_K_RHS);
    return SR_OK;
}

sr_status enq_wb(sr_sb_ctx* c) {
    const int mode = c->p.w_mode;
    const int passes = mode == SR_W_FIXED_POINT ? c->p.w_iters : 1;
    for (int r = 0; r < passes; r++) {
        const int last = (r == passes - 1) ? 1 : 0;
        prof_begin(c);
        c->wb[mode][last]<<<c->sgrid, c->sblock, c->ssmem, c->s>>>(c->phi, c->w[c->wcur], c->w[c->wcur ^ 1], c->b,
                                                                   c->g, c->flag, c->sa);
        prof_end(c, SR_K_WB);
        c->wcur ^= 1;
    }
    return SR_OK;
}

sr_status enq_iteration(sr_sb_ctx* c) {
    for (int s = 0; s < c->p.S; s++) {
        enq_rhs(c, c->F);
        enq_solve(c, c->F, c->phi, (s == c->p.S - 1) ? c->p.phi_clip : 0.f, 1);
    }
    enq_wb(c);
    return SR_OK;
}

sr_status check_launch(sr_sb_ctx* c) {
    CK(cudaGetLastError());
    return SR_OK;
}

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DevGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// order the private stream after the caller's stream, and back
sr_status begin(sr_sb_ctx* c) {
    CK(cudaEventRecord(c->ev_in, c->user));
    CK(cudaStreamWaitEvent(c->s, c->ev_in, 0));
    return SR_OK;
}
sr_status end(sr_sb_ctx* c) {
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_out, c->s));
    CK(cudaStreamWaitEvent(c->user, c->ev_out, 0));
    return SR_OK;
}

sr_status copy_in(sr_sb_ctx* c, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->s));
    return SR_OK;
}

}  // namespace

#define RET(x)                          \
    do {                                \
        sr_status r_ = (x);             \
        if (r_ != SR_OK) return r_;     \
    } while (0)

extern "C" {

int sr_sb_abi_version(void) { return SRSB_ABI_VERSION; }

void sr_sb_default_params(sr_sb_params* p, int M, int N, int batch, int window) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->M = M;
    p->N = N;
    p->batch = batch;
    p->gamma = 1.f;
    p->alpha = 4.f;
    // reading Q24: beta * sum_W G = 0.2 * (the same sum for the caption's 5x5 window, d = 5)
    {
        auto wsum = [](int R, double d, int shape) {
            double s = 0.0;
            for (int q1 = -R; q1 <= R; q1++)
                for (int q2 = -R; q2 <= R; q2++)
                    if (shape == 1 || q1 * q1 + q2 * q2 <= R * R) s += std::exp(-(double)(q1 * q1 + q2 * q2) / (d * d));
            return s;
        };
        const double d = window > 0 ? (double)window : 1.0;
        p->beta = (float)(0.2 * wsum(2, 5.0, 1) / wsum(window < 0 ? 0 : window, d, 0));
    }
    p->mu = 8.f;
    p->epsilon = 0.5f;
    p->l = 0.5f;
    p->window = window;
    p->d = (float)window > 0 ? (float)window : 1.f;
    p->window_shape = SR_WIN_DISC;
    p->tau = 0.05f;
    p->S = 3;
    p->rho = 30.f;
    p->sigma = 1.f;
    p->s = 2;
    p->phi_clip = 1.f;
    p->w_proj = SR_WPROJ_BALL;
    p->w_mode = SR_W_THRESHOLD;
    p->w_iters = 1;
    p->b_max = 50.f;
}

sr_status sr_sb_create(const sr_sb_params* p, int device, void* stream, sr_sb_ctx** out) {
    if (!out) { g_create_err = "out is NULL"; return SR_ERR_ARG; }
    *out = nullptr;
    std::string msg;
    sr_status st = validate(p, msg);
    if (st != SR_OK) { g_create_err = msg; return st; }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        g_create_err = "no CUDA device " + std::to_string(device);
        return SR_ERR_CUDA;
    }
    DevGuard dg(device);
    sr_sb_ctx* c = new sr_sb_ctx();
    c->p = *p;
    c->device = device;
    c->user = (cudaStream_t)stream;
    c->plane = (size_t)p->M * p->N;
    const size_t n = c->plane * p->batch;
    auto alloc = [&](void** ptr, size_t bytes) -> bool {
        if (cudaMalloc(ptr, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
        return true;
    };
    bool ok = cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) { g_create_err = "stream/event creation failed"; sr_sb_destroy(c); return SR_ERR_CUDA; }
    ok = alloc((void**)&c->phi, n * 4) && alloc((void**)&c->F, n * 4) && alloc((void**)&c->w[0], 2 * n * 4) &&
         alloc((void**)&c->w[1], 2 * n * 4) && alloc((void**)&c->b, 2 * n * 4) && alloc((void**)&c->g, n * 4) &&
         alloc((void**)&c->spec, n / 2 * sizeof(float2)) && alloc((void**)&c->twH, p->N / 2 * sizeof(float2)) &&
         alloc((void**)&c->twM, p->M * sizeof(float2)) && alloc((void**)&c->twR, p->N / 2 * sizeof(float2)) &&
         alloc((void**)&c->cM, p->M * sizeof(float)) && alloc((void**)&c->cN, (p->N / 2 + 1) * sizeof(float)) &&
         alloc((void**)&c->flag, sizeof(int));
    if (!ok) { g_create_err = "device allocation failed"; sr_sb_destroy(c); return SR_ERR_OOM; }
    if (cudaMemsetAsync(c->flag, 0, sizeof(int), c->s) != cudaSuccess) {
        g_create_err = "memset failed"; sr_sb_destroy(c); return SR_ERR_CUDA;
    }
    st = configure(c);
    if (st == SR_OK) st = make_tables(c);
    if (st != SR_OK) { g_create_err = c->err; sr_sb_destroy(c); return st; }
    *out = c;
    return SR_OK;
}

sr_status sr_sb_set_image(sr_sb_ctx* c, const float* image, const float* phi0) {
    if (!c) return SR_ERR_ARG;
    if (!image || !phi0) return fail(c, SR_ERR_ARG, "image and phi0 must be non-NULL");
    DevGuard dg(c->device);
    const size_t n = c->plane * c->p.batch;
    RET(begin(c));
    // F and spec serve as scratch for the one-time edge indicator
    RET(copy_in(c, c->F, image, n * 4));
    RET(copy_in(c, c->phi, phi0, n * 4));
    EdgeArgs ea{};
    ea.M = c->p.M;
    ea.N = c->p.N;
    ea.r = (int)std::ceil(3.0 * c->p.sigma);
    double ks = 0.0, kk[17];
    for (int t = -ea.r; t <= ea.r; t++) { kk[t + ea.r] = std::exp(-(double)t * t / (2.0 * c->p.sigma * c->p.sigma)); ks += kk[t + ea.r]; }
    for (int t = 0; t <= 2 * ea.r; t++) ea.k[t] = (float)(kk[t] / ks);
    ea.rho = c->p.rho;
    ea.s = c->p.s;
    const dim3 blk(128), grd((c->p.N + 127) / 128, c->p.M, c->p.batch);
    float* tmp = reinterpret_cast<float*>(c->spec);   // n/2 complex = n floats
    k_blur_rows<<<grd, blk, 0, c->s>>>(c->F, tmp, ea);
    k_blur_cols<<<grd, blk, 0, c->s>>>(tmp, c->F, ea);
    k_edge_g<<<grd, blk, 0, c->s>>>(c->F, c->g, ea);
    c->wcur = 0;
    k_init_w<<<grd, blk, 0, c->s>>>(c->phi, c->w[0], c->b, c->p.M, c->p.N);
    CK(cudaMemsetAsync(c->flag, 0, sizeof(int), c->s));
    RET(end(c));
    c->k = 0;
    c->have_state = true;
    return SR_OK;
}

static sr_status build_graph(sr_sb_ctx* c) {
    if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }
    cudaGraph_t gr;
    const int w0 = c->wcur;
    CK(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kGraphIters; i++) enq_iteration(c);
    cudaError_t e = cudaStreamEndCapture(c->s, &gr);
    c->wcur = w0;   // capture did not execute anything
    if (e != cudaSuccess) return fail(c, SR_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->graph, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) { c->graph = nullptr; return fail(c, SR_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e)); }
    c->graph_wcur = w0;
    return SR_OK;
}

sr_status sr_sb_iterate(sr_sb_ctx* c, int K) {
    if (!c) return SR_ERR_ARG;
    if (K < 0) return fail(c, SR_ERR_ARG, "K must be >= 0");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "iterate before set_image/set_state");
    if (K == 0) return SR_OK;
    DevGuard dg(c->device);
    RET(begin(c));
    int done = 0;
    if (K >= kGraphIters) {
        if (!c->graph || c->graph_wcur != c->wcur) RET(build_graph(c));
        for (; done + kGraphIters <= K; done += kGraphIters) CK(cudaGraphLaunch(c->graph, c->s));
        // the graph's w ping-pong flips are even, so wcur is unchanged
    }
    for (; done < K; done++) enq_iteration(c);
    RET(end(c));
    c->k += K;
    return SR_OK;
}

sr_status sr_sb_sync(sr_sb_ctx* c) {
    if (!c) return SR_ERR_ARG;
    DevGuard dg(c->device);
    CK(cudaStreamSynchronize(c->s));
    CK(cudaStreamSynchronize(c->user));
    int flag = 0;
    CK(cudaMemcpy(&flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) return fail(c, SR_ERR_NONFINITE, "non-finite value or |b| > b_max detected in the w/b update");
    return SR_OK;
}

sr_status sr_sb_get_phi(sr_sb_ctx* c, float* phi_out) {
    if (!c) return SR_ERR_ARG;
    if (!phi_out) return fail(c, SR_ERR_ARG, "phi_out is NULL");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    DevGuard dg(c->device);
    RET(begin(c));
    CK(cudaMemcpyAsync(phi_out, c->phi, c->plane * c->p.batch * 4, cudaMemcpyDefault, c->s));
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_get_state(sr_sb_ctx* c, float* phi, float* w, float* b, float* g) {
    if (!c) return SR_ERR_ARG;
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    DevGuard dg(c->device);
    const size_t n = c->plane * c->p.batch;
    RET(begin(c));
    if (phi) CK(cudaMemcpyAsync(phi, c->phi, n * 4, cudaMemcpyDefault, c->s));
    if (w) CK(cudaMemcpyAsync(w, c->w[c->wcur], 2 * n * 4, cudaMemcpyDefault, c->s));
    if (b) CK(cudaMemcpyAsync(b, c->b, 2 * n * 4, cudaMemcpyDefault, c->s));
    if (g) CK(cudaMemcpyAsync(g, c->g, n * 4, cudaMemcpyDefault, c->s));
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_set_state(sr_sb_ctx* c, const float* phi, const float* w, const float* b, const float* g) {
    if (!c) return SR_ERR_ARG;
    if (!phi || !w || !b) return fail(c, SR_ERR_ARG, "phi, w and b must be non-NULL");
    if (!g && !c->have_state) return fail(c, SR_ERR_STATE, "g is required before set_image");
    DevGuard dg(c->device);
    const size_t n = c->plane * c->p.batch;
    RET(begin(c));
    RET(copy_in(c, c->phi, phi, n * 4));
    RET(copy_in(c, c->w[c->wcur], w, 2 * n * 4));
    RET(copy_in(c, c->b, b, 2 * n * 4));
    if (g) RET(copy_in(c, c->g, g, n * 4));
    CK(cudaMemsetAsync(c->flag, 0, sizeof(int), c->s));
    RET(end(c));
    c->k = 0;
    c->have_state = true;
    return SR_OK;
}

long long sr_sb_iteration(const sr_sb_ctx* c) { return c ? c->k : -1; }

sr_status sr_sb_debug_solve(sr_sb_ctx* c, const float* F, float* phi_out) {
    if (!c) return SR_ERR_ARG;
    if (!F || !phi_out) return fail(c, SR_ERR_ARG, "NULL pointer");
    DevGuard dg(c->device);
    const size_t n = c->plane * c->p.batch;
    RET(begin(c));
    RET(copy_in(c, c->F, F, n * 4));
    // solve into F's own buffer is not allowed (rows read F while c2r writes); use a temporary
    float* tmp = nullptr;
    CK(cudaMallocAsync((void**)&tmp, n * 4, c->s));
    enq_solve(c, c->F, tmp, 0.f, 0);
    CK(cudaMemcpyAsync(phi_out, tmp, n * 4, cudaMemcpyDefault, c->s));
    CK(cudaFreeAsync(tmp, c->s));
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_debug_rhs(sr_sb_ctx* c, float* F_out) {
    if (!c) return SR_ERR_ARG;
    if (!F_out) return fail(c, SR_ERR_ARG, "NULL pointer");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    DevGuard dg(c->device);
    RET(begin(c));
    enq_rhs(c, c->F);
    CK(cudaMemcpyAsync(F_out, c->F, c->plane * c->p.batch * 4, cudaMemcpyDefault, c->s));
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_debug_wb(sr_sb_ctx* c) {
    if (!c) return SR_ERR_ARG;
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    DevGuard dg(c->device);
    RET(begin(c));
    enq_wb(c);
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_profile(sr_sb_ctx* c, int K, float* ms_out, int* launches_out) {
    if (!c) return SR_ERR_ARG;
    if (K < 1 || !ms_out || !launches_out) return fail(c, SR_ERR_ARG, "K >= 1 and non-NULL outputs required");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "profile before set_image/set_state");
    DevGuard dg(c->device);
    RET(begin(c));
    c->prof = true;
    c->ev_used = 0;
    c->ev_cls.clear();
    for (int i = 0; i < K; i++) enq_iteration(c);
    c->prof = false;
    RET(end(c));
    CK(cudaStreamSynchronize(c->s));
    for (int k = 0; k < SR_K_NCLASSES; k++) { ms_out[k] = 0.f; launches_out[k] = 0; }
    for (size_t i = 0; i < c->ev_cls.size(); i++) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
        ms_out[c->ev_cls[i]] += ms;
        launches_out[c->ev_cls[i]] += 1;
    }
    c->k += K;
    return SR_OK;
}

int sr_sb_launches_per_iteration(const sr_sb_ctx* c) {
    if (!c) return -1;
    return 4 * c->p.S + (c->p.w_mode == SR_W_FIXED_POINT ? c->p.w_iters : 1);
}

void sr_sb_destroy(sr_sb_ctx* c) {
    if (!c) return;
    DevGuard dg(c->device);
    if (c->s) cudaStreamSynchronize(c->s);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    void* ptrs[] = {c->phi, c->F, c->w[0], c->w[1], c->b, c->g, c->spec, c->twH, c->twM, c->twR, c->cM, c->cN, c->flag};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_out) cudaEventDestroy(c->ev_out);
    if (c->s) cudaStreamDestroy(c->s);
    delete c;
}

const char* sr_sb_last_error(const sr_sb_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

}  // extern "C"
