// srsb.cu -- contexts, launch configuration, slab exchanges, CUDA graph and C ABI of libsrsb.so.
// See include/srsb.h for the contract and DESIGN.md for the design.
//
// A context holds B images of M_local x N pixels.  Every field is stored with gh ghost rows above
// and below each image plane; kernels address local row 0 and may read rows -gh .. M_local+gh-1.
// A whole-image context never reads its ghost rows (periodic neighbours wrap in-kernel).  In slab
// mode (one image split into P row slabs) the ghost rows are filled by halo
// exchanges and the FFT's column pass runs on the all-to-all-transposed spectrum; the exchanges
// are device copies between the slab contexts of one process (LOCAL backend: the single-GPU
// emulation used by the tests) or NCCL send/recv + all-to-all between processes (one per GPU).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/srsb.h"
#include "sr_kernels.h"
#include "sr_tri.cuh"
#include "sr_solve_cl.cuh"
#include <cudaTypedefs.h>
#include "sr_setup.cuh"
#include "sr_aos.cuh"

using namespace srsb;

namespace {

constexpr int kMaxWindow = 8;
constexpr int kGraphIters = 2;   // iterations per captured graph (even: restores the w ping-pong parity)
enum Backend { BK_NONE = 0, BK_LOCAL = 1, BK_NCCL = 2 };

int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) r++;
    return r;
}
bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

}  // namespace

struct sr_sb_ctx {
    sr_sb_params p;                // p.M = GLOBAL rows
    int device = 0;
    cudaStream_t user = nullptr;   // caller's stream
    cudaStream_t s = nullptr;      // work stream (private; shared by the members of a LOCAL group)
    bool own_stream = true;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    // slab geometry
    int nranks = 1, rank = 0;      // row slabs of the image, this context's slab
    int Ml = 0, row_off = 0;       // local rows, global index of local row 0
    int gh = 1;                    // ghost rows above / below each image plane
    bool slab = false;             // neighbours of rows 0 / Ml-1 come from ghost rows
    int backend = BK_NONE;
    long long pitch = 0;           // floats per image plane (Ml + 2 gh) * N
    std::vector<sr_sb_ctx*> members;   // LOCAL group leader: the slab contexts (leader has no fields)
    ncclComm_t comm = nullptr;
    // slab exchanges: a comm stream and fork/join events so the all-to-all of column chunk k + 1
    // overlaps the column solve of chunk k; a2a_chunks = 1: no pipelining
    cudaStream_t sc = nullptr;
    static constexpr int kMaxChunks = 8;
    cudaEvent_t xev[2 * kMaxChunks + 2] = {};
    int a2a_chunks = 1;
    // fields: *_base = allocation, field = base + gh * N (local row 0 of image 0)
    float *phi_base = nullptr, *F_base = nullptr, *w_base[2] = {nullptr, nullptr}, *b_base = nullptr,
          *g_base = nullptr;
    float *phi = nullptr, *F = nullptr, *w[2] = {nullptr, nullptr}, *b = nullptr, *g = nullptr;
    float2* spec = nullptr;        // [B][H/G][Ml][G]
    float2* spec_cols = nullptr;   // slab: [P][H/(P G)][Ml][G] (all-to-all receive buffer)
    float2 *twH = nullptr, *twM = nullptr, *twR = nullptr;
    float *cM = nullptr, *cN = nullptr;
    float* sym = nullptr;          // [H + 1][M] scale / symbol table (FftColArgs::sym), when small enough
    bool use_sym = false;          // configure(): the column solve reads the table (SRSB_SYMTAB)
    int* flag = nullptr;
    int wcur = 0;
    long long k = 0;
    bool have_state = false;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};   // captured kGraphIters iterations, per w ping-pong parity
    std::string err;
    // launch configuration
    RowKernel rfwd = nullptr;
    RowInvKernel rinv = nullptr;
    ColKernel cols = nullptr;
    ColPKernel cols_p = nullptr;   // persistent prefetching column solve for long contiguous columns
    int cp_grid = 0, cp_smem = 0, cp_threads = 0;
    ColTriKernel cols_tri = nullptr;   // cyclic tridiagonal column solve (sr_tri.cuh): whole image, G = 1, M >= 16
    TriCol* tri_tab = nullptr;         // [H] per-column constants
    SolveClKernel solve_cl = nullptr;  // small images: the whole solve in one cluster kernel (sr_solve_cl.cuh)
    TriCol* tri_tab_cl = nullptr;      // its per-column constants (chunk length = rows per CTA)
    SolveClArgs scl{};
    int scl_nc = 0, scl_threads = 0, scl_smem = 0, scl_lg_rpc = 0;
    ColTriRmKernel cols_tri_rm = nullptr;   // the same on a row-major spectrum (G = N/2), spec -> spec2
    float2* spec2 = nullptr;           // row-major mode: the solved spectrum (k_cols_tri_rm is out of place)
    dim3 trm_grid;
    int trm_threads = 0, trm_smem = 0, trm_mmax = 0;
    dim3 tri_grid;
    int tri_threads = 0, tri_smem = 0, tri_lg_cpc = 0;
    RhsKernel rhs = nullptr;
    RhsTmaKernel rhs_tma = nullptr;   // TMA-staged stencils (default; SRSB_TMA=0 selects k_rhs / k_wb)
    WbTmaKernel wb_tma[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    WbTmaKernel wb_tma_mon = nullptr;
    RhsMaps tmaps[2];                 // tensor maps, per w ping-pong buffer
    dim3 tgrid;
    int tsmem = 0, tsmem_wb = 0;
    RhsR2cKernel rhs_r2c = nullptr;   // fused RHS + row R2C cluster kernel (whole image, FFT solve, 128 <= N <= 1024)
    int fsmem = 0, fsr = 0, fnct = 0;  // its shared bytes, FFT row stride (float2), cluster size (CTAs per band)
    WbKernel wb[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    WbKernel wb_mon = nullptr;     // monitor variant (threshold mode, last pass)
    FftRowArgs ra{};
    FftColArgs ca{};
    StencilArgs sa{};
    dim3 rgrid, rblock, cgrid, cblock, sgrid, sblock;
    int rsmem = 0, csmem = 0, ssmem = 0;
    FftRowArgs ra_inv{};            // c2r launch shape (may use fewer rows per CTA than r2c when G = 1)
    dim3 rgrid_inv, rblock_inv;
    int rsmem_inv = 0;
    // NEXT-1 monitor: per image [E_g, E_a, E_r, E_pen, (|dphi_s|^2, |phi_s|^2) x S]
    double* stats = nullptr;
    int stats_stride = 0;
    float* prev_phi = nullptr;     // phi at the previous convergence check (sr_sb_iterate_until)
    double last_change = -1.0;     // outer relative change measured at the last check
    // NEXT-4 AOS phi solver: LR factors of (I - 2 tau mu A) along columns (M) and rows (N)
    float *aos_cpM = nullptr, *aos_rM = nullptr, *aos_cpN = nullptr, *aos_rN = nullptr;
    double* conv = nullptr;        // [batch][2] sums of the outer change
    double* mon_part = nullptr;    // per-CTA monitor partials (sr_reduce.cuh): [wb tiles][4] | [S][c2r CTAs][2] | [conv][2]
    size_t part_c2r = 0, part_conv = 0;   // offsets (doubles) of the c2r and outer-change regions
    // sr_sb_profile
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_cls;
    size_t ev_used = 0;
};

namespace {

constexpr int kConvBlocks = 64;   // CTAs per image of k_phi_change (sr_sb_iterate_until)

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

#define NK(call)                                                                               \
    do {                                                                                       \
        ncclResult_t r_ = (call);                                                              \
        if (r_ != ncclSuccess)                                                                 \
            return fail(c, SR_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));   \
    } while (0)

#define RET(x)                          \
    do {                                \
        sr_status r_ = (x);             \
        if (r_ != SR_OK) return r_;     \
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
    if (p->phi_solver != SR_PHI_FFT && p->phi_solver != SR_PHI_AOS) { msg = "bad phi_solver"; return SR_ERR_ARG; }
    if (p->phi_solver == SR_PHI_AOS && p->N > 8192) { msg = "AOS rows are staged in shared memory: N <= 8192"; return SR_ERR_ARG; }
    return SR_OK;
}

int ghost_rows(const sr_sb_params& p) {
    const int rblur = (int)std::ceil(3.0 * p.sigma);
    int gh = p.window > 1 ? p.window : 1;       // window halo, Laplacian / gradient / divergence
    if (rblur + 1 > gh) gh = rblur + 1;          // edge indicator: blur radius + central difference
    return gh;
}

// 3-D tiled tensor map over a field allocation: {N columns, rows per plane, planes}, fp32, box
// {bw, bh, 1}; out-of-bounds boxes are zero-filled.
bool encode_map3d(CUtensorMap* m, float* base, int N, int rows, int planes, int bw, int bh) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return false;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)rows, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)N * rows * 4};
    const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

sr_status configure(sr_sb_ctx* c) {
    const sr_sb_params& p = c->p;
    const int M = p.M, Ml = c->Ml, N = p.N, H = N / 2, B = p.batch, P = c->nranks;
    const int lgH = ilog2(H), lgM = ilog2(M);
    c->rfwd = pick_row_fwd(lgH);
    c->rinv = pick_row_inv(lgH);
    if (!c->rfwd || !c->rinv || !pick_col(lgM, false, false)) return fail(c, SR_ERR_SHAPE, "no FFT kernel for this size");
    {   // scale / symbol table of the column solve (fp64-computed, rounded once; L2-resident, <= 16 MB).
        // The column solve stages its column's entries into shared memory with cp.async at its start, so
        // the L2 latency hides behind the forward FFT (C3: 0.149 ms per launch; the correctly rounded
        // reciprocal of the fp32 symbol, SRSB_SYMTAB=0, also IEEE (Q20): 0.183 ms; round-1 table reads in
        // the middle of the kernel: 0.189 ms).
        const size_t nsym = (size_t)(H + 1) * M;
        const char* ev = std::getenv("SRSB_SYMTAB");
        c->use_sym = nsym <= ((size_t)4 << 20) && !(ev && ev[0] == '0');
    }
    // Launch shapes (measured on B200, C3: smaller CTAs overlap load and FFT phases better):
    //  rows: rpc rows per CTA, 64..512 threads, <= ~72 KB shared;  E = min(16, H) values per thread
    const int E_h = H < 16 ? H : 16, T_h = H / E_h;
    int rpc = 8;
    while (rpc * T_h < 64 && rpc < 32) rpc <<= 1;
    while ((rpc * T_h > 512 || rpc * (H + H / 16 + 32) * 8 > 72 * 1024) && rpc > 1) rpc >>= 1;
    if (rpc > Ml) rpc = Ml;
    if (const char* ev = std::getenv("SRSB_RPC")) {   // tuning knob (power of two)
        const int v = std::atoi(ev);
        if (v >= 1 && v <= Ml && v * T_h <= 512 && (v & (v - 1)) == 0) rpc = v;
    }
    //  column-group interleave of the transposed spectrum: rpc * G >= 8 complex = 64 B contiguous
    int G = 8 / rpc;
    if (G < 1) G = 1;
    if (M >= 4096 && !c->slab) G = 1;   // long columns: contiguous, so the column solve reads whole sectors
                                        // and can prefetch a column with one bulk copy (C5 +1.7 %; C4 14.46k -> 14.86k)
    const bool tri_on = !(std::getenv("SRSB_COLS_TRI") && std::getenv("SRSB_COLS_TRI")[0] == '0');
    if (c->slab && tri_on && p.phi_solver == SR_PHI_FFT) G = 1;   // the tridiagonal column pass wants contiguous column segments
    if (G > H / P) G = H / P;
    if (const char* ev = std::getenv("SRSB_G")) {     // tuning knob (power of two)
        const int v = std::atoi(ev);
        if (v >= 1 && v <= H / P && (v & (v - 1)) == 0) G = v;
    }
    // Row-major spectrum (G = N/2) with the cyclic tridiagonal column pass on it (sr_tri.cuh, k_cols_tri_rm): both
    // row passes then move whole lines instead of transposed chunks (measured with the generic row kernels: c2r
    // C3 0.185 -> 0.153 ms, C4 0.066 -> 0.046, C5 0.312 -> 0.208; r2c C5 0.194 -> 0.166).  Needs few carry terms
    // (tau mu not extreme), else the transposed layout stays.  Default for N >= 1024 (C1 / C2 measured slower: 313 vs
    // 342 and 4.2k vs 5.1k Mpx-iter/s); SRSB_SPEC_RM=1 forces it for N >= 64, SRSB_SPEC_RM=0: off.
    bool rm = false;
    int rm_mmax = 0;
    {
        const char* ev = std::getenv("SRSB_SPEC_RM");
        const char* et = std::getenv("SRSB_COLS_TRI");
        const int L = 1 << kTriLogL;
        if (!c->slab && p.phi_solver == SR_PHI_FFT && H >= (std::getenv("SRSB_SPEC_RM") ? 32 : 512) && M >= L && !(ev && ev[0] == '0') && !(et && et[0] == '0') &&
            !std::getenv("SRSB_G")) {
            const double a = (double)p.tau * (double)p.mu;
            const double r0 = tri_ratio(a, 1.0 + 2.0 * a, nullptr);   // k2 = 0: the slowest decay
            rm_mmax = tri_carry_terms(std::pow(r0, L), M / L, nullptr);
            rm = rm_mmax <= kTriRmMaxCarry;
        }
    }
    if (rm) {
        G = H;
        if (!std::getenv("SRSB_RPC")) {
            rpc = 64 / T_h > 1 ? 64 / T_h : 1;   // >= 64 threads per CTA (measured: C3 2-4 rows, C4 / C5 1 row)
            if (rpc > Ml) rpc = Ml;
        }
    }
    c->cols = pick_col(lgM, !c->slab && G == 1, c->use_sym);   // whole image, contiguous columns: immediate-offset access
    c->rfwd = pick_row_fwd_shape(lgH, ilog2(rpc), ilog2(G));
    //  columns per CTA: >= 64 threads, <= 512 (a CTA may cover part of a column group)
    const int Hl = H / P;                            // spectrum columns this context solves
    const int E_m = M < 16 ? M : 16, T_m = M / E_m;
    int cpc = 1;
    while (cpc * T_m < 64 && cpc * 2 <= Hl) cpc *= 2;
    if (const char* ev = std::getenv("SRSB_CPC")) {   // tuning knob (power of two)
        const int v = std::atoi(ev);
        if (v >= 1 && v <= Hl && v * T_m <= 512 && (v & (v - 1)) == 0) cpc = v;
    }
    if (cpc * T_m > 512) return fail(c, SR_ERR_SHAPE, "column FFT too large for one CTA");
    auto padded = [](int n, int extra) {   // float2 slots: one pad per 16, rounded to 16, + extra
        int sz = n + (n >> 4);
        sz = (sz + 15) & ~15;
        return sz + extra;
    };
    c->ra.plane = c->pitch;
    c->ra.M = Ml;
    c->ra.lg_rpc = ilog2(rpc);
    c->ra.lg_G = ilog2(G);
    // Row stride of the shared rows: the transposed store/gather visits (rr, k2) with rr in [0, rpc) and
    // G * rpc consecutive k2 per half-warp; SR = 16 / rpc (mod 16) makes rr * SR + k2 distinct mod 16,
    // i.e. conflict-free 8-byte accesses (the former SR = G (mod 16) gave 2-way conflicts).
    c->ra.SR = padded(H, rpc >= 16 ? 1 : (16 / rpc) & 15);
    c->ra.clip = 0.f;
    c->ra.accum = 0;
    c->rgrid = dim3(Ml / rpc, B, 1);
    c->rblock = dim3(rpc * T_h, 1, 1);
    c->rsmem = rpc * c->ra.SR * (int)sizeof(float2);
    {   // c2r: with contiguous columns (G = 1, whole image) the spectrum layout does not depend on the rows
        // per CTA, so the inverse pass may take its own (SRSB_RPC_INV, tuning knob)
        int ri = rpc;
        const char* ev = std::getenv("SRSB_RPC_INV");
        if (rm) {
            ri = 64 / T_h > 1 ? 64 / T_h : 1;       // row-major: >= 64 threads per CTA (C3: 2 rows 0.146 ms, 1 row 0.158; C4 / C5: 1 row)
            if (ri > Ml) ri = Ml;
        }
        if (ev && (G == 1 || rm) && !c->slab) {
            const int v = std::atoi(ev);
            if (v >= 2 && v <= Ml && v * T_h <= 512 && (v & (v - 1)) == 0) ri = v;
        }
        c->ra_inv = c->ra;
        c->ra_inv.lg_rpc = ilog2(ri);
        c->ra_inv.SR = padded(H, ri >= 16 ? 1 : (16 / ri) & 15);
        c->rgrid_inv = dim3(Ml / ri, B, 1);
        c->rblock_inv = dim3(ri * T_h, 1, 1);
        c->rsmem_inv = ri * c->ra_inv.SR * (int)sizeof(float2);
        if (SRSB_C2R_OLD_SMEM) c->rsmem_inv += ri * H * (int)sizeof(float2);   // psi staged in shared memory
        c->rinv = pick_row_inv_shape(lgH, ilog2(ri), ilog2(G));
    }
    {   // wide r2c (after the c2r took its own shape): with contiguous columns a 1024-thread CTA of 2 x rpc rows
        // writes 32-byte transposed chunks instead of 16 (C5, H = 4096: rpc = 2 -> 4; SRSB_R2C_WIDE=0: off)
        const char* ev = std::getenv("SRSB_R2C_WIDE");
        const int r2 = 2 * rpc;
        if (G == 1 && !c->slab && rpc * T_h == 512 && r2 <= Ml && !(ev && ev[0] == '0') &&
            pick_row_fwd_shape(lgH, ilog2(r2), 0) != pick_row_fwd(lgH)) {
            c->rfwd = pick_row_fwd_shape(lgH, ilog2(r2), 0);
            c->ra.lg_rpc = ilog2(r2);
            c->ra.SR = padded(H, r2 >= 16 ? 1 : (16 / r2) & 15);
            c->rgrid = dim3(Ml / r2, B, 1);
            c->rblock = dim3(r2 * T_h, 1, 1);
            c->rsmem = r2 * c->ra.SR * (int)sizeof(float2);
        }
    }
    c->ca.H = H;
    c->ca.lg_G = ilog2(G);
    c->ca.lg_cpc = ilog2(cpc);
    c->ca.SC = padded(M, 1);
    c->ca.taumu = p.tau * p.mu;
    c->ca.scale = (float)(1.0 / ((double)M * (double)H));
    if (c->slab) {   // columns of the all-to-all receive buffer: P segments of Ml rows
        c->ca.lg_seg = ilog2(Ml);
        c->ca.seg_stride = (long long)Hl * Ml;
        c->ca.bstride = (long long)H * Ml;           // unused (slab mode has one image)
        c->ca.k2_off = c->rank * Hl;
    } else {
        c->ca.lg_seg = ilog2(M);
        c->ca.seg_stride = 0;
        c->ca.bstride = (long long)H * M;
        c->ca.k2_off = 0;
    }
    {   // long contiguous columns (whole image, G = 1, M >= 4096): persistent prefetching solve
        const char* ev = std::getenv("SRSB_COLS_P");
        c->cols_p = (!c->slab && G == 1 && !(ev && ev[0] == '0')) ? pick_col_p(lgM, c->use_sym) : nullptr;
    }
    {   // cyclic tridiagonal column solve instead of FFT -> divide -> inverse FFT (sr_tri.cuh; SRSB_COLS_TRI=0: off)
        const char* ev = std::getenv("SRSB_COLS_TRI");
        const int L = 1 << kTriLogL;
        c->cols_tri = nullptr;
        if (G == 1 && M >= L && Ml >= L && !(ev && ev[0] == '0')) {   // slab: a chunk lies inside one segment (Ml >= L)
            const int C = M / L;                       // threads per column
            int tcpc = 1;
            int want = 128;   // threads per CTA (M <= 2048; one column needs M / 16): measured C3 0.0875 ms at 128, 0.0899 at 256, 0.105 at 512
            if (const char* e2 = std::getenv("SRSB_TRI_THREADS")) want = std::atoi(e2);
            while (tcpc * 2 * C <= want && tcpc * 2 <= Hl) tcpc *= 2;
            if (tcpc * C <= 512) {
                c->cols_tri = pick_col_tri();
                c->tri_lg_cpc = ilog2(tcpc);
                c->tri_threads = tcpc * C;
                c->tri_smem = tcpc * (M + 3 * C) * (int)sizeof(float2);
                c->tri_grid = dim3(Hl / tcpc, B, 1);
            }
        }
    }
    c->cols_tri_rm = nullptr;
    if (rm) {
        const int L = 1 << kTriLogL, C = M / L;
        int W = 8;    // chunk warps per CTA (measured C3 0.093 ms at 8, 0.101 at 16; C5 0.095 / 0.107)
        if (const char* e2 = std::getenv("SRSB_TRI_W")) W = std::atoi(e2);
        if (W < 1 || !is_pow2(W) || W > 16) W = 16;
        if (W > C) W = C;
        c->cols_tri_rm = pick_col_tri_rm();
        c->trm_mmax = rm_mmax;
        c->trm_threads = 32 * W;
        c->trm_smem = (W * L + 2 * (rm_mmax + W)) * 32 * (int)sizeof(float2);
        c->trm_grid = dim3(H / 32, C / W, B);
        if (!c->spec2 && cudaMalloc((void**)&c->spec2, (size_t)H * M * B * sizeof(float2)) != cudaSuccess)
            return fail(c, SR_ERR_OOM, "spectrum allocation failed");
    }
    c->solve_cl = nullptr;
    {   // small-image latency path: r2c + column solve + c2r in one cluster kernel (sr_solve_cl.cuh).  Default only for
        // images up to 128 x 128 (C1: 346 -> 379 Mpx-iter/s); a cluster is at most 16 CTAs, so larger images lose more
        // from running on 16 SMs than they gain from two launches fewer (C2 512^2: 5.1k -> 4.3k).  SRSB_SOLVE_CL=1 (or 5:
        // 32 rows per CTA) forces it wherever it applies (M <= 512, 128 <= N <= 512), 0 turns it off.
        const char* ev = std::getenv("SRSB_SOLVE_CL");
        const char* et = std::getenv("SRSB_COLS_TRI");
        const bool want = ev ? ev[0] != '0' : (M <= 128 && N <= 128);
        if (!c->slab && p.phi_solver == SR_PHI_FFT && want && !(et && et[0] == '0') && M >= 16 && M <= 512 &&
            H >= 64 && H <= 256) {
            int lr = M / 16 <= 16 ? 4 : 5;
            if (ev && ev[0] == '5' && M >= 32) lr = 5;
            const int nc = M >> lr, nt = (H / 16) << lr;
            SolveClKernel k = (nc >= 1 && nc <= 16 && nt >= H && nt <= 1024) ? pick_solve_cluster(lgH, lr) : nullptr;
            if (k) {
                const int SR = padded(H, 1);
                const int smem_b = ((1 << lr) * SR + 2 * H) * (int)sizeof(float2);
                bool ok = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_b) == cudaSuccess;
                if (ok && nc > 8)
                    ok = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = nc;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3(nc, B, 1);
                cfg.blockDim = dim3(nt, 1, 1);
                cfg.dynamicSmemBytes = smem_b;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int ncl = 0;
                if (ok && cudaOccupancyMaxActiveClusters(&ncl, (const void*)k, &cfg) == cudaSuccess && ncl > 0) {
                    c->solve_cl = k;
                    c->scl_nc = nc;
                    c->scl_threads = nt;
                    c->scl_smem = smem_b;
                    c->scl_lg_rpc = lr;
                    c->scl.plane = c->pitch;
                    c->scl.SR = SR;
                } else {
                    cudaGetLastError();
                }
            }
        }
    }
    c->cgrid = dim3(Hl / cpc, B, 1);
    if (c->slab) {   // all-to-all chunks (column groups) pipelined with the column solve; SRSB_A2A_CHUNKS
        int nk = 4;
        if (const char* ev = std::getenv("SRSB_A2A_CHUNKS")) nk = std::atoi(ev);
        const int unit = std::max(std::max(G, cpc), c->cols_tri ? (1 << c->tri_lg_cpc) : 1);   // a chunk holds whole column groups and whole column CTAs
        while (nk > 1 && (!is_pow2(nk) || nk > sr_sb_ctx::kMaxChunks || Hl / nk < unit || (Hl / nk) % unit)) nk--;
        c->a2a_chunks = std::max(nk, 1);
    }
    c->cblock = dim3(cpc * T_m, 1, 1);
    c->csmem = cpc * c->ca.SC * (int)sizeof(float2) + (c->use_sym ? cpc * M * (int)sizeof(float) : 0);
    // stencils
    int smem = 0;
    bool ok = pick_stencil(p.window, p.window_shape, p.l == p.epsilon, c->rhs, c->wb, c->wb_mon, smem);
    if (!ok) return fail(c, SR_ERR_ARG, "window radius not supported");
    c->ssmem = smem;
    c->sblock = dim3(32, ST_BY, 1);
    StencilArgs& a = c->sa;
    a.tiles_x = (N + ST_TW - 1) / ST_TW;
    a.tiles_y = (Ml + ST_TH - 1) / ST_TH;
    a.ntiles = a.tiles_x * a.tiles_y * B;
    a.M = Ml;
    a.N = N;
    a.Mg = M;
    a.row_off = c->row_off;
    a.slab = c->slab ? 1 : 0;
    a.plane = c->pitch;
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
    a.aos = p.phi_solver == SR_PHI_AOS ? 1 : 0;
    {
        const char* e = getenv("SRSB_BAND_SKIP");
        a.band_skip = (e && e[0] == '0') ? 0 : 1;
    }
    a.gh = c->gh;
    {   // TMA-staged RHS
        const char* e = getenv("SRSB_TMA");
        if (!(e && e[0] == '0') && pick_tma(p.window, p.window_shape, p.l == p.epsilon, c->rhs_tma, c->wb_tma,
                                             c->wb_tma_mon, c->tsmem, c->tsmem_wb)) {
            const int R = p.window, rows = Ml + 2 * c->gh;
            const int pw = tma_pw(R), ph = tma_ph(R);
            bool mok = true;
            for (int u = 0; u < 2; u++) {
                RhsMaps& m = c->tmaps[u];
                mok = mok && encode_map3d(&m.phi, c->phi_base, N, rows, B, pw, ph) &&
                      encode_map3d(&m.w, c->w_base[u], N, rows, 2 * B, pw, ph) &&
                      encode_map3d(&m.b, c->b_base, N, rows, 2 * B, TMA_BW, TMA_BH) &&
                      encode_map3d(&m.g, c->g_base, N, rows, B, ST_TW, TMA_TH) &&
                      encode_map3d(&m.bt, c->b_base, N, rows, 2 * B, ST_TW, TMA_TH);
            }
            if (!mok) return fail(c, SR_ERR_CUDA, "cuTensorMapEncodeTiled failed");
            c->tgrid = dim3(a.tiles_x, (Ml + TMA_TH - 1) / TMA_TH, B);
            CK(cudaFuncSetAttribute((const void*)c->rhs_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, c->tsmem));
            for (int m = 0; m < 2; m++)
                for (int u = 0; u < 2; u++)
                    CK(cudaFuncSetAttribute((const void*)c->wb_tma[m][u], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            c->tsmem_wb));
            CK(cudaFuncSetAttribute((const void*)c->wb_tma_mon, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    c->tsmem_wb));
        } else {
            c->rhs_tma = nullptr;
        }
    }
    {   // fused RHS + row R2C (sr_fused.cuh): one cluster per 32-row band, N / 64 CTAs.  Opt-in (SRSB_FUSE=1):
        // measured 2x slower than k_rhs_tma + k_rows_r2c on C3 (1.11 vs 0.555 ms per sweep): 16-CTA clusters
        // reach 21 active clusters (76 % of the CTA slots) and stall on the cluster barriers
        const char* e = getenv("SRSB_FUSE");
        c->rhs_r2c = nullptr;
        if (c->rhs_tma && !c->slab && p.phi_solver == SR_PHI_FFT && G == 1 && N >= 128 && N <= 1024 &&
            e && e[0] == '1') {
            int fs = 0;
            RhsR2cKernel k = pick_fused(p.window, p.window_shape, p.l == p.epsilon, lgH, fs);
            const int nct = N / ST_TW, rows = TMA_TH / nct;
            if (k) {
                CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, fs));
                if (nct > 8) CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = nct;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.gridDim = c->tgrid;
                cfg.blockDim = c->sblock;
                cfg.dynamicSmemBytes = fs;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)k, &cfg) == cudaSuccess && ncl > 0) {
                    c->rhs_r2c = k;
                    c->fsmem = fs;
                    c->fnct = nct;
                    c->fsr = padded(H, rows >= 16 ? 1 : (16 / rows) & 15);
                } else {
                    cudaGetLastError();
                }
            }
        }
    }
    // opt-in shared memory above 48 KB
    CK(cudaFuncSetAttribute((const void*)c->rfwd, cudaFuncAttributeMaxDynamicSharedMemorySize, c->rsmem));
    CK(cudaFuncSetAttribute((const void*)c->rinv, cudaFuncAttributeMaxDynamicSharedMemorySize, c->rsmem_inv));
    CK(cudaFuncSetAttribute((const void*)c->cols, cudaFuncAttributeMaxDynamicSharedMemorySize, c->csmem));
    if (c->cols_tri_rm)
        CK(cudaFuncSetAttribute((const void*)c->cols_tri_rm, cudaFuncAttributeMaxDynamicSharedMemorySize, c->trm_smem));
    if (c->cols_tri)
        CK(cudaFuncSetAttribute((const void*)c->cols_tri, cudaFuncAttributeMaxDynamicSharedMemorySize, c->tri_smem));
    if (c->cols_p) {
        c->cp_threads = M / 16;
        c->cp_smem = (M + c->ca.SC) * (int)sizeof(float2) + 16;
        CK(cudaFuncSetAttribute((const void*)c->cols_p, cudaFuncAttributeMaxDynamicSharedMemorySize, c->cp_smem));
        int per_sm = 0, nsm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->cols_p, c->cp_threads, c->cp_smem));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        c->cp_grid = std::max(1, std::min(B * (N / 2), per_sm * nsm));
    }
    CK(cudaFuncSetAttribute((const void*)c->rhs, cudaFuncAttributeMaxDynamicSharedMemorySize, c->ssmem));
    for (int m = 0; m < 2; m++)
        for (int u = 0; u < 2; u++)
            CK(cudaFuncSetAttribute((const void*)c->wb[m][u], cudaFuncAttributeMaxDynamicSharedMemorySize, c->ssmem));
    CK(cudaFuncSetAttribute((const void*)c->wb_mon, cudaFuncAttributeMaxDynamicSharedMemorySize, c->ssmem));
    if (p.phi_solver == SR_PHI_AOS)
        CK(cudaFuncSetAttribute((const void*)k_aos_horiz, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)aos_horiz_smem(N)));
    c->sgrid = dim3(a.tiles_x, a.tiles_y, B);
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
    if (c->use_sym) {   // scale / symbol(k1, k2) of Eq. (32) in fp64, rounded once to fp32 (Q10, Q20)
        std::vector<float> sym((size_t)(H + 1) * M);
        if (!c->sym && cudaMalloc((void**)&c->sym, sym.size() * sizeof(float)) != cudaSuccess)
            return fail(c, SR_ERR_OOM, "symbol table allocation failed");
        const double tm = (double)c->p.tau * (double)c->p.mu, scale = 1.0 / ((double)M * (double)H);
        for (int k2 = 0; k2 <= H; k2++)
            for (int k1 = 0; k1 < M; k1++)
                sym[(size_t)k2 * M + k1] = (float)(scale / (1.0 + tm * (4.0 - 2.0 * std::cos(2 * pi * k1 / M) -
                                                                        2.0 * std::cos(2 * pi * k2 / N))));
        CK(cudaMemcpyAsync(c->sym, sym.data(), sym.size() * sizeof(float), cudaMemcpyHostToDevice, c->s));
    }
    c->ca.sym = c->sym;
    // per-column constants of the cyclic tridiagonal solve for chunk length L (C chunks per column), fp64 -> fp32
    auto tri_table = [&](int L, int C, TriCol** dst, int* mmax_out) -> sr_status {
        std::vector<TriCol> tab(H);
        const double a = (double)c->p.tau * (double)c->p.mu;
        int mall = 1;
        auto fill = [&](TriCol& t, int comp, int k2, int& mmax) {
            double sq = 1.0, clos = 1.0;
            const double r = tri_ratio(a, 1.0 + a * (4.0 - 2.0 * std::cos(2 * pi * k2 / N)), &sq);
            const double rho = std::pow(r, L);
            const int m = tri_carry_terms(rho, C, &clos);
            t.r[comp] = (float)r;
            t.ks[comp] = (float)(1.0 / (sq * (double)H));
            t.rho[comp] = (float)rho;
            t.clos[comp] = (float)clos;
            mmax = std::max(mmax, m);
        };
        for (int k2 = 0; k2 < H; k2++) {
            int mm = 1;
            fill(tab[k2], 0, k2, mm);
            fill(tab[k2], 1, k2 == 0 ? H : k2, mm);   // slot 0: imaginary part = the real column k2 = N/2
            tab[k2].mmax = mm;
            tab[k2].pad_[0] = tab[k2].pad_[1] = tab[k2].pad_[2] = 0;
            mall = std::max(mall, mm);
        }
        if (!*dst && cudaMalloc((void**)dst, H * sizeof(TriCol)) != cudaSuccess)
            return fail(c, SR_ERR_OOM, "tridiagonal table allocation failed");
        CK(cudaMemcpyAsync(*dst, tab.data(), H * sizeof(TriCol), cudaMemcpyHostToDevice, c->s));
        CK(cudaStreamSynchronize(c->s));   // tab is a local
        if (mmax_out) *mmax_out = mall;
        return SR_OK;
    };
    if (c->cols_tri || c->cols_tri_rm) RET(tri_table(1 << kTriLogL, M >> kTriLogL, &c->tri_tab, nullptr));
    if (c->solve_cl) RET(tri_table(1 << c->scl_lg_rpc, c->scl_nc, &c->tri_tab_cl, &c->scl.mmax));
    if (c->p.phi_solver == SR_PHI_AOS) {   // LR factors once, fp64 -> fp32
        auto factors = [&](int n, std::vector<float>& cp, std::vector<float>& r) {
            const double cc = 2.0 * (double)c->p.tau * (double)c->p.mu, a = -cc;
            cp.assign(n, 0.f);
            r.assign(n, 0.f);
            double cprev = 0.0;
            for (int i = 0; i < n; i++) {
                const double diag = (i == 0 || i == n - 1) ? 1.0 + cc : 1.0 + 2.0 * cc;
                const double d = diag - (i > 0 ? a * cprev : 0.0);
                r[i] = (float)(1.0 / d);
                cprev = a / d;
                cp[i] = (float)cprev;
            }
        };
        std::vector<float> cpM, rM, cpN, rN;
        factors(M, cpM, rM);
        factors(N, cpN, rN);
        CK(cudaMemcpyAsync(c->aos_cpM, cpM.data(), M * 4, cudaMemcpyHostToDevice, c->s));
        CK(cudaMemcpyAsync(c->aos_rM, rM.data(), M * 4, cudaMemcpyHostToDevice, c->s));
        CK(cudaMemcpyAsync(c->aos_cpN, cpN.data(), N * 4, cudaMemcpyHostToDevice, c->s));
        CK(cudaMemcpyAsync(c->aos_rN, rN.data(), N * 4, cudaMemcpyHostToDevice, c->s));
    }
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

void enq_r2c(sr_sb_ctx* c, const float* F) {
    prof_begin(c);
    c->rfwd<<<c->rgrid, c->rblock, c->rsmem, c->s>>>(F, c->spec, c->twH, c->twR, c->ra);
    prof_end(c, SR_K_ROWS_R2C);
}
void enq_cols(sr_sb_ctx* c) {
    prof_begin(c);
    if (c->cols_tri_rm)
        c->cols_tri_rm<<<c->trm_grid, c->trm_threads, c->trm_smem, c->s>>>(c->spec, c->spec2, c->tri_tab, ilog2(c->p.M),
                                                                           c->ca.lg_G, c->p.N / 2, c->trm_mmax, 0);
    else if (c->cols_tri)
        c->cols_tri<<<c->tri_grid, c->tri_threads, c->tri_smem, c->s>>>(c->slab ? c->spec_cols : c->spec,
                                                                        c->tri_tab + c->ca.k2_off, ilog2(c->p.M),
                                                                        c->tri_lg_cpc, c->ca.bstride, c->ca.lg_seg,
                                                                        c->ca.seg_stride);
    else if (c->cols_p)
        c->cols_p<<<c->cp_grid, c->cp_threads, c->cp_smem, c->s>>>(c->spec, c->twM, c->cM, c->cN, c->ca,
                                                                  c->p.batch * (c->p.N / 2), ilog2(c->p.N / 2));
    else
        c->cols<<<c->cgrid, c->cblock, c->csmem, c->s>>>(c->slab ? c->spec_cols : c->spec, c->twM, c->cM, c->cN,
                                                         c->ca);
    prof_end(c, SR_K_COLS_SOLVE);
}
// slab mode: the column solve of chunk k of nk (columns [k, k+1) Hl/nk of this slab), on stream st
void enq_cols_chunk(sr_sb_ctx* c, int k, int nk, cudaStream_t st) {
    const int Hl = c->p.N / 2 / c->nranks, Hk = Hl / nk;
    FftColArgs ca = c->ca;
    ca.k2_off += k * Hk;
    prof_begin(c);
    if (c->cols_tri)
        c->cols_tri<<<dim3(Hk >> c->tri_lg_cpc, 1, 1), c->tri_threads, c->tri_smem, st>>>(
            c->spec_cols + (size_t)k * Hk * c->Ml, c->tri_tab + ca.k2_off, ilog2(c->p.M), c->tri_lg_cpc, ca.bstride,
            ca.lg_seg, ca.seg_stride);
    else
        c->cols<<<dim3(Hk >> ca.lg_cpc, 1, 1), c->cblock, c->csmem, st>>>(c->spec_cols + (size_t)k * Hk * c->Ml, c->twM,
                                                                           c->cM, c->cN, ca);
    prof_end(c, SR_K_COLS_SOLVE);
}
void enq_c2r(sr_sb_ctx* c, float* out, float clip, int accum, int sweep = -1) {
    FftRowArgs ra = c->ra_inv;
    ra.accum = accum;
    ra.clip = clip;
    const bool mon = c->stats && sweep >= 0;
    ra.stats = mon ? c->mon_part + c->part_c2r + (size_t)sweep * c->rgrid_inv.x * c->p.batch * 2 : nullptr;
    ra.stats_stride = c->stats_stride;
    prof_begin(c);
    c->rinv<<<c->rgrid_inv, c->rblock_inv, c->rsmem_inv, c->s>>>(c->cols_tri_rm ? c->spec2 : c->spec, out, c->twH, c->twR, ra);
    prof_end(c, SR_K_ROWS_C2R);
    if (mon)   // ||phi^{s+1} - phi^s||^2, ||phi^s||^2 per image, summed in a fixed order
        k_reduce_partials<<<c->p.batch * 2, 32, 0, c->s>>>(ra.stats, (int)c->rgrid_inv.x, 2, c->stats + 4 + 2 * sweep,
                                                           c->stats_stride);
}
// the phi solve of one sweep: F -> out (+= when accum), clamped when clip > 0.  Small images: one cluster kernel
// (not with the NEXT-1 monitor, whose per-sweep sums live in the c2r pass)
void enq_solve(sr_sb_ctx* c, const float* F, float* out, float clip, int accum, int sweep = -1) {
    if (c->solve_cl && !(c->stats && sweep >= 0)) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c->scl_nc;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(c->scl_nc, c->p.batch, 1);
        cfg.blockDim = dim3(c->scl_threads, 1, 1);
        cfg.dynamicSmemBytes = c->scl_smem;
        cfg.stream = c->s;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SolveClArgs a = c->scl;
        a.clip = clip;
        a.accum = accum;
        prof_begin(c);
        cudaLaunchKernelEx(&cfg, c->solve_cl, F, out, (const float2*)c->twH, (const float2*)c->twR,
                           (const TriCol*)c->tri_tab_cl, a);
        prof_end(c, SR_K_SOLVE_CLUSTER);
        return;
    }
    enq_r2c(c, F);
    enq_cols(c);
    enq_c2r(c, out, clip, accum, sweep);
}
void enq_rhs(sr_sb_ctx* c, float* F) {
    prof_begin(c);
    if (c->rhs_tma)
        c->rhs_tma<<<c->tgrid, c->sblock, c->tsmem, c->s>>>(c->tmaps[c->wcur], c->phi, F, c->sa);
    else
        c->rhs<<<c->sgrid, c->sblock, c->ssmem, c->s>>>(c->phi, c->w[c->wcur], c->b, c->g, F, c->sa);
    prof_end(c, SR_K_RHS);
}
// fused RHS + row R2C: D of Eq. (37) (increment form) straight into the transposed half spectrum
void enq_rhs_r2c(sr_sb_ctx* c) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->fnct;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = c->tgrid;
    cfg.blockDim = c->sblock;
    cfg.dynamicSmemBytes = c->fsmem;
    cfg.stream = c->s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    prof_begin(c);
    cudaLaunchKernelEx(&cfg, c->rhs_r2c, (const RhsMaps)c->tmaps[c->wcur], (const float*)c->phi, c->spec,
                       (const float2*)c->twH, (const float2*)c->twR, c->sa, c->fsr);
    prof_end(c, SR_K_RHS_R2C);
}
void enq_wb_pass(sr_sb_ctx* c, int last) {
    prof_begin(c);
    const bool mon = c->stats && last && c->p.w_mode == SR_W_THRESHOLD;
    if (c->rhs_tma) {
        WbTmaKernel k = mon ? c->wb_tma_mon : c->wb_tma[c->p.w_mode][last];
        k<<<c->tgrid, c->sblock, c->tsmem_wb, c->s>>>(c->tmaps[c->wcur], c->w[c->wcur ^ 1], c->b, c->flag, c->sa);
    } else {
        WbKernel k = mon ? c->wb_mon : c->wb[c->p.w_mode][last];
        k<<<c->sgrid, c->sblock, c->ssmem, c->s>>>(c->phi, c->w[c->wcur], c->w[c->wcur ^ 1], c->b, c->g, c->flag,
                                                   c->sa);
    }
    prof_end(c, SR_K_WB);
    if (mon) {   // Eq. (22) terms per image from the per-tile partials, in a fixed order
        const dim3 gr = c->rhs_tma ? c->tgrid : c->sgrid;
        k_reduce_partials<<<c->p.batch * 4, 32, 0, c->s>>>(c->mon_part, (int)(gr.x * gr.y), 4, c->stats,
                                                           c->stats_stride);
    }
    c->wcur ^= 1;
}

// ------------------------------------------------------------------ slab exchanges
enum HaloField { HF_PHI = 0, HF_W = 1, HF_B = 2, HF_IMG = 3 };

// plane pointer (local row 0) of channel ch of field f (B = 1 in slab mode)
float* field_rows(sr_sb_ctx* c, int f, int ch) {
    switch (f) {
        case HF_PHI: return c->phi;
        case HF_W: return c->w[c->wcur] + ch * c->pitch;
        case HF_B: return c->b + ch * c->pitch;
        default: return c->F;   // HF_IMG: the image staged in F during set_image
    }
}

// ---- the exchange schedule (host-only; no CUDA): one list of point-to-point ops per rank.  Both
// backends execute exactly these lists -- NCCL as grouped ncclSend / ncclRecv, LOCAL as device
// copies pairing the k-th send from r to d with the k-th receive on d from r (NCCL's per-peer FIFO
// matching) -- and sr_sb_slab_schedule exports them so the CPU tests can run the same lists across
// processes (gloo) and check every offset, count and pairing without a GPU.
struct XOp {
    int send;         // 1 send, 0 receive
    int peer;         // the other rank
    int buf;          // halo: channel of the field; a2a: 0 = row-pass spectrum, 1 = column buffer
    long long off;    // elements from the buffer's base (halo: local row 0 of the channel plane)
    long long cnt;    // elements
};

// Ghost rows of one channel plane: A: last gh rows of r -> top ghost of r+1; B: first gh rows of r
// -> bottom ghost of r-1; C (wrap = phi, the periodic Laplacian rows of Eq. (32)): last rows of P-1
// -> top ghost of 0, first rows of 0 -> bottom ghost of P-1.  Same phase order on every rank.
void halo_ops(int P, int r, int Ml, int gh, int N, bool wrap, int ch, std::vector<XOp>& ops) {
    const long long cnt = (long long)gh * N, top = -(long long)gh * N, bot = (long long)Ml * N,
                    last = (long long)(Ml - gh) * N;
    if (r + 1 < P) ops.push_back({1, r + 1, ch, last, cnt});
    if (r > 0) ops.push_back({0, r - 1, ch, top, cnt});
    if (r > 0) ops.push_back({1, r - 1, ch, 0, cnt});
    if (r + 1 < P) ops.push_back({0, r + 1, ch, bot, cnt});
    if (wrap) {
        if (r == P - 1) ops.push_back({1, 0, ch, last, cnt});
        if (r == 0) ops.push_back({0, P - 1, ch, top, cnt});
        if (r == 0) ops.push_back({1, P - 1, ch, 0, cnt});
        if (r == P - 1) ops.push_back({0, 0, ch, bot, cnt});
    }
}

// Spectrum transpose, chunk `k` of `nk`: the row pass leaves slab r's spectrum as [H/G][Ml][G], so
// the columns [d H/P, (d+1) H/P) bound for slab d are one contiguous block of blk = (H/P) Ml
// complex; chunk k is the contiguous sub-block of its columns [k, k+1) (H/P)/nk, sub = blk / nk.
// Slab d stores the block from src as segment src of its column buffer [P][H/(P G)][Ml][G]
// (offset src blk + k sub).  fwd: spectrum -> column buffer; bwd: the reverse.  Counts in floats.
void a2a_ops(int P, int r, long long blk, int k, int nk, bool fwd, std::vector<XOp>& ops) {
    const long long sub = blk / nk;
    for (int d = 0; d < P; d++) {
        // send to d its block, receive from d our segment d (same chunk of the same columns)
        const long long soff = (long long)d * blk + (long long)k * sub;
        ops.push_back({1, d, fwd ? 0 : 1, 2 * soff, 2 * sub});
        ops.push_back({0, d, fwd ? 1 : 0, 2 * soff, 2 * sub});
    }
}

// plane pointer (local row 0) of channel ch of field f (B = 1 in slab mode)
float* xbuf(sr_sb_ctx* c, int f, int buf) {
    if (f < 0) return reinterpret_cast<float*>(buf == 0 ? c->spec : c->spec_cols);
    return field_rows(c, f, buf);
}

// Execute per-rank op lists.  LOCAL: ops[r] for every slab r of `m`; NCCL: ops[0] for this rank.
sr_status run_ops(std::vector<sr_sb_ctx*>& m, int f, const std::vector<std::vector<XOp>>& ops, cudaStream_t st) {
    sr_sb_ctx* c = m[0];
    if (c->backend == BK_LOCAL) {
        const int P = (int)m.size();
        // recv queues per (dst, src) pair in program order
        std::vector<std::vector<size_t>> nxt(P * P, std::vector<size_t>());
        for (int d = 0; d < P; d++)
            for (size_t i = 0; i < ops[d].size(); i++)
                if (!ops[d][i].send) nxt[d * P + ops[d][i].peer].push_back(i);
        std::vector<size_t> used(P * P, 0);
        for (int r = 0; r < P; r++)
            for (const XOp& o : ops[r]) {
                if (!o.send) continue;
                const int d = o.peer;
                auto& q = nxt[d * P + r];
                size_t& u = used[d * P + r];
                if (u >= q.size()) return fail(c, SR_ERR_STATE, "slab schedule: a send without a matching receive");
                const XOp& rv = ops[d][q[u++]];
                if (rv.cnt != o.cnt) return fail(c, SR_ERR_STATE, "slab schedule: send/receive counts differ");
                CK(cudaMemcpyAsync(xbuf(m[d], f, rv.buf) + rv.off, xbuf(m[r], f, o.buf) + o.off,
                                   (size_t)o.cnt * sizeof(float), cudaMemcpyDeviceToDevice, st));
            }
        for (int i = 0; i < P * P; i++)
            if (used[i] != nxt[i].size()) return fail(c, SR_ERR_STATE, "slab schedule: a receive without a send");
        return SR_OK;
    }
    if (c->backend == BK_NCCL) {
        const std::vector<XOp>& L = ops[0];
        if (c->nranks == 1) {   // a one-rank communicator: self pairs as local copies (FIFO order)
            std::vector<const XOp*> sends, recvs;
            for (const XOp& o : L) (o.send ? sends : recvs).push_back(&o);
            if (sends.size() != recvs.size()) return fail(c, SR_ERR_STATE, "slab schedule: unpaired self op");
            for (size_t i = 0; i < sends.size(); i++)
                CK(cudaMemcpyAsync(xbuf(c, f, recvs[i]->buf) + recvs[i]->off, xbuf(c, f, sends[i]->buf) + sends[i]->off,
                                   (size_t)sends[i]->cnt * sizeof(float), cudaMemcpyDeviceToDevice, st));
            return SR_OK;
        }
        NK(ncclGroupStart());
        for (const XOp& o : L) {
            float* p = xbuf(c, f, o.buf) + o.off;
            if (o.send) NK(ncclSend(p, (size_t)o.cnt, ncclFloat, o.peer, c->comm, st));
            else NK(ncclRecv(p, (size_t)o.cnt, ncclFloat, o.peer, c->comm, st));
        }
        NK(ncclGroupEnd());
    }
    return SR_OK;
}

sr_status halo(std::vector<sr_sb_ctx*>& m, int f, bool wrap) {
    sr_sb_ctx* c = m[0];
    const int nch = (f == HF_W || f == HF_B) ? 2 : 1;
    std::vector<std::vector<XOp>> ops(m.size());
    for (size_t i = 0; i < m.size(); i++)
        for (int ch = 0; ch < nch; ch++)
            halo_ops(c->nranks, m[i]->rank, c->Ml, c->gh, c->p.N, wrap, ch, ops[i]);
    return run_ops(m, f, ops, c->s);
}

// Spectrum transpose chunk k of nk between the row pass and the column pass (fwd) and back (bwd).
sr_status alltoall(std::vector<sr_sb_ctx*>& m, bool fwd, int k, int nk, cudaStream_t st) {
    sr_sb_ctx* c = m[0];
    const long long blk = (long long)(c->p.N / 2 / c->nranks) * c->Ml;   // complex per (src, dst) pair
    std::vector<std::vector<XOp>> ops(m.size());
    for (size_t i = 0; i < m.size(); i++) a2a_ops(c->nranks, m[i]->rank, blk, k, nk, fwd, ops[i]);
    return run_ops(m, -1, ops, st);
}

// ------------------------------------------------------------------ the iteration
// NEXT-4: phi = 1/2 [(I - c A_1)^-1 + (I - c A_2)^-1] F with F the full RHS (AOS)
void enq_aos(sr_sb_ctx* c, const float* F, float* out, float clip) {
    AosArgs q;
    q.M = c->Ml;
    q.N = c->p.N;
    q.plane = c->pitch;
    q.a = -2.f * c->p.tau * c->p.mu;
    q.clip = clip;
    float* Y = c->w[c->wcur ^ 1];          // scratch: the w ping-pong target is free during the sweeps
    float* Xv = Y + c->pitch * c->p.batch;  // its second half (the [B][2] planes hold 2 B planes)
    prof_begin(c);
    if (q.M <= AOS_VREG_MAXM) {
        const int L = q.M < 32 ? q.M : 32, CH = q.M / L;
        const int CW = std::min(std::min(32, AOS_VT / CH), q.N);
        const dim3 grd(q.N / CW, c->p.batch), blk(CW, CH);
        const size_t sm = 4 * (size_t)CH * CW * sizeof(float);
        if (L == 8) k_aos_vert_reg<8><<<grd, blk, sm, c->s>>>(F, Xv, c->aos_cpM, c->aos_rM, q);
        else if (L == 16) k_aos_vert_reg<16><<<grd, blk, sm, c->s>>>(F, Xv, c->aos_cpM, c->aos_rM, q);
        else k_aos_vert_reg<32><<<grd, blk, sm, c->s>>>(F, Xv, c->aos_cpM, c->aos_rM, q);
    } else {
        k_aos_vert<<<dim3((q.N + 127) / 128, c->p.batch), 128, 0, c->s>>>(F, Y, Xv, c->aos_cpM, c->aos_rM, q);
    }
    prof_end(c, SR_K_AOS_VERT);
    prof_begin(c);
    const int wpb = aos_horiz_wpb(q.N);
    k_aos_horiz<<<dim3((q.M + wpb - 1) / wpb, c->p.batch), 32 * wpb, aos_horiz_smem(q.N), c->s>>>(
        F, Xv, out, c->aos_cpN, c->aos_rN, q);
    prof_end(c, SR_K_AOS_HORIZ);
}

sr_status enq_iteration(sr_sb_ctx* c) {   // whole-image context
    if (c->stats) cudaMemsetAsync(c->stats, 0, sizeof(double) * c->stats_stride * c->p.batch, c->s);
    for (int s = 0; s < c->p.S; s++) {
        const float clip = (s == c->p.S - 1) ? c->p.phi_clip : 0.f;
        if (c->rhs_r2c) {
            enq_rhs_r2c(c);
            enq_cols(c);
            enq_c2r(c, c->phi, clip, 1, s);
            continue;
        }
        enq_rhs(c, c->F);
        if (c->p.phi_solver == SR_PHI_AOS) {
            enq_aos(c, c->F, c->phi, clip);
        } else {
            enq_solve(c, c->F, c->phi, clip, 1, s);
        }
    }
    const int passes = c->p.w_mode == SR_W_FIXED_POINT ? c->p.w_iters : 1;
    for (int r = 0; r < passes; r++) enq_wb_pass(c, r == passes - 1);
    return SR_OK;
}

// slab schedule over the member contexts.  The phi solve of each sweep runs
//   r2c -> [all-to-all chunk 0 .. nk-1 on the comm stream] -> per chunk k: wait chunk k, column solve
//   of chunk k on the work stream, then its backward all-to-all on the comm stream -> join -> c2r,
// so the transfer of chunk k + 1 (and the return of chunk k - 1) overlaps the column solve of chunk k.
sr_status slab_phi_solve(std::vector<sr_sb_ctx*>& m, float clip) {
    sr_sb_ctx* c0 = m[0];
    for (auto* x : m) enq_r2c(x, x->F);
    const int nk = c0->a2a_chunks;
    if (nk <= 1) {
        RET(alltoall(m, true, 0, 1, c0->s));
        for (auto* x : m) enq_cols_chunk(x, 0, 1, c0->s);
        RET(alltoall(m, false, 0, 1, c0->s));
    } else {
        sr_sb_ctx* c = c0;
        cudaEvent_t* fwd = c0->xev + 1;
        cudaEvent_t* col = c0->xev + 1 + nk;
        cudaEvent_t fork = c0->xev[0], join = c0->xev[2 * sr_sb_ctx::kMaxChunks + 1];
        CK(cudaEventRecord(fork, c0->s));
        CK(cudaStreamWaitEvent(c0->sc, fork, 0));
        for (int k = 0; k < nk; k++) {
            RET(alltoall(m, true, k, nk, c0->sc));
            CK(cudaEventRecord(fwd[k], c0->sc));
        }
        for (int k = 0; k < nk; k++) {
            CK(cudaStreamWaitEvent(c0->s, fwd[k], 0));
            for (auto* x : m) enq_cols_chunk(x, k, nk, c0->s);
            CK(cudaEventRecord(col[k], c0->s));
            CK(cudaStreamWaitEvent(c0->sc, col[k], 0));
            RET(alltoall(m, false, k, nk, c0->sc));
        }
        CK(cudaEventRecord(join, c0->sc));
        CK(cudaStreamWaitEvent(c0->s, join, 0));
    }
    for (auto* x : m) enq_c2r(x, x->phi, clip, 1);
    return SR_OK;
}

sr_status slab_iteration(std::vector<sr_sb_ctx*>& m) {
    sr_sb_ctx* c0 = m[0];
    const sr_sb_params& p = c0->p;
    for (int s = 0; s < p.S; s++) {
        RET(halo(m, HF_PHI, true));
        for (auto* x : m) enq_rhs(x, x->F);
        RET(slab_phi_solve(m, (s == p.S - 1) ? p.phi_clip : 0.f));
    }
    RET(halo(m, HF_PHI, true));
    const int passes = p.w_mode == SR_W_FIXED_POINT ? p.w_iters : 1;
    for (int r = 0; r < passes; r++) {
        if (r > 0) RET(halo(m, HF_W, false));
        for (auto* x : m) enq_wb_pass(x, r == passes - 1);
    }
    RET(halo(m, HF_W, false));
    RET(halo(m, HF_B, false));
    return SR_OK;
}

std::vector<sr_sb_ctx*> group_of(sr_sb_ctx* c) {
    if (c->backend == BK_LOCAL) return c->members;
    return std::vector<sr_sb_ctx*>{c};
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

// order the work stream after the caller's stream, and back
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

// copy `nplanes` image planes of Ml rows between a dense caller buffer ([nplanes][Ml][N], host or
// device) and a field with ghost rows (planes `pitch` floats apart)
sr_status copy_planes(sr_sb_ctx* c, float* field, const float* dense, int nplanes, bool to_field) {
    const size_t rowbytes = (size_t)c->Ml * c->p.N * 4;
    if (to_field)
        CK(cudaMemcpy2DAsync(field, (size_t)c->pitch * 4, dense, rowbytes, rowbytes, nplanes, cudaMemcpyDefault, c->s));
    else
        CK(cudaMemcpy2DAsync(const_cast<float*>(dense), rowbytes, field, (size_t)c->pitch * 4, rowbytes, nplanes,
                             cudaMemcpyDefault, c->s));
    return SR_OK;
}

// ------------------------------------------------------------------ creation
sr_status create_one(const sr_sb_params* p, int device, cudaStream_t stream, int nranks, int rank, int backend,
                     cudaStream_t shared_work, sr_sb_ctx** out) {
    *out = nullptr;
    sr_sb_ctx* c = new sr_sb_ctx();
    c->p = *p;
    c->device = device;
    c->user = stream;
    c->nranks = nranks;
    c->rank = rank;
    c->backend = backend;
    c->slab = backend != BK_NONE;
    c->Ml = p->M / nranks;
    c->row_off = rank * c->Ml;
    c->gh = ghost_rows(*p);
    c->pitch = (long long)(c->Ml + 2 * c->gh) * p->N;
    const size_t nplane = (size_t)c->pitch * p->batch;           // floats per scalar field
    const size_t nspec = (size_t)(p->N / 2) * c->Ml * p->batch;  // complex per spectrum
    auto alloc = [&](void** ptr, size_t bytes) -> bool {
        if (cudaMalloc(ptr, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
        return true;
    };
    bool ok = true;
    if (shared_work) {
        c->s = shared_work;
        c->own_stream = false;
    } else {
        ok = cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking) == cudaSuccess;
    }
    ok = ok && cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) == cudaSuccess;
    if (ok && c->slab) {
        ok = cudaStreamCreateWithFlags(&c->sc, cudaStreamNonBlocking) == cudaSuccess;
        for (auto& e : c->xev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) { g_create_err = "stream/event creation failed"; sr_sb_destroy(c); return SR_ERR_CUDA; }
    ok = alloc((void**)&c->phi_base, nplane * 4) && alloc((void**)&c->F_base, nplane * 4) &&
         alloc((void**)&c->w_base[0], 2 * nplane * 4) && alloc((void**)&c->w_base[1], 2 * nplane * 4) &&
         alloc((void**)&c->b_base, 2 * nplane * 4) && alloc((void**)&c->g_base, nplane * 4) &&
         alloc((void**)&c->spec, nspec * sizeof(float2)) && alloc((void**)&c->twH, p->N / 2 * sizeof(float2)) &&
         alloc((void**)&c->twM, p->M * sizeof(float2)) && alloc((void**)&c->twR, p->N / 2 * sizeof(float2)) &&
         alloc((void**)&c->cM, p->M * sizeof(float)) && alloc((void**)&c->cN, (p->N / 2 + 1) * sizeof(float)) &&
         alloc((void**)&c->flag, sizeof(int));
    if (ok && c->slab) ok = alloc((void**)&c->spec_cols, nspec * sizeof(float2));
    if (ok && p->phi_solver == SR_PHI_AOS)
        ok = alloc((void**)&c->aos_cpM, p->M * 4) && alloc((void**)&c->aos_rM, p->M * 4) &&
             alloc((void**)&c->aos_cpN, p->N * 4) && alloc((void**)&c->aos_rN, p->N * 4);
    if (!ok) { g_create_err = "device allocation failed"; sr_sb_destroy(c); return SR_ERR_OOM; }
    const size_t off = (size_t)c->gh * p->N;
    c->phi = c->phi_base + off;
    c->F = c->F_base + off;
    c->w[0] = c->w_base[0] + off;
    c->w[1] = c->w_base[1] + off;
    c->b = c->b_base + off;
    c->g = c->g_base + off;
    // ghost rows start defined (zero): never read as data outside the image
    bool zok = cudaMemsetAsync(c->phi_base, 0, nplane * 4, c->s) == cudaSuccess &&
               cudaMemsetAsync(c->F_base, 0, nplane * 4, c->s) == cudaSuccess &&
               cudaMemsetAsync(c->w_base[0], 0, 2 * nplane * 4, c->s) == cudaSuccess &&
               cudaMemsetAsync(c->w_base[1], 0, 2 * nplane * 4, c->s) == cudaSuccess &&
               cudaMemsetAsync(c->b_base, 0, 2 * nplane * 4, c->s) == cudaSuccess &&
               cudaMemsetAsync(c->g_base, 0, nplane * 4, c->s) == cudaSuccess &&
               cudaMemsetAsync(c->flag, 0, sizeof(int), c->s) == cudaSuccess;
    if (!zok) { g_create_err = "memset failed"; sr_sb_destroy(c); return SR_ERR_CUDA; }
    sr_status st = configure(c);
    if (st == SR_OK) st = make_tables(c);
    if (st != SR_OK) { g_create_err = c->err; sr_sb_destroy(c); return st; }
    *out = c;
    return SR_OK;
}

sr_status check_device(int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        g_create_err = "no CUDA device " + std::to_string(device);
        return SR_ERR_CUDA;
    }
    return SR_OK;
}

sr_status validate_slab(const sr_sb_params* p, int nranks, std::string& msg) {
    if (nranks < 1 || !is_pow2(nranks)) { msg = "nranks must be a power of two"; return SR_ERR_ARG; }
    if (p->batch != 1) { msg = "slab mode decomposes one image: batch must be 1"; return SR_ERR_ARG; }
    if (p->phi_solver != SR_PHI_FFT) { msg = "slab mode uses the FFT phi solver"; return SR_ERR_ARG; }
    const int Ml = p->M / nranks, gh = ghost_rows(*p);
    if (Ml < 8 || Ml < gh) { msg = "too many slabs: local rows must be >= 8 and >= the ghost rows"; return SR_ERR_SHAPE; }
    if ((p->N / 2) % nranks != 0) { msg = "N/2 must be divisible by nranks"; return SR_ERR_SHAPE; }
    return SR_OK;
}

// set_image for a list of slab contexts or one whole-image context; image/phi0 already staged
// into F / phi of each context (local rows)
sr_status enq_setup(std::vector<sr_sb_ctx*>& m) {
    sr_sb_ctx* c = m[0];
    const sr_sb_params& p = c->p;
    EdgeArgs ea{};
    ea.N = p.N;
    ea.Mg = p.M;
    ea.r = (int)std::ceil(3.0 * p.sigma);
    double ks = 0.0, kk[17];
    for (int t = -ea.r; t <= ea.r; t++) { kk[t + ea.r] = std::exp(-(double)t * t / (2.0 * p.sigma * p.sigma)); ks += kk[t + ea.r]; }
    for (int t = 0; t <= 2 * ea.r; t++) ea.k[t] = (float)(kk[t] / ks);
    ea.rho = p.rho;
    ea.s = p.s;
    ea.plane = c->pitch;
    if (c->slab) {
        RET(halo(m, HF_IMG, false));   // image rows for the blur (ghost rows >= r + 1)
        RET(halo(m, HF_PHI, true));    // phi0 rows for w0 = grad phi0
    }
    for (auto* x : m) {
        EdgeArgs e = ea;
        e.M = x->Ml;
        e.row_off = x->row_off;
        const int ext = x->slab ? ea.r + 1 : 0;
        float* tmp = x->w[1];   // scratch: free until the first w/b update
        const dim3 blk(128);
        e.ext = ext;
        k_blur_rows<<<dim3((p.N + 127) / 128, x->Ml + 2 * ext, p.batch), blk, 0, x->s>>>(x->F, tmp, e);
        e.ext = x->slab ? 1 : 0;
        k_blur_cols<<<dim3((p.N + 127) / 128, x->Ml + 2 * e.ext, p.batch), blk, 0, x->s>>>(tmp, x->F, e);
        e.ext = 0;
        k_edge_g<<<dim3((p.N + 127) / 128, x->Ml, p.batch), blk, 0, x->s>>>(x->F, x->g, e);
        x->wcur = 0;
        k_init_w<<<dim3((p.N + 127) / 128, x->Ml, p.batch), blk, 0, x->s>>>(x->phi, x->w[0], x->b, p.N, p.M, x->row_off,
                                                                             x->pitch);
        sr_sb_ctx* c = x;
        CK(cudaMemsetAsync(x->flag, 0, sizeof(int), x->s));
    }
    if (c->slab) {
        RET(halo(m, HF_W, false));
        RET(halo(m, HF_B, false));
    }
    return SR_OK;
}

}  // namespace

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
    p->phi_solver = SR_PHI_FFT;
}

sr_status sr_sb_create(const sr_sb_params* p, int device, void* stream, sr_sb_ctx** out) {
    if (!out) { g_create_err = "out is NULL"; return SR_ERR_ARG; }
    *out = nullptr;
    std::string msg;
    sr_status st = validate(p, msg);
    if (st != SR_OK) { g_create_err = msg; return st; }
    RET(check_device(device));
    DevGuard dg(device);
    return create_one(p, device, (cudaStream_t)stream, 1, 0, BK_NONE, nullptr, out);
}

sr_status sr_sb_create_slab_group(const sr_sb_params* p, int device, void* stream, int nslabs, sr_sb_ctx** out) {
    if (!out) { g_create_err = "out is NULL"; return SR_ERR_ARG; }
    *out = nullptr;
    std::string msg;
    sr_status st = validate(p, msg);
    if (st == SR_OK) st = validate_slab(p, nslabs, msg);
    if (st != SR_OK) { g_create_err = msg; return st; }
    RET(check_device(device));
    DevGuard dg(device);
    sr_sb_ctx* L = new sr_sb_ctx();
    L->p = *p;
    L->device = device;
    L->user = (cudaStream_t)stream;
    L->nranks = nslabs;
    L->backend = BK_LOCAL;
    L->slab = true;
    L->Ml = p->M;
    if (cudaStreamCreateWithFlags(&L->s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_out, cudaEventDisableTiming) != cudaSuccess) {
        g_create_err = "stream/event creation failed";
        sr_sb_destroy(L);
        return SR_ERR_CUDA;
    }
    for (int r = 0; r < nslabs; r++) {
        sr_sb_ctx* m = nullptr;
        st = create_one(p, device, L->s, nslabs, r, BK_LOCAL, L->s, &m);
        if (st != SR_OK) { sr_sb_destroy(L); return st; }
        L->members.push_back(m);
    }
    *out = L;
    return SR_OK;
}

sr_status sr_sb_nccl_unique_id(void* id_out, int bytes) {
    if (!id_out || bytes < (int)sizeof(ncclUniqueId)) { g_create_err = "need NCCL_UNIQUE_ID_BYTES"; return SR_ERR_ARG; }
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) { g_create_err = ncclGetErrorString(r); return SR_ERR_NCCL; }
    std::memcpy(id_out, &id, sizeof(id));
    return SR_OK;
}

sr_status sr_sb_create_slab_nccl(const sr_sb_params* p, int device, void* stream, int nranks, int rank,
                                 const void* nccl_id, sr_sb_ctx** out) {
    if (!out || !nccl_id) { g_create_err = "out and nccl_id must be non-NULL"; return SR_ERR_ARG; }
    *out = nullptr;
    std::string msg;
    sr_status st = validate(p, msg);
    if (st == SR_OK) st = validate_slab(p, nranks, msg);
    if (st == SR_OK && (rank < 0 || rank >= nranks)) { msg = "bad rank"; st = SR_ERR_ARG; }
    if (st != SR_OK) { g_create_err = msg; return st; }
    RET(check_device(device));
    DevGuard dg(device);
    st = create_one(p, device, (cudaStream_t)stream, nranks, rank, BK_NCCL, nullptr, out);
    if (st != SR_OK) return st;
    sr_sb_ctx* c = *out;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        g_create_err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        c->comm = nullptr;
        sr_sb_destroy(c);
        *out = nullptr;
        return SR_ERR_NCCL;
    }
    return SR_OK;
}

sr_status sr_sb_create_dist(const sr_sb_params* p, int device, void* stream, const void* nccl_unique_id,
                            int nranks, int rank, sr_sb_ctx** out) {
    return sr_sb_create_slab_nccl(p, device, stream, nranks, rank, nccl_unique_id, out);
}

int sr_sb_local_rows(const sr_sb_ctx* c) { return c ? c->Ml : -1; }

sr_status sr_sb_set_image(sr_sb_ctx* c, const float* image, const float* phi0) {
    if (!c) return SR_ERR_ARG;
    if (!image || !phi0) return fail(c, SR_ERR_ARG, "image and phi0 must be non-NULL");
    DevGuard dg(c->device);
    RET(begin(c));
    std::vector<sr_sb_ctx*> m = group_of(c);
    for (auto* x : m) {   // LOCAL group: scatter the slabs' rows of the full image
        const size_t off = (c->backend == BK_LOCAL) ? (size_t)x->row_off * c->p.N : 0;
        sr_status st = copy_planes(x, x->F, image + off, c->p.batch, true);
        if (st == SR_OK) st = copy_planes(x, x->phi, phi0 + off, c->p.batch, true);
        if (st != SR_OK) return fail(c, st, x->err);
    }
    sr_status st = enq_setup(m);
    if (st != SR_OK) return fail(c, st, m[0]->err);
    RET(end(c));
    for (auto* x : m) {
        x->k = 0;
        x->have_state = true;
    }
    c->k = 0;
    c->have_state = true;
    return SR_OK;
}

void drop_graphs(sr_sb_ctx* c) {
    for (auto& g : c->graph)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

// w ping-pong parity of the context (a LOCAL group: of its slabs, which flip together)
int group_wcur(sr_sb_ctx* c) { return c->backend == BK_LOCAL ? c->members[0]->wcur : c->wcur; }

// Capture kGraphIters iterations (whole image: the 13-kernel iteration; slab mode: kernels, the
// halo / all-to-all exchanges -- NCCL calls or the LOCAL device copies -- and the comm-stream
// fork/join of the chunked transpose) into the graph of the current w parity.
static sr_status build_graph(sr_sb_ctx* c) {
    const int par = group_wcur(c);
    if (c->graph[par]) { cudaGraphExecDestroy(c->graph[par]); c->graph[par] = nullptr; }
    std::vector<sr_sb_ctx*> m = group_of(c);
    std::vector<int> w0;
    for (auto* x : m) w0.push_back(x->wcur);
    cudaGraph_t gr;
    CK(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
    sr_status st = SR_OK;
    for (int i = 0; i < kGraphIters && st == SR_OK; i++) st = c->slab ? slab_iteration(m) : enq_iteration(c);
    cudaError_t e = cudaStreamEndCapture(c->s, &gr);
    for (size_t i = 0; i < m.size(); i++) m[i]->wcur = w0[i];   // capture did not execute anything
    if (st != SR_OK) {
        if (e == cudaSuccess) cudaGraphDestroy(gr);
        return fail(c, st, m[0]->err);
    }
    if (e != cudaSuccess) return fail(c, SR_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->graph[par], gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) { c->graph[par] = nullptr; return fail(c, SR_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e)); }
    return SR_OK;
}

sr_status sr_sb_iterate(sr_sb_ctx* c, int K) {
    if (!c) return SR_ERR_ARG;
    if (K < 0) return fail(c, SR_ERR_ARG, "K must be >= 0");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "iterate before set_image/set_state");
    if (K == 0) return SR_OK;
    DevGuard dg(c->device);
    RET(begin(c));
    std::vector<sr_sb_ctx*> m = group_of(c);
    const char* ev = std::getenv("SRSB_GRAPH");   // 0: direct launches only (A/B and debugging)
    const bool use_graph = !(ev && ev[0] == '0');
    int done = 0;
    if (use_graph && K >= kGraphIters) {
        const int par = group_wcur(c);
        if (!c->graph[par]) RET(build_graph(c));
        for (; done + kGraphIters <= K; done += kGraphIters) CK(cudaGraphLaunch(c->graph[par], c->s));
        // the graph's w ping-pong flips are even, so the parity is unchanged
    }
    for (; done < K; done++) {
        const sr_status st = c->slab ? slab_iteration(m) : enq_iteration(c);
        if (st != SR_OK) return fail(c, st, m[0]->err);
    }
    RET(end(c));
    if (c->backend == BK_LOCAL)
        for (auto* x : c->members) x->k += K;
    c->k += K;
    return SR_OK;
}

sr_status sr_sb_sync(sr_sb_ctx* c) {
    if (!c) return SR_ERR_ARG;
    DevGuard dg(c->device);
    CK(cudaStreamSynchronize(c->s));
    CK(cudaStreamSynchronize(c->user));
    if (c->comm) {
        ncclResult_t ae = ncclSuccess;
        NK(ncclCommGetAsyncError(c->comm, &ae));
        if (ae != ncclSuccess) return fail(c, SR_ERR_NCCL, std::string("NCCL async: ") + ncclGetErrorString(ae));
    }
    for (auto* x : group_of(c)) {
        int flag = 0;
        CK(cudaMemcpy(&flag, x->flag, sizeof(int), cudaMemcpyDeviceToHost));
        if (flag) return fail(c, SR_ERR_NONFINITE, "non-finite value or |b| > b_max detected in the w/b update");
    }
    return SR_OK;
}

sr_status sr_sb_get_phi(sr_sb_ctx* c, float* phi_out) {
    if (!c) return SR_ERR_ARG;
    if (!phi_out) return fail(c, SR_ERR_ARG, "phi_out is NULL");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    DevGuard dg(c->device);
    RET(begin(c));
    for (auto* x : group_of(c)) {
        const size_t off = (c->backend == BK_LOCAL) ? (size_t)x->row_off * c->p.N : 0;
        sr_status st = copy_planes(x, x->phi, phi_out + off, c->p.batch, false);
        if (st != SR_OK) return fail(c, st, x->err);
    }
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_get_state(sr_sb_ctx* c, float* phi, float* w, float* b, float* g) {
    if (!c) return SR_ERR_ARG;
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    if (c->backend == BK_LOCAL && (w || b)) return fail(c, SR_ERR_ARG, "slab groups expose phi and g only");
    DevGuard dg(c->device);
    RET(begin(c));
    for (auto* x : group_of(c)) {
        const size_t off = (c->backend == BK_LOCAL) ? (size_t)x->row_off * c->p.N : 0;
        sr_status st = SR_OK;
        if (phi && st == SR_OK) st = copy_planes(x, x->phi, phi + off, c->p.batch, false);
        if (w && st == SR_OK) st = copy_planes(x, x->w[x->wcur], w, 2 * c->p.batch, false);
        if (b && st == SR_OK) st = copy_planes(x, x->b, b, 2 * c->p.batch, false);
        if (g && st == SR_OK) st = copy_planes(x, x->g, g + off, c->p.batch, false);
        if (st != SR_OK) return fail(c, st, x->err);
    }
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_set_state(sr_sb_ctx* c, const float* phi, const float* w, const float* b, const float* g) {
    if (!c) return SR_ERR_ARG;
    if (!phi || !w || !b) return fail(c, SR_ERR_ARG, "phi, w and b must be non-NULL");
    if (!g && !c->have_state) return fail(c, SR_ERR_STATE, "g is required before set_image");
    if (c->slab) return fail(c, SR_ERR_ARG, "set_state is not available in slab mode");
    DevGuard dg(c->device);
    RET(begin(c));
    RET(copy_planes(c, c->phi, phi, c->p.batch, true));
    RET(copy_planes(c, c->w[c->wcur], w, 2 * c->p.batch, true));
    RET(copy_planes(c, c->b, b, 2 * c->p.batch, true));
    if (g) RET(copy_planes(c, c->g, g, c->p.batch, true));
    CK(cudaMemsetAsync(c->flag, 0, sizeof(int), c->s));
    RET(end(c));
    c->k = 0;
    c->have_state = true;
    return SR_OK;
}

long long sr_sb_iteration(const sr_sb_ctx* c) { return c ? c->k : -1; }
sr_status sr_sb_set_iteration(sr_sb_ctx* c, long long k) {
    if (!c) return SR_ERR_ARG;
    if (k < 0) return fail(c, SR_ERR_ARG, "k must be >= 0");
    c->k = k;
    return SR_OK;
}

sr_status sr_sb_debug_solve(sr_sb_ctx* c, const float* F, float* phi_out) {
    if (!c) return SR_ERR_ARG;
    if (!F || !phi_out) return fail(c, SR_ERR_ARG, "NULL pointer");
    if (c->slab) return fail(c, SR_ERR_ARG, "debug entries are for whole-image contexts");
    DevGuard dg(c->device);
    RET(begin(c));
    RET(copy_planes(c, c->F, F, c->p.batch, true));
    // solve into F's own buffer is not allowed (rows read F while c2r writes); use w[1] as output
    if (c->p.phi_solver == SR_PHI_AOS) {   // AOS: F is the full RHS; k_aos_horiz may write in place
        enq_aos(c, c->F, c->F, 0.f);
        RET(copy_planes(c, c->F, phi_out, c->p.batch, false));
    } else {
        float* tmp = c->w[c->wcur ^ 1];
        enq_solve(c, c->F, tmp, 0.f, 0);
        RET(copy_planes(c, tmp, phi_out, c->p.batch, false));
    }
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_debug_rhs(sr_sb_ctx* c, float* F_out) {
    if (!c) return SR_ERR_ARG;
    if (!F_out) return fail(c, SR_ERR_ARG, "NULL pointer");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    if (c->slab) return fail(c, SR_ERR_ARG, "debug entries are for whole-image contexts");
    DevGuard dg(c->device);
    RET(begin(c));
    enq_rhs(c, c->F);
    RET(copy_planes(c, c->F, F_out, c->p.batch, false));
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_debug_wb(sr_sb_ctx* c) {
    if (!c) return SR_ERR_ARG;
    if (!c->have_state) return fail(c, SR_ERR_STATE, "no state");
    if (c->slab) return fail(c, SR_ERR_ARG, "debug entries are for whole-image contexts");
    DevGuard dg(c->device);
    RET(begin(c));
    const int passes = c->p.w_mode == SR_W_FIXED_POINT ? c->p.w_iters : 1;
    for (int r = 0; r < passes; r++) enq_wb_pass(c, r == passes - 1);
    RET(end(c));
    return SR_OK;
}

sr_status sr_sb_profile(sr_sb_ctx* c, int K, float* ms_out, int* launches_out) {
    if (!c) return SR_ERR_ARG;
    if (K < 1 || !ms_out || !launches_out) return fail(c, SR_ERR_ARG, "K >= 1 and non-NULL outputs required");
    if (!c->have_state) return fail(c, SR_ERR_STATE, "profile before set_image/set_state");
    if (c->slab) return fail(c, SR_ERR_ARG, "profile is for whole-image contexts");
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

sr_status sr_sb_set_monitor(sr_sb_ctx* c, int enable) {
    if (!c) return SR_ERR_ARG;
    if (c->slab) return fail(c, SR_ERR_ARG, "the monitor is for whole-image contexts");
    DevGuard dg(c->device);
    CK(cudaStreamSynchronize(c->s));
    if (enable && !c->stats) {
        c->stats_stride = 4 + 2 * c->p.S;
        CK(cudaMalloc((void**)&c->stats, sizeof(double) * c->stats_stride * c->p.batch));
        CK(cudaMemset(c->stats, 0, sizeof(double) * c->stats_stride * c->p.batch));
        CK(cudaMalloc((void**)&c->prev_phi, sizeof(float) * c->pitch * c->p.batch));
        CK(cudaMemset(c->prev_phi, 0, sizeof(float) * c->pitch * c->p.batch));
        CK(cudaMalloc((void**)&c->conv, sizeof(double) * 2 * c->p.batch));
        const size_t B = c->p.batch;
        const size_t nwb = (size_t)c->sgrid.x * std::max(c->sgrid.y, c->tgrid.y) * B * 4;
        const size_t nc2r = (size_t)c->p.S * c->rgrid_inv.x * B * 2;
        c->part_c2r = nwb;
        c->part_conv = nwb + nc2r;
        CK(cudaMalloc((void**)&c->mon_part, sizeof(double) * (nwb + nc2r + kConvBlocks * B * 2)));
    } else if (!enable && c->stats) {
        CK(cudaFree(c->stats));
        CK(cudaFree(c->prev_phi));
        CK(cudaFree(c->conv));
        CK(cudaFree(c->mon_part));
        c->stats = nullptr;
        c->prev_phi = nullptr;
        c->conv = nullptr;
        c->mon_part = nullptr;
    }
    c->sa.stats = c->mon_part;
    c->sa.stats_stride = c->stats_stride;
    drop_graphs(c);   // the captured graphs bake the kernel arguments: rebuild on the next iterate
    return SR_OK;
}

sr_status sr_sb_get_monitor(sr_sb_ctx* c, double* out) {
    if (!c || !out) return SR_ERR_ARG;
    if (!c->stats) return fail(c, SR_ERR_STATE, "monitor not enabled (sr_sb_set_monitor)");
    DevGuard dg(c->device);
    CK(cudaStreamSynchronize(c->s));
    CK(cudaMemcpy(out, c->stats, sizeof(double) * c->stats_stride * c->p.batch, cudaMemcpyDeviceToHost));
    return SR_OK;
}

sr_status sr_sb_iterate_until(sr_sb_ctx* c, int K_max, double tol, int every, int* k_done) {
    if (!c) return SR_ERR_ARG;
    if (K_max < 0 || every < 1 || !(tol >= 0.0)) return fail(c, SR_ERR_ARG, "need K_max >= 0, every >= 1, tol >= 0");
    if (!c->stats) return fail(c, SR_ERR_STATE, "monitor not enabled (sr_sb_set_monitor)");
    DevGuard dg(c->device);
    const int B = c->p.batch;
    const dim3 grd(kConvBlocks, B), blk(256);
    const size_t off = (size_t)c->gh * c->p.N;
    std::vector<double> cv(2 * B);
    // snapshot phi^k
    double* part = c->mon_part + c->part_conv;
    k_phi_change<<<grd, blk, 0, c->s>>>(c->phi, c->prev_phi + off, part, c->Ml, c->p.N, c->pitch, 2);
    int done = 0;
    while (done < K_max) {
        const int n = (K_max - done) < every ? (K_max - done) : every;
        RET(sr_sb_iterate(c, n));
        done += n;
        // outer relative change ||phi^k - phi^{k-n}|| / (||phi^{k-n}|| + 1e-6)  (SPEC's outer rule)
        k_phi_change<<<grd, blk, 0, c->s>>>(c->phi, c->prev_phi + off, part, c->Ml, c->p.N, c->pitch, 2);
        k_reduce_partials<<<B * 2, 32, 0, c->s>>>(part, kConvBlocks, 2, c->conv, 2);
        CK(cudaMemcpyAsync(cv.data(), c->conv, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        double worst = 0.0;
        for (int b = 0; b < B; b++) {
            const double r = std::sqrt(cv[2 * b]) / (std::sqrt(cv[2 * b + 1]) + 1e-6);
            if (r > worst) worst = r;
        }
        c->last_change = worst;
        if (worst <= tol) break;
    }
    if (k_done) *k_done = done;
    return SR_OK;
}

double sr_sb_last_change(const sr_sb_ctx* c) { return c ? c->last_change : -1.0; }

int sr_sb_launches_per_iteration(const sr_sb_ctx* c) {
    if (!c) return -1;
    // rhs + (r2c, cols, c2r | vert, horiz | the one-kernel cluster solve); fused: rhs_r2c, cols, c2r
    const int per_sweep = (c->p.phi_solver == SR_PHI_AOS || c->rhs_r2c) ? 3 : (c->solve_cl && !c->stats) ? 2 : 4;
    const int per = per_sweep * c->p.S + (c->p.w_mode == SR_W_FIXED_POINT ? c->p.w_iters : 1);
    return c->backend == BK_LOCAL ? per * (int)c->members.size() : per;
}

void sr_sb_destroy(sr_sb_ctx* c) {
    if (!c) return;
    DevGuard dg(c->device);
    if (c->s) cudaStreamSynchronize(c->s);
    for (auto* m : c->members) sr_sb_destroy(m);
    c->members.clear();
    if (c->comm) ncclCommDestroy(c->comm);
    drop_graphs(c);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    void* ptrs[] = {c->phi_base, c->F_base, c->w_base[0], c->w_base[1], c->b_base, c->g_base, c->spec,
                    c->spec_cols, c->twH, c->twM, c->twR, c->cM, c->cN, c->sym, c->tri_tab, c->tri_tab_cl, c->spec2, c->flag, c->stats, c->prev_phi, c->conv, c->mon_part,
                    c->aos_cpM, c->aos_rM, c->aos_cpN, c->aos_rN};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_out) cudaEventDestroy(c->ev_out);
    for (cudaEvent_t e : c->xev)
        if (e) cudaEventDestroy(e);
    if (c->sc) cudaStreamDestroy(c->sc);
    if (c->s && c->own_stream) cudaStreamDestroy(c->s);
    delete c;
}

const char* sr_sb_last_error(const sr_sb_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int sr_sb_slab_schedule(int kind, int P, int r, int Ml, int gh, int N, int k, int nk, long long* out, int max_ops) {
    if (P < 1 || r < 0 || r >= P || Ml < 1 || gh < 1 || N < 2 || nk < 1 || k < 0 || k >= nk || kind < 0 || kind > 3)
        return -1;
    std::vector<XOp> ops;
    if (kind <= 1) {
        halo_ops(P, r, Ml, gh, N, kind == 0, 0, ops);
    } else {
        const long long blk = (long long)(N / 2 / P) * Ml;
        if ((N / 2) % P || blk % nk) return -1;
        a2a_ops(P, r, blk, k, nk, kind == 2, ops);
    }
    if (out) {
        if ((int)ops.size() > max_ops) return -1;
        for (size_t i = 0; i < ops.size(); i++) {
            long long* q = out + 5 * i;
            q[0] = ops[i].send; q[1] = ops[i].peer; q[2] = ops[i].buf; q[3] = ops[i].off; q[4] = ops[i].cnt;
        }
    }
    return (int)ops.size();
}

int sr_sb_tri_constants(float tau, float mu, int N, int k2, int L, int C, double* out) {
    if (!out || N < 2 || k2 < 0 || k2 > N / 2 || L < 1 || C < 1 || !(tau >= 0.f) || !(mu > 0.f)) return -1;
    const double a = (double)tau * (double)mu;
    double sq = 1.0, clos = 1.0;
    const double r = tri_ratio(a, 1.0 + a * (4.0 - 2.0 * std::cos(2 * 3.14159265358979323846 * k2 / N)), &sq);
    const double rho = std::pow(r, L);
    const int m = tri_carry_terms(rho, C, &clos);
    out[0] = r;
    out[1] = 1.0 / sq;
    out[2] = rho;
    out[3] = clos;
    out[4] = (double)m;
    return 0;
}

int sr_sb_a2a_chunks(const sr_sb_ctx* c) { return c ? (c->backend == BK_LOCAL ? c->members[0]->a2a_chunks : c->a2a_chunks) : -1; }

}  // extern "C"
