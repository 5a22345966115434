/*
 * srsb.h -- C ABI of the B200-native Split Bregman Self-repelling Snake library (libsrsb.so).
 *
 * Method: Pan et al., "Using the Split Bregman Algorithm to Solve the
 * Self-repelling Snake Model", arXiv 2003.12693.  "P:n" is line n of the
 * paper's LaTeX source; equation numbers are LaTeX's.  Readings
 * where the paper is silent or garbled are the Q-items of DESIGN.md §2.
 *
 * What the library computes: for a batch of B images of
 * M x N pixels (fp32), Algorithm 1:
 *   set_image:  g = 1/(1 + rho |grad(G_sigma * f)|^s)              Eq. (1)
 *               phi = phi0, w = grad phi0, b = 0                    Alg. 1 (1)
 *   iterate(K): K times { S times { F = Eq. (37) RHS; phi = Re F^-1(F(F)/symbol) Eq. (33) };
 *                         phi = clamp(phi, -phi_clip, phi_clip)     (north star, Q9)
 *                         w = proj(shrink(B)) Eq. (41),(42),(40);  b += grad phi - w  Eq. (23) }
 * All arithmetic runs in hand-written sm_100a CUDA kernels; there is no
 * CPU fallback.
 *
 * Conventions (all calls):
 *  - Fields are row-major float32: scalar fields [batch][M][N]; vector fields
 *    (w, b) [batch][2][M][N] with channel 0 the row (i) component and channel
 *    1 the column (j) component of Eq. (35).  phi < 0 is INSIDE (Eq. 3).
 *  - Pointers may be device pointers on the context's device OR host
 *    pointers (pinned or pageable); copies use cudaMemcpyDefault under UVA.
 *    The caller owns every buffer; the library copies in/out during the call
 *    and never retains caller pointers.
 *  - All calls are stream-ordered on the context's stream and asynchronous
 *    with respect to the host for device pointers; call sr_sb_sync before
 *    reading outputs.  With pageable host pointers the copy is synchronous.
 *  - Argument validation is synchronous and happens before any enqueue;
 *    errors return a negative sr_status and set sr_sb_last_error(ctx).
 *  - A context is bound to one device and one stream and is not thread-safe.
 */
#ifndef SRSB_H
#define SRSB_H

#ifdef __cplusplus
extern "C" {
#endif

#define SRSB_ABI_VERSION 3   /* 2: SR_K_RHS_R2C (SR_K_NCLASSES 7 -> 8); 3: SR_K_SOLVE_CLUSTER (8 -> 9) */

typedef enum {
    SR_OK = 0,
    SR_ERR_ARG = -1,        /* invalid parameter or NULL pointer */
    SR_ERR_SHAPE = -2,      /* M, N not powers of two in [8, 8192], batch < 1 */
    SR_ERR_CUDA = -3,       /* CUDA runtime error; message in sr_sb_last_error */
    SR_ERR_NCCL = -4,       /* NCCL error (slab mode); message in sr_sb_last_error */
    SR_ERR_NONFINITE = -5,  /* NaN/Inf or |b| > b_max latched by the w/b kernel */
    SR_ERR_STATE = -6,      /* call order violated (e.g. iterate before set_image) */
    SR_ERR_OOM = -7         /* device allocation failed */
} sr_status;

typedef enum { SR_WIN_DISC = 0, SR_WIN_SQUARE = 1 } sr_window_shape;   /* Q2 */
typedef enum { SR_WPROJ_BALL = 0, SR_WPROJ_SPHERE = 1, SR_WPROJ_NONE = 2 } sr_wproj;  /* Eq. (40), Q1 */
typedef enum { SR_W_THRESHOLD = 0, SR_W_FIXED_POINT = 1 } sr_wmode;   /* Eq. (42) / Eq. (39) */

typedef struct {
    int   M, N, batch;         /* rows, columns (powers of two, 8..8192), images in this context */
    float gamma, alpha, beta;  /* Eq. (7): geodesic length, balloon, repulsion weights */
    float mu;                  /* Eq. (22): Bregman penalty */
    float epsilon;             /* Eq. (5),(6): half-width of the regularized H / delta */
    float l;                   /* Eq. (11): narrow-band offset of h (the PAPER's l) */
    float d;                   /* Eq. (10): Gaussian scale exp(-|x-y|^2/d^2) */
    int   window;              /* summation radius R of the window (BASELINE's "l"), 0..8 */
    int   window_shape;        /* sr_window_shape: disc p^2+q^2 <= R^2 (default) or square */
    float tau;                 /* Eq. (30),(37): time step of a phi sweep */
    int   S;                   /* phi sweeps (FFT solves) per outer iteration, >= 1 (Q7) */
    float rho, sigma;          /* Eq. (1): edge scale, Gaussian pre-smoothing std (radius ceil(3 sigma) <= 8) */
    int   s;                   /* Eq. (1): power, 1 or 2 */
    float phi_clip;            /* > 0: clamp phi^{k+1} to [-phi_clip, phi_clip] after the last sweep; 0: off */
    int   w_proj;              /* sr_wproj (Q1) */
    int   w_mode;              /* sr_wmode */
    int   w_iters;             /* fixed-point sweeps r for SR_W_FIXED_POINT (Eq. 38-39), >= 1 */
    float b_max;               /* guard: |b| > b_max latches SR_ERR_NONFINITE (SPEC S:366 uses 50); <= 0 off */
    int   phi_solver;          /* sr_phi_solver: FFT solve of Eq. (31)-(33) (default) or the AOS variant of P:427 */
} sr_sb_params;

typedef enum { SR_PHI_FFT = 0, SR_PHI_AOS = 1 } sr_phi_solver;   /* AOS: whole-image contexts only */

typedef struct sr_sb_ctx sr_sb_ctx;

/* Fill *p with the defaults of DESIGN.md §2 (Fig. 1 caption P:465 with readings Q17, Q22). */
void sr_sb_default_params(sr_sb_params* p, int M, int N, int batch, int window);

/* Validate p, allocate all state on `device` (fields, spectrum, tables) and bind
 * the context to `stream` (a cudaStream_t; NULL = the legacy default stream).
 * Device memory: about 44 bytes per pixel plus 2 x max(window, ceil(3 sigma)+1) ghost rows per
 * image plane. */
sr_status sr_sb_create(const sr_sb_params* p, int device, void* stream, sr_sb_ctx** out);

/* ---- Slab decomposition of ONE large image (batch must be 1) into P = nranks row slabs
 * (BASELINE configs[4]).  Slab r holds global rows [r M/P, (r+1) M/P); the
 * repulsion / divergence / gradient stencils read ghost rows filled by halo exchanges with the
 * neighbouring slabs, the phi solve transposes the packed half spectrum with an all-to-all
 * between its row pass and its column pass and back (Eq. 31-33 unchanged: the same butterflies
 * as one GPU, so P slabs reproduce P = 1 bitwise).  Requirements: P a power of two,
 * (N/2) % P == 0, M/P >= 8 and >= the ghost rows (max(window, ceil(3 sigma) + 1)).
 *
 * sr_sb_create_slab_group: all P slab contexts in this process on `device`, exchanges as device
 *   copies (the single-GPU emulation of the multi-GPU schedule).  The returned handle presents
 *   the FULL image: set_image / get_phi / get_state(phi, g) take [1][M][N] buffers; set_state,
 *   profile and the debug entries are not available.
 * sr_sb_create_slab_nccl: this process's slab `rank` of `nranks`, one process per GPU; halos by
 *   ncclSend/ncclRecv, the transpose by ncclAlltoAll, on the context's stream (NVLink /
 *   NVSwitch).  `nccl_id` = NCCL_UNIQUE_ID_BYTES (128) bytes from sr_sb_nccl_unique_id on one
 *   rank, broadcast by the caller.  Buffers of set_image / get_phi / get_state are the LOCAL rows
 *   [1][M/P][N] (sr_sb_local_rows). */
sr_status sr_sb_create_slab_group(const sr_sb_params* p, int device, void* stream, int nslabs, sr_sb_ctx** out);
sr_status sr_sb_nccl_unique_id(void* id_out, int bytes);
sr_status sr_sb_create_slab_nccl(const sr_sb_params* p, int device, void* stream, int nranks, int rank,
                                 const void* nccl_id, sr_sb_ctx** out);
/* SURVEY §8(b)'s name and argument order for the NCCL slab context: the same as
 * sr_sb_create_slab_nccl(p, device, stream, nranks, rank, nccl_unique_id, out). */
sr_status sr_sb_create_dist(const sr_sb_params* p, int device, void* stream, const void* nccl_unique_id,
                            int nranks, int rank, sr_sb_ctx** out);
/* Rows per image held in the caller-visible buffers of this context (M, or M/P for an NCCL slab). */
int sr_sb_local_rows(const sr_sb_ctx* ctx);

/* The slab exchange schedule (host-only, needs no GPU).  Both slab backends execute
 * exactly these per-rank lists of point-to-point ops: NCCL as grouped ncclSend / ncclRecv, the
 * LOCAL group as device copies pairing the k-th send from r to d with the k-th receive on d from r
 * (NCCL's per-peer order).  kind 0: ghost rows of one channel plane with the periodic wrap rows
 * (phi, Eq. 32); 1: ghost rows without wrap (w, b, image); 2 / 3: chunk k of nk of the forward /
 * backward spectrum all-to-all of an M/P x N slab.  Writes 5 int64 per op to `ops`
 * (if non-NULL, at most max_ops): send (1) or receive (0), peer rank, buffer (halo: channel 0;
 * a2a: 0 = the row-pass spectrum [H/G][M/P][G], 1 = the column buffer [P][H/(P G)][M/P][G]),
 * offset and count in floats (halo offsets are relative to local row 0, the top ghost rows are
 * negative).  Returns the number of ops, or -1 on bad arguments (P, r, Ml >= 1, gh >= 1, 0 <= k < nk,
 * (N/2) % P == 0 and the chunk dividing the block). */
int sr_sb_slab_schedule(int kind, int P, int r, int Ml, int gh, int N, int k, int nk, long long* ops, int max_ops);
/* Spectrum all-to-all chunks this slab context pipelines with its column solve (1 = unchunked;
 * SRSB_A2A_CHUNKS overrides the default 4 at creation). */
int sr_sb_a2a_chunks(const sr_sb_ctx* ctx);

/* Host logic of the tridiagonal column pass (needs no GPU).  After the row FFT, Eq. (31)-(33)
 * (symbol of Eq. 32 as read in Q10) leave per spectrum column k2 in [0, N/2] the cyclic system
 *   c x_i - a (x_{i-1} + x_{i+1}) = d_i,   a = tau mu,  c = 1 + tau mu (4 - 2 cos(2 pi k2 / N)),
 * solved by two first-order recurrences cut into C chunks of L elements.  Writes the constants the kernels
 * use, exactly as the context tabulates them (fp64):
 *   out[0] = r = 2a / (c + sqrt(c^2 - 4 a^2))     recurrence ratio
 *   out[1] = kappa = 1 / sqrt(c^2 - 4 a^2)        Green's function scale (the kernels fold 2/N into it)
 *   out[2] = rho = r^L                            chunk-to-chunk carry ratio
 *   out[3] = closure factor 1 / (1 - rho^C) if the carry sum runs a full wrap of the column, else 1
 *   out[4] = carry terms mmax in [1, C]: the smallest m with rho^m < 2^-48
 * Returns 0, or -1 on bad arguments (N >= 2, 0 <= k2 <= N/2, L >= 1, C >= 1, tau >= 0, mu > 0). */
int sr_sb_tri_constants(float tau, float mu, int N, int k2, int L, int C, double* out);

/* Algorithm 1 step (1): image f and initial level set phi0 ([batch][M][N]) ->
 * g (Eq. 1), phi = phi0, w = grad phi0 (Q12), b = 0.  Resets k to 0. */
sr_status sr_sb_set_image(sr_sb_ctx* ctx, const float* image, const float* phi0);

/* Enqueue K outer iterations of Algorithm 1 (each: S sweeps of Eq. 37 + Eq. 33,
 * the clamp, Eq. 42/40 and Eq. 23).  K >= 0.  Asynchronous. */
sr_status sr_sb_iterate(sr_sb_ctx* ctx, int K);

/* Copy phi ([batch][M][N]) to phi_out.  Also reports a latched SR_ERR_NONFINITE. */
sr_status sr_sb_get_phi(sr_sb_ctx* ctx, float* phi_out);

/* Copy the full state; any pointer may be NULL to skip it.  w, b: [batch][2][M][N]. */
sr_status sr_sb_get_state(sr_sb_ctx* ctx, float* phi, float* w, float* b, float* g);

/* Overwrite the state (checkpoint resume / teacher forcing).  g may be NULL to keep it. */
sr_status sr_sb_set_state(sr_sb_ctx* ctx, const float* phi, const float* w, const float* b, const float* g);

/* Outer iterations completed since set_image / set_state. */
long long sr_sb_iteration(const sr_sb_ctx* ctx);
/* Set the outer-iteration counter k (checkpoint / resume with sr_sb_set_state). */
sr_status sr_sb_set_iteration(sr_sb_ctx* ctx, long long k);

/* Block the host until the context's stream is idle; returns pending CUDA / non-finite errors. */
sr_status sr_sb_sync(sr_sb_ctx* ctx);

/* Debug / parity entry points (single steps of the hot path, same kernels):
 *  sr_sb_debug_solve: phi_out = Re F^-1(F(F)/symbol) (Eq. 33) for F [batch][M][N];
 *                     uses the context's spectrum scratch, leaves the state untouched.
 *  sr_sb_debug_rhs:   D_out = F - (1 - tau mu Delta_per) psi: the Eq. (37) RHS F in the increment
 *                     form the solve consumes, evaluated on the current state
 *                     (psi = phi); Delta_per is the periodic 5-point Laplacian of Eq. (35).
 *  sr_sb_debug_wb:    one w/b update (Eq. 41/42 or 38/39, 40, 23) on the current state,
 *                     treating the current phi as phi^{k+1}. */
sr_status sr_sb_debug_solve(sr_sb_ctx* ctx, const float* F, float* phi_out);
sr_status sr_sb_debug_rhs(sr_sb_ctx* ctx, float* F_out);
sr_status sr_sb_debug_wb(sr_sb_ctx* ctx);

/* Kernel classes of the hot path, in launch order within a sweep / iteration. */
typedef enum { SR_K_RHS = 0, SR_K_ROWS_R2C = 1, SR_K_COLS_SOLVE = 2, SR_K_ROWS_C2R = 3, SR_K_WB = 4,
               SR_K_AOS_VERT = 5, SR_K_AOS_HORIZ = 6,   /* phi_solver = SR_PHI_AOS replaces classes 1-3 */
               SR_K_RHS_R2C = 7,   /* the fused RHS (Eq. 37) + row R2C cluster kernel: replaces classes 0-1 for
                                      whole-image FFT contexts with 128 <= N <= 1024 */
               SR_K_SOLVE_CLUSTER = 8,   /* small images (M <= 512, 128 <= N <= 512): the whole solve of Eq. (31)-(33) in one
                                            thread-block-cluster kernel, replaces classes 1-3 */
               SR_K_NCLASSES = 9 } sr_kernel_class;

/* Diagnostics: run K outer iterations WITHOUT the CUDA graph, bracketing every launch with CUDA
 * events on the context's work stream, and return per kernel class (sr_kernel_class) the summed
 * device time in ms (ms_out[SR_K_NCLASSES]) and the number of launches (launches_out[SR_K_NCLASSES]).  Synchronizes the
 * host.  Advances the state exactly like sr_sb_iterate(ctx, K). */
sr_status sr_sb_profile(sr_sb_ctx* ctx, int K, float* ms_out, int* launches_out);

/* ---- Monitoring and convergence (whole-image contexts).
 * sr_sb_set_monitor(ctx, 1) makes every outer iteration also accumulate, per image, in double:
 *   [0] E_g = sum g |w| delta(phi)            [1] E_a = sum g (1 - H(phi))
 *   [2] E_r = -sum_x sum_{y in W(x)} G w(x).w(y) h(phi(x)) h(phi(y))
 *   [3] E_pen = (mu/2) sum |w - grad phi - b|^2                     (the terms of Eq. (22) at the
 *       state (phi^{k+1}, w^k, b^k) entering the w-update; total = gamma[0] + alpha[1] + beta[2] + [3])
 *   [4 + 2s], [5 + 2s] = ||phi^{k+1,s+1} - phi^{k+1,s}||^2 and ||phi^{k+1,s}||^2 for sweep s
 * for the LAST iteration enqueued (energies in the threshold w-mode).  sr_sb_get_monitor copies
 * [batch][4 + 2 S] doubles (synchronous).
 * sr_sb_iterate_until runs up to K_max iterations in chunks of `every`, stopping after the first
 * chunk with ||phi^k - phi^{k-every}|| / (||phi^{k-every}|| + 1e-6) <= tol for every image (the
 * relative phi change; Alg. 1's outer test "(13) converges", is unspecified; the inner
 * sweep rule of P:366 is reported by the monitor but is not a fixed-point test under the clamp:
 * the sweeps push phi past +-1 and the clamp resets it).  *k_done = iterations run;
 * sr_sb_last_change returns the last measured relative change. */
sr_status sr_sb_set_monitor(sr_sb_ctx* ctx, int enable);
sr_status sr_sb_get_monitor(sr_sb_ctx* ctx, double* out);
sr_status sr_sb_iterate_until(sr_sb_ctx* ctx, int K_max, double tol, int every, int* k_done);
double sr_sb_last_change(const sr_sb_ctx* ctx);

/* Number of kernel launches one outer iteration enqueues (for bench accounting). */
int sr_sb_launches_per_iteration(const sr_sb_ctx* ctx);

/* Free everything the context owns.  NULL is a no-op. */
void sr_sb_destroy(sr_sb_ctx* ctx);

/* Message of the last error on ctx (ctx-owned, valid until the next call); ctx may be NULL
 * for errors of sr_sb_create. */
const char* sr_sb_last_error(const sr_sb_ctx* ctx);

int sr_sb_abi_version(void);

/* ---- 3-D extension ("The algorithm can also be extended to 3D",
 * Fig. 6 caption P:568; reading Q26 of DESIGN.md).  One volume of D x M x N voxels per context,
 * all powers of two (M, N >= 8, N <= 8192, D <= 1024; thin volumes with D < 16 or M < 32 additionally need
 * D (M + 1) <= 25600: their D x M spectrum planes are solved in shared memory),
 * p->batch = 1, window radius <= 4, FFT phi solver; every other parameter as in 2-D.
 * Every operator gains the depth axis z: grad = forward differences along (i, j, z) with 0 on
 * the last index of each axis (Eq. 35), div its Neumann adjoint (Eq. 36), the window the ball
 * p^2 + q^2 + r^2 <= R^2 (window_shape 0) or the cube (1), the solve's symbol
 * 1 + tau mu (6 - 2 cos z1 - 2 cos z2 - 2 cos z3) (Eq. 32), shrink / projection on 3-vectors,
 * the edge indicator with a 3-D Gaussian.
 * Layouts (dense, C order, host or device pointers): volume / phi / g [D][M][N] fp32; w, b
 * [3][D][M][N] with components (along i, along j, along z).  Ownership and error behaviour as
 * in 2-D (the context owns its device buffers; errors return a negative status and set
 * sr_sb3_last_error). */
typedef struct sr_sb3_ctx sr_sb3_ctx;
sr_status sr_sb3_create(const sr_sb_params* p, int D, int device, void* stream, sr_sb3_ctx** out);
/* Eq. (1) in 3-D and Alg. 1 (1): g from the volume, phi = phi0, w = grad phi0, b = 0. */
sr_status sr_sb3_set_image(sr_sb3_ctx* ctx, const float* volume, const float* phi0);
/* K outer iterations of Algorithm 1 in 3-D (S FFT sweeps, clamp, w/b update). */
sr_status sr_sb3_iterate(sr_sb3_ctx* ctx, int K);
sr_status sr_sb3_get_phi(sr_sb3_ctx* ctx, float* phi_out);
sr_status sr_sb3_get_state(sr_sb3_ctx* ctx, float* phi, float* w, float* b, float* g);
sr_status sr_sb3_set_state(sr_sb3_ctx* ctx, const float* phi, const float* w, const float* b, const float* g);
/* Single steps on the same kernels: the 3-D solve of F (Eq. 33, no clamp); the RHS in increment
 * form D = F - (1 - tau mu Delta_per) psi at the current state. */
sr_status sr_sb3_debug_solve(sr_sb3_ctx* ctx, const float* F, float* phi_out);
sr_status sr_sb3_debug_rhs(sr_sb3_ctx* ctx, float* D_out);
/* As sr_sb_profile (classes: rhs, rows_r2c, cols_solve = the plane solve, rows_c2r, wb). */
sr_status sr_sb3_profile(sr_sb3_ctx* ctx, int K, float* ms_out, int* launches_out);
/* Synchronize; SR_ERR_NONFINITE if the w/b guard tripped. */
sr_status sr_sb3_sync(sr_sb3_ctx* ctx);
void sr_sb3_destroy(sr_sb3_ctx* ctx);
const char* sr_sb3_last_error(const sr_sb3_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SRSB_H */
