/*
 * sr_oracle.c -- plain, slow, float64 CPU oracle for the Split Bregman
 * Self-repelling Snake iteration (Pan et al., arXiv 2003.12693).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path (paper_2003_12693_b200/csrc); neither includes the other.
 *
 * Citations: "P:n" is line n of PAPER.md (the LaTeX source); equation numbers
 * are LaTeX's.  Readings of the paper where it is silent or garbled are the
 * "Q" items of DESIGN.md §2 (= SURVEY.md §8(c)).
 *
 * Everything is written in the paper's order and notation, without blocking,
 * fusion or reordering:
 *   - regularizers: Eq. (5), (6), (29), (11), (28);
 *   - stencils: Eq. (35), (36) as the Neumann-adjoint pair (Q6);
 *   - edge indicator: Eq. (1) with a normalized Gaussian of radius ceil(3 sigma) (Q16);
 *   - FFT: recursive radix-2 complex DFT, unnormalized forward, 1/n inverse;
 *   - phi solve: Eq. (31)-(33), full complex 2-D FFT, divide by the symbol of Eq. (32) (Q10);
 *     or the AOS variant of P:427 (Thomas solves of the Neumann 1-D operators, NEXT-4);
 *   - window sum: the direct double loop of P:368 (disc or square window, Q2, Q5);
 *   - RHS: Eq. (37) with phi^{k+1,s} in every term (Q8);
 *   - w/b update: Eq. (41), (42), projection Eq. (40) as BALL/SPHERE/NONE (Q1), Eq. (23);
 *   - fixed-point w update: Eq. (38)-(40) (NEXT-2);
 *   - Algorithm 1 with fixed S sweeps (Q7) and the north-star clamp (Q9);
 *   - connected-component labelling by flood fill (validation);
 *   - the 3-D extension (orc3_*, NEXT-3, reading Q26): the same steps with the depth axis.
 *
 * Parity pins: every function is pinned by tests/test_oracle_*.py against
 * closed forms, brute force, numpy/scipy library routines or invariants
 * (DESIGN.md §4).  Round 1 claimed this while two branches were only pinned
 * where they vanish: the fixed-point w update (Eq. 38) with beta != 0 and
 * several passes, and the depth axis / third channel of the 3-D functions.
 * Those pins were added in round 2 (test_oracle_wb.py::test_fixed_point_
 * passes_*, test_oracle_3d.py::test_edge3_matches_scipy_*, ::test_axis_
 * permutation_*), each checked to fail on an injected bug.  What has no
 * external pin is the long-trajectory behaviour on C2-C5:
 * the paper prints no values for those images.
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 * OpenMP parallelises only independent per-pixel / per-row loops, so results
 * are bitwise deterministic regardless of the thread count.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct {
    double gamma, alpha, beta, mu;   /* Eq. (7), (22) weights */
    double epsilon, l;               /* Eq. (5)-(6) half-width; Eq. (11) band offset */
    double d;                        /* Eq. (10)/(38) Gaussian scale */
    int window;                      /* summation radius R of P:368 (BASELINE's "l") */
    int window_shape;                /* 0 = disc p^2+q^2 <= R^2, 1 = square |p|,|q| <= R */
    double tau;                      /* Eq. (30)/(37) time step */
    int S;                           /* phi sweeps per outer iteration (Q7) */
    double phi_clip;                 /* >0: clamp phi^{k+1} to [-phi_clip, phi_clip] (Q9) */
    int w_proj;                      /* 0 BALL, 1 SPHERE, 2 NONE (Q1) */
    int w_mode;                      /* 0 threshold Eq. (41)-(42); 1 fixed point Eq. (38)-(39) */
    int w_iters;                     /* fixed-point sweeps r = 0..w_iters-1 */
    int phi_solver;                  /* 0 FFT, Eq. (31)-(33); 1 AOS with constant coefficients (NEXT-4) */
} orc_params;

#define IDX(i, j) ((size_t)(i) * (size_t)N + (size_t)(j))

/* ------------------------------------------------------------------ */
/* Regularizers                                                        */
/* ------------------------------------------------------------------ */

/* Eq. (5) */
double orc_H(double phi, double eps)
{
    if (phi > eps) return 1.0;
    if (phi < -eps) return 0.0;
    return 0.5 * (1.0 + phi / eps + sin(M_PI * phi / eps) / M_PI);
}

/* Eq. (6) */
double orc_delta(double phi, double eps)
{
    if (fabs(phi) > eps) return 0.0;
    return (1.0 + cos(M_PI * phi / eps)) / (2.0 * eps);
}

/* Eq. (29) */
double orc_delta_prime(double phi, double eps)
{
    if (fabs(phi) > eps) return 0.0;
    return -(M_PI / (2.0 * eps * eps)) * sin(M_PI * phi / eps);
}

/* Eq. (11): h = H(phi + l) (1 - H(phi - l)) */
double orc_h(double phi, double eps, double l)
{
    return orc_H(phi + l, eps) * (1.0 - orc_H(phi - l, eps));
}

/* Eq. (28): h' = delta(phi + l)(1 - H(phi - l)) - H(phi + l) delta(phi - l) */
double orc_h_prime(double phi, double eps, double l)
{
    return orc_delta(phi + l, eps) * (1.0 - orc_H(phi - l, eps))
         - orc_H(phi + l, eps) * orc_delta(phi - l, eps);
}

/* ------------------------------------------------------------------ */
/* Stencils, Eq. (35)-(36) as the exact adjoint pair (reading Q6)      */
/* ------------------------------------------------------------------ */

/* Eq. (35): forward differences; zero on the last row / last column. */
void orc_grad(int M, int N, const double *phi, double *g1, double *g2)
{
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            g1[IDX(i, j)] = (i < M - 1) ? phi[IDX(i + 1, j)] - phi[IDX(i, j)] : 0.0;
            g2[IDX(i, j)] = (j < N - 1) ? phi[IDX(i, j + 1)] - phi[IDX(i, j)] : 0.0;
        }
}

/* Eq. (36): backward differences; u1 is dropped on the last row and u2 on
 * the last column (where grad is defined as 0), out-of-range terms are 0. */
void orc_div(int M, int N, const double *u1, const double *u2, double *out)
{
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double s = 0.0;
            if (i < M - 1) s += u1[IDX(i, j)];
            if (i > 0) s -= u1[IDX(i - 1, j)];
            if (j < N - 1) s += u2[IDX(i, j)];
            if (j > 0) s -= u2[IDX(i, j - 1)];
            out[IDX(i, j)] = s;
        }
}

/* ------------------------------------------------------------------ */
/* Edge indicator, Eq. (1)                                    */
/* ------------------------------------------------------------------ */

/* g = 1 / (1 + rho |grad(G_sigma * f)|^s); G_sigma: normalized Gaussian
 * exp(-t^2/(2 sigma^2)), t = -r..r, r = ceil(3 sigma), separable rows then
 * columns with replicate padding (Q16); grad by central differences with
 * replicate padding. */
void orc_edge(int M, int N, const double *f, double sigma, double rho, int s, double *g)
{
    int r = (int)ceil(3.0 * sigma);
    double *k = (double *)malloc(sizeof(double) * (2 * r + 1));
    double ks = 0.0;
    for (int t = -r; t <= r; t++) { k[t + r] = exp(-(double)(t * t) / (2.0 * sigma * sigma)); ks += k[t + r]; }
    for (int t = 0; t <= 2 * r; t++) k[t] /= ks;
    double *tmp = (double *)malloc(sizeof(double) * (size_t)M * N);
    double *fs = (double *)malloc(sizeof(double) * (size_t)M * N);
    /* rows: convolve along j */
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double a = 0.0;
            for (int t = -r; t <= r; t++) {
                int jj = j + t; if (jj < 0) jj = 0; if (jj > N - 1) jj = N - 1;
                a += k[t + r] * f[IDX(i, jj)];
            }
            tmp[IDX(i, j)] = a;
        }
    /* columns: convolve along i */
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double a = 0.0;
            for (int t = -r; t <= r; t++) {
                int ii = i + t; if (ii < 0) ii = 0; if (ii > M - 1) ii = M - 1;
                a += k[t + r] * tmp[IDX(ii, j)];
            }
            fs[IDX(i, j)] = a;
        }
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            int ip = i + 1 < M ? i + 1 : M - 1, im = i > 0 ? i - 1 : 0;
            int jp = j + 1 < N ? j + 1 : N - 1, jm = j > 0 ? j - 1 : 0;
            double gx = (fs[IDX(ip, j)] - fs[IDX(im, j)]) / 2.0;
            double gy = (fs[IDX(i, jp)] - fs[IDX(i, jm)]) / 2.0;
            double m2 = gx * gx + gy * gy;
            double mag = (s == 2) ? m2 : sqrt(m2);
            g[IDX(i, j)] = 1.0 / (1.0 + rho * mag);
        }
    free(k); free(tmp); free(fs);
}

/* ------------------------------------------------------------------ */
/* FFT: recursive radix-2, X[k] = sum_n x[n] exp(-2 pi i k n / n)      */
/* ------------------------------------------------------------------ */

static void fft_rec(int n, double *re, double *im, int stride, double *ore, double *oim, int sign)
{
    if (n == 1) { ore[0] = re[0]; oim[0] = im[0]; return; }
    int h = n / 2;
    /* even samples -> first half of the output, odd samples -> second half */
    fft_rec(h, re, im, 2 * stride, ore, oim, sign);
    fft_rec(h, re + stride, im + stride, 2 * stride, ore + h, oim + h, sign);
    for (int k = 0; k < h; k++) {
        double a = sign * 2.0 * M_PI * (double)k / (double)n;
        double c = cos(a), s = sin(a);
        double er = ore[k], ei = oim[k];
        double orr = ore[k + h], oi = oim[k + h];
        double tr = c * orr - s * oi, ti = c * oi + s * orr;
        ore[k] = er + tr;  oim[k] = ei + ti;
        ore[k + h] = er - tr;  oim[k + h] = ei - ti;
    }
}

/* In place; n a power of two; inverse = 1 gives (1/n) sum x[k] exp(+2 pi i k n / n). */
int orc_fft(int n, double *re, double *im, int inverse)
{
    if (n < 1 || (n & (n - 1))) return -1;
    double *xr = (double *)malloc(sizeof(double) * n), *xi = (double *)malloc(sizeof(double) * n);
    memcpy(xr, re, sizeof(double) * n); memcpy(xi, im, sizeof(double) * n);
    fft_rec(n, xr, xi, 1, re, im, inverse ? +1 : -1);
    if (inverse) for (int k = 0; k < n; k++) { re[k] /= n; im[k] /= n; }
    free(xr); free(xi);
    return 0;
}

/* 2-D FFT of an M x N complex array: rows, then columns. */
int orc_fft2(int M, int N, double *re, double *im, int inverse)
{
    if (M < 1 || N < 1 || (M & (M - 1)) || (N & (N - 1))) return -1;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++) orc_fft(N, re + IDX(i, 0), im + IDX(i, 0), inverse);
    #pragma omp parallel
    {
        double *cr = (double *)malloc(sizeof(double) * M), *ci = (double *)malloc(sizeof(double) * M);
        #pragma omp for schedule(static)
        for (int j = 0; j < N; j++) {
            for (int i = 0; i < M; i++) { cr[i] = re[IDX(i, j)]; ci[i] = im[IDX(i, j)]; }
            orc_fft(M, cr, ci, inverse);
            for (int i = 0; i < M; i++) { re[IDX(i, j)] = cr[i]; im[IDX(i, j)] = ci[i]; }
        }
        free(cr); free(ci);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* phi sub-problem, Eq. (31)-(33)                           */
/* ------------------------------------------------------------------ */

/* Symbol of (1 - tau mu Delta) under the periodic DFT, Eq. (32) with the
 * garbled bracket read as 1 - tau mu (2 cos z1 + 2 cos z2 - 4) (Q10),
 * z1 = 2 pi k1 / M, z2 = 2 pi k2 / N, 0-based k. */
double orc_symbol(int M, int N, double tau, double mu, int k1, int k2)
{
    double z1 = 2.0 * M_PI * (double)k1 / (double)M;
    double z2 = 2.0 * M_PI * (double)k2 / (double)N;
    return 1.0 - tau * mu * (2.0 * cos(z1) + 2.0 * cos(z2) - 4.0);
}

/* phi = Re F^{-1}( F(F) / symbol ), Eq. (33).  Returns 1 if the discarded
 * imaginary part exceeds 1e-12 max|F| (Q11), else 0. */
int orc_solve(int M, int N, double tau, double mu, const double *F, double *phi)
{
    size_t n = (size_t)M * N;
    double *re = (double *)malloc(sizeof(double) * n), *im = (double *)calloc(n, sizeof(double));
    memcpy(re, F, sizeof(double) * n);
    orc_fft2(M, N, re, im, 0);
    for (int k1 = 0; k1 < M; k1++)
        for (int k2 = 0; k2 < N; k2++) {
            double sg = orc_symbol(M, N, tau, mu, k1, k2);
            re[IDX(k1, k2)] /= sg;
            im[IDX(k1, k2)] /= sg;
        }
    orc_fft2(M, N, re, im, 1);
    double fmax = 0.0, imax = 0.0;
    for (size_t q = 0; q < n; q++) {
        if (fabs(F[q]) > fmax) fmax = fabs(F[q]);
        if (fabs(im[q]) > imax) imax = fabs(im[q]);
        phi[q] = re[q];
    }
    free(re); free(im);
    return imax > 1e-12 * (fmax > 0 ? fmax : 1.0) ? 1 : 0;
}

/* ------------------------------------------------------------------ */
/* phi sub-problem by AOS (the AOS splitting of Eq. (19)-(20)) */
/* ------------------------------------------------------------------ */

/* Solve (I - c A) x = f for one line of n values, A the 1-D second difference with Neumann
 * (reflecting) ends: (A x)_0 = x_1 - x_0, (A x)_{n-1} = x_{n-2} - x_{n-1}.  Thomas algorithm
 * (LR decomposition, forward and backward substitution). */
void orc_thomas_neumann(int n, double c, const double *f, double *x)
{
    if (n == 1) { x[0] = f[0]; return; }
    double *cp = malloc(sizeof(double) * n), *y = malloc(sizeof(double) * n);
    const double a = -c;                       /* sub- and super-diagonal */
    double d = 1.0 + c;                        /* first row: 1 - c (x_1 - x_0) -> diag 1 + c */
    cp[0] = a / d;
    y[0] = f[0] / d;
    for (int i = 1; i < n; i++) {
        d = (i == n - 1 ? 1.0 + c : 1.0 + 2.0 * c) - a * cp[i - 1];
        cp[i] = a / d;
        y[i] = (f[i] - a * y[i - 1]) / d;
    }
    x[n - 1] = y[n - 1];
    for (int i = n - 2; i >= 0; i--) x[i] = y[i] - cp[i] * x[i + 1];
    free(cp); free(y);
}

/* AOS: phi = 1/2 [ (I - 2 tau mu A_1)^{-1} + (I - 2 tau mu A_2)^{-1} ] F, A_1 along columns
 * (index i), A_2 along rows (index j), m = 2 directions (the splitting of Eq. (19)-(20) with the
 * constant coefficients of the phi sub-problem). */
void orc_solve_aos(int M, int N, double tau, double mu, const double *F, double *phi)
{
    const double c = 2.0 * tau * mu;
    double *x1 = malloc(sizeof(double) * (size_t)M * N);
    #pragma omp parallel
    {
        double *col = malloc(sizeof(double) * M), *sol = malloc(sizeof(double) * M);
        #pragma omp for schedule(static)
        for (int j = 0; j < N; j++) {
            for (int i = 0; i < M; i++) col[i] = F[IDX(i, j)];
            orc_thomas_neumann(M, c, col, sol);
            for (int i = 0; i < M; i++) x1[IDX(i, j)] = sol[i];
        }
        free(col); free(sol);
    }
    #pragma omp parallel
    {
        double *sol = malloc(sizeof(double) * N);
        #pragma omp for schedule(static)
        for (int i = 0; i < M; i++) {
            orc_thomas_neumann(N, c, F + IDX(i, 0), sol);
            for (int j = 0; j < N; j++) phi[IDX(i, j)] = 0.5 * (x1[IDX(i, j)] + sol[j]);
        }
        free(sol);
    }
    free(x1);
}

/* ------------------------------------------------------------------ */
/* Non-local window sum, P:368-369 (and Eq. 38)                        */
/* ------------------------------------------------------------------ */

/* v(i,j) = sum_{(p,q) in W} exp(-(p^2+q^2)/d^2) u(i+p, j+q); terms outside
 * the image are 0 (Q5).  W: disc p^2+q^2 <= R^2 (shape 0) or square (1). */
void orc_window_sum(int M, int N, int R, double d, int shape,
                    const double *u1, const double *u2, double *v1, double *v2)
{
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double a1 = 0.0, a2 = 0.0;
            for (int p = -R; p <= R; p++)
                for (int q = -R; q <= R; q++) {
                    if (shape == 0 && p * p + q * q > R * R) continue;
                    int ii = i + p, jj = j + q;
                    if (ii < 0 || ii >= M || jj < 0 || jj >= N) continue;
                    double G = exp(-(double)(p * p + q * q) / (d * d));
                    a1 += G * u1[IDX(ii, jj)];
                    a2 += G * u2[IDX(ii, jj)];
                }
            v1[IDX(i, j)] = a1;
            v2[IDX(i, j)] = a2;
        }
}

/* ------------------------------------------------------------------ */
/* RHS of the phi sweep, Eq. (37)                           */
/* ------------------------------------------------------------------ */

/* F = psi + tau [ -gamma g |w| delta'(psi) + alpha g delta(psi)
 *                 + 2 beta h'(psi) w . v + mu div(b - w) ],
 * v = window_sum(h(psi) w) (with phi^{k+1,s} = psi, Q8). */
void orc_rhs(int M, int N, const orc_params *P, const double *psi,
             const double *w1, const double *w2, const double *b1, const double *b2,
             const double *g, double *F)
{
    size_t n = (size_t)M * N;
    double *u1 = malloc(sizeof(double) * n), *u2 = malloc(sizeof(double) * n);
    double *v1 = malloc(sizeof(double) * n), *v2 = malloc(sizeof(double) * n);
    double *c1 = malloc(sizeof(double) * n), *c2 = malloc(sizeof(double) * n);
    double *dv = malloc(sizeof(double) * n);
    for (size_t q = 0; q < n; q++) {
        double hq = orc_h(psi[q], P->epsilon, P->l);
        u1[q] = hq * w1[q];
        u2[q] = hq * w2[q];
        c1[q] = b1[q] - w1[q];
        c2[q] = b2[q] - w2[q];
    }
    orc_window_sum(M, N, P->window, P->d, P->window_shape, u1, u2, v1, v2);
    orc_div(M, N, c1, c2, dv);
    #pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; q++) {
        double wn = sqrt(w1[q] * w1[q] + w2[q] * w2[q]);
        double t = -P->gamma * g[q] * wn * orc_delta_prime(psi[q], P->epsilon)
                 + P->alpha * g[q] * orc_delta(psi[q], P->epsilon)
                 + 2.0 * P->beta * orc_h_prime(psi[q], P->epsilon, P->l) * (w1[q] * v1[q] + w2[q] * v2[q])
                 + P->mu * dv[q];
        F[q] = psi[q] + P->tau * t;
    }
    free(u1); free(u2); free(v1); free(v2); free(c1); free(c2); free(dv);
}

/* ------------------------------------------------------------------ */
/* w sub-problem                                                       */
/* ------------------------------------------------------------------ */

/* Generalized soft threshold, Eq. (42), with 0 * 0/|0| = 0. */
void orc_shrink(double B1, double B2, double t, double *o1, double *o2)
{
    double nb = sqrt(B1 * B1 + B2 * B2);
    if (nb > 0.0) {
        double m = nb - t; if (m < 0.0) m = 0.0;
        *o1 = m * B1 / nb;
        *o2 = m * B2 / nb;
    } else {
        *o1 = 0.0; *o2 = 0.0;
    }
}

/* Projection, Eq. (40), "used afterwards" P:400; modes per Q1. */
void orc_project(int mode, double a1, double a2, double *o1, double *o2)
{
    double n = sqrt(a1 * a1 + a2 * a2);
    if (mode == 0) {                       /* BALL: w / max(1, |w|) */
        double s = n > 1.0 ? n : 1.0;
        *o1 = a1 / s; *o2 = a2 / s;
    } else if (mode == 1) {                /* SPHERE: w / |w| where |w| > 1e-4 */
        if (n > 1e-4) { *o1 = a1 / n; *o2 = a2 / n; } else { *o1 = a1; *o2 = a2; }
    } else {                               /* NONE */
        *o1 = a1; *o2 = a2;
    }
}

/* w^{k+1} by Eq. (41)-(42) (w_mode 0) or the fixed point Eq. (38)-(39)
 * (w_mode 1), projected (Eq. 40), then b^{k+1} = b^k + grad phi^{k+1} - w^{k+1}
 * (Eq. 23).  phi is phi^{k+1}; w, b hold w^k, b^k on entry. */
void orc_wb(int M, int N, const orc_params *P, const double *phi,
            double *w1, double *w2, double *b1, double *b2, const double *g)
{
    size_t n = (size_t)M * N;
    double *gp1 = malloc(sizeof(double) * n), *gp2 = malloc(sizeof(double) * n);
    double *u1 = malloc(sizeof(double) * n), *u2 = malloc(sizeof(double) * n);
    double *v1 = malloc(sizeof(double) * n), *v2 = malloc(sizeof(double) * n);
    double *hh = malloc(sizeof(double) * n);
    double *n1 = malloc(sizeof(double) * n), *n2 = malloc(sizeof(double) * n);
    orc_grad(M, N, phi, gp1, gp2);
    for (size_t q = 0; q < n; q++) hh[q] = orc_h(phi[q], P->epsilon, P->l);
    if (P->w_mode == 0) {
        /* Eq. (41): B = grad phi^{k+1} + b^k + (2 beta/mu) h(phi^{k+1}) sum G w^k h(phi^{k+1}) */
        for (size_t q = 0; q < n; q++) { u1[q] = hh[q] * w1[q]; u2[q] = hh[q] * w2[q]; }
        orc_window_sum(M, N, P->window, P->d, P->window_shape, u1, u2, v1, v2);
        for (size_t q = 0; q < n; q++) {
            double B1 = gp1[q] + b1[q] + (2.0 * P->beta / P->mu) * hh[q] * v1[q];
            double B2 = gp2[q] + b2[q] + (2.0 * P->beta / P->mu) * hh[q] * v2[q];
            double t = (P->gamma / P->mu) * g[q] * orc_delta(phi[q], P->epsilon);
            double s1, s2;
            orc_shrink(B1, B2, t, &s1, &s2);
            orc_project(P->w_proj, s1, s2, &n1[q], &n2[q]);
        }
    } else {
        /* Eq. (38)-(39): w^{k+1,0} = w^k; w~^{r+1} = (mu grad phi + mu b + 2 beta h v^r)/(gamma g delta + mu) */
        memcpy(n1, w1, sizeof(double) * n); memcpy(n2, w2, sizeof(double) * n);
        for (int r = 0; r < P->w_iters; r++) {
            for (size_t q = 0; q < n; q++) { u1[q] = hh[q] * n1[q]; u2[q] = hh[q] * n2[q]; }
            orc_window_sum(M, N, P->window, P->d, P->window_shape, u1, u2, v1, v2);
            for (size_t q = 0; q < n; q++) {
                double den = P->gamma * g[q] * orc_delta(phi[q], P->epsilon) + P->mu;
                double a1 = (P->mu * gp1[q] + P->mu * b1[q] + 2.0 * P->beta * hh[q] * v1[q]) / den;
                double a2 = (P->mu * gp2[q] + P->mu * b2[q] + 2.0 * P->beta * hh[q] * v2[q]) / den;
                orc_project(P->w_proj, a1, a2, &n1[q], &n2[q]);
            }
        }
    }
    for (size_t q = 0; q < n; q++) {
        b1[q] = b1[q] + gp1[q] - n1[q];
        b2[q] = b2[q] + gp2[q] - n2[q];
        w1[q] = n1[q];
        w2[q] = n2[q];
    }
    free(gp1); free(gp2); free(u1); free(u2); free(v1); free(v2); free(hh); free(n1); free(n2);
}

/* ------------------------------------------------------------------ */
/* Energy of the split problem, Eq. (22) (NEXT-1 monitoring)           */
/* ------------------------------------------------------------------ */

/* Terms of E(phi, w) in Eq. (22) at the state (phi, w, b), discretized on the pixel grid:
 *   out[0] = E_g   = sum_x g |w| delta(phi)                         (first line, / gamma)
 *   out[1] = E_a   = sum_x g (1 - H(phi))                            (first line, / alpha)
 *   out[2] = E_r   = - sum_x sum_{y in W(x)} G(x-y) w(x).w(y) h(phi(x)) h(phi(y))   (second line, / beta)
 *   out[3] = E_pen = (mu/2) sum_x |w - grad phi - b|^2               (third line)
 * The library reports them at the state entering the w-update: (phi^{k+1}, w^k, b^k). */
void orc_energy(int M, int N, const orc_params *P, const double *phi, const double *w1, const double *w2,
                const double *b1, const double *b2, const double *g, double *out)
{
    size_t n = (size_t)M * N;
    double *u1 = malloc(sizeof(double) * n), *u2 = malloc(sizeof(double) * n);
    double *v1 = malloc(sizeof(double) * n), *v2 = malloc(sizeof(double) * n);
    double *gp1 = malloc(sizeof(double) * n), *gp2 = malloc(sizeof(double) * n);
    for (size_t q = 0; q < n; q++) {
        double hq = orc_h(phi[q], P->epsilon, P->l);
        u1[q] = hq * w1[q];
        u2[q] = hq * w2[q];
    }
    orc_window_sum(M, N, P->window, P->d, P->window_shape, u1, u2, v1, v2);
    orc_grad(M, N, phi, gp1, gp2);
    double eg = 0.0, ea = 0.0, er = 0.0, ep = 0.0;
    for (size_t q = 0; q < n; q++) {
        double wn = sqrt(w1[q] * w1[q] + w2[q] * w2[q]);
        eg += g[q] * wn * orc_delta(phi[q], P->epsilon);
        ea += g[q] * (1.0 - orc_H(phi[q], P->epsilon));
        er -= u1[q] * v1[q] + u2[q] * v2[q];     /* h(x) w(x) . sum_y G w(y) h(y) */
        double r1 = w1[q] - gp1[q] - b1[q], r2 = w2[q] - gp2[q] - b2[q];
        ep += 0.5 * P->mu * (r1 * r1 + r2 * r2);
    }
    out[0] = eg; out[1] = ea; out[2] = er; out[3] = ep;
    free(u1); free(u2); free(v1); free(v2); free(gp1); free(gp2);
}

/* ------------------------------------------------------------------ */
/* Algorithm 1                                              */
/* ------------------------------------------------------------------ */

/* Initialization (1): phi = phi0, w^0 = grad phi^0 (Q12), b^0 = 0. */
void orc_init(int M, int N, const double *phi0, double *phi, double *w1, double *w2, double *b1, double *b2)
{
    size_t n = (size_t)M * N;
    memcpy(phi, phi0, sizeof(double) * n);
    orc_grad(M, N, phi0, w1, w2);
    memset(b1, 0, sizeof(double) * n);
    memset(b2, 0, sizeof(double) * n);
}

/* One sweep: psi <- solve(rhs(psi)).  Returns the solve's imaginary-part flag. */
int orc_sweep(int M, int N, const orc_params *P, double *psi, const double *w1, const double *w2,
              const double *b1, const double *b2, const double *g)
{
    size_t n = (size_t)M * N;
    double *F = malloc(sizeof(double) * n);
    orc_rhs(M, N, P, psi, w1, w2, b1, b2, g, F);
    int bad = 0;
    if (P->phi_solver == 1) orc_solve_aos(M, N, P->tau, P->mu, F, psi);
    else bad = orc_solve(M, N, P->tau, P->mu, F, psi);
    free(F);
    return bad;
}

/* K outer iterations (2) of Algorithm 1 with S sweeps each (Q7), the clamp
 * of phi^{k+1} after the last sweep (Q9), then w (Eq. 42 / 39, 40) and b (Eq. 23).
 * Returns the number of solves whose imaginary-part check failed. */
int orc_iterate(int M, int N, const orc_params *P, double *phi, double *w1, double *w2,
                double *b1, double *b2, const double *g, int K)
{
    int bad = 0;
    size_t n = (size_t)M * N;
    for (int k = 0; k < K; k++) {
        for (int s = 0; s < P->S; s++) bad += orc_sweep(M, N, P, phi, w1, w2, b1, b2, g);
        if (P->phi_clip > 0.0)
            for (size_t q = 0; q < n; q++) {
                if (phi[q] > P->phi_clip) phi[q] = P->phi_clip;
                if (phi[q] < -P->phi_clip) phi[q] = -P->phi_clip;
            }
        orc_wb(M, N, P, phi, w1, w2, b1, b2, g);
    }
    return bad;
}

/* ------------------------------------------------------------------ */
/* Validation: connected components of a mask by flood fill            */
/* ------------------------------------------------------------------ */

/* labels[q] = 0 for background, 1..count for components; conn = 4 or 8. */
int orc_label(int M, int N, const unsigned char *mask, int conn, int *labels)
{
    size_t n = (size_t)M * N;
    int *stack = (int *)malloc(sizeof(int) * n);
    int count = 0;
    for (size_t q = 0; q < n; q++) labels[q] = 0;
    for (size_t q0 = 0; q0 < n; q0++) {
        if (!mask[q0] || labels[q0]) continue;
        count++;
        size_t top = 0;
        stack[top++] = (int)q0;
        labels[q0] = count;
        while (top) {
            int q = stack[--top];
            int i = q / N, j = q % N;
            for (int di = -1; di <= 1; di++)
                for (int dj = -1; dj <= 1; dj++) {
                    if (!di && !dj) continue;
                    if (conn == 4 && di && dj) continue;
                    int ii = i + di, jj = j + dj;
                    if (ii < 0 || ii >= M || jj < 0 || jj >= N) continue;
                    size_t r = IDX(ii, jj);
                    if (mask[r] && !labels[r]) { labels[r] = count; stack[top++] = (int)r; }
                }
        }
    }
    free(stack);
    return count;
}

/* ================================================================== */
/* 3-D extension ("The algorithm can also be extended to 3D";   */
/* Fig. 6 caption P:568).  Reading Q26: every     */
/* operator gains the depth axis z (D planes of M x N):                 */
/*   grad = (d_i, d_j, d_z) forward differences (Eq. 35 per axis),      */
/*   div its Neumann adjoint (Eq. 36 per axis), the window a ball        */
/*   p^2+q^2+r^2 <= R^2 (or a cube), the solve's symbol                  */
/*   1 + tau mu (6 - 2cos z1 - 2cos z2 - 2cos z3) (Eq. 32 in 3-D),       */
/*   shrink / projection on 3-vectors, the edge indicator with a 3-D     */
/*   Gaussian.  Component order (1, 2, 3) = (rows i, columns j, depth z) */
/*   so that a D = 1 volume reduces to the 2-D functions above exactly.  */
/* ================================================================== */

#define IDX3(z, i, j) (((size_t)(z) * (size_t)M + (size_t)(i)) * (size_t)N + (size_t)(j))

void orc3_grad(int D, int M, int N, const double *phi, double *g1, double *g2, double *g3)
{
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                size_t q = IDX3(z, i, j);
                g1[q] = (i < M - 1) ? phi[IDX3(z, i + 1, j)] - phi[q] : 0.0;
                g2[q] = (j < N - 1) ? phi[IDX3(z, i, j + 1)] - phi[q] : 0.0;
                g3[q] = (z < D - 1) ? phi[IDX3(z + 1, i, j)] - phi[q] : 0.0;
            }
}

void orc3_div(int D, int M, int N, const double *u1, const double *u2, const double *u3, double *out)
{
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double s = 0.0;
                if (i < M - 1) s += u1[IDX3(z, i, j)];
                if (i > 0) s -= u1[IDX3(z, i - 1, j)];
                if (j < N - 1) s += u2[IDX3(z, i, j)];
                if (j > 0) s -= u2[IDX3(z, i, j - 1)];
                if (z < D - 1) s += u3[IDX3(z, i, j)];
                if (z > 0) s -= u3[IDX3(z - 1, i, j)];
                out[IDX3(z, i, j)] = s;
            }
}

/* Eq. (1) in 3-D: separable normalized Gaussian along j, i, z (replicate padding), central
 * differences (replicate padding) along the three axes. */
void orc3_edge(int D, int M, int N, const double *f, double sigma, double rho, int s, double *g)
{
    int r = (int)ceil(3.0 * sigma);
    double *k = (double *)malloc(sizeof(double) * (2 * r + 1));
    double ks = 0.0;
    for (int t = -r; t <= r; t++) { k[t + r] = exp(-(double)(t * t) / (2.0 * sigma * sigma)); ks += k[t + r]; }
    for (int t = 0; t <= 2 * r; t++) k[t] /= ks;
    size_t n = (size_t)D * M * N;
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n);
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double acc = 0.0;
                for (int t = -r; t <= r; t++) {
                    int jj = j + t; if (jj < 0) jj = 0; if (jj > N - 1) jj = N - 1;
                    acc += k[t + r] * f[IDX3(z, i, jj)];
                }
                a[IDX3(z, i, j)] = acc;
            }
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double acc = 0.0;
                for (int t = -r; t <= r; t++) {
                    int ii = i + t; if (ii < 0) ii = 0; if (ii > M - 1) ii = M - 1;
                    acc += k[t + r] * a[IDX3(z, ii, j)];
                }
                b[IDX3(z, i, j)] = acc;
            }
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double acc = 0.0;
                for (int t = -r; t <= r; t++) {
                    int zz = z + t; if (zz < 0) zz = 0; if (zz > D - 1) zz = D - 1;
                    acc += k[t + r] * b[IDX3(zz, i, j)];
                }
                a[IDX3(z, i, j)] = acc;   /* a = G_sigma * f */
            }
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                int ip = i + 1 < M ? i + 1 : M - 1, im = i > 0 ? i - 1 : 0;
                int jp = j + 1 < N ? j + 1 : N - 1, jm = j > 0 ? j - 1 : 0;
                int zp = z + 1 < D ? z + 1 : D - 1, zm = z > 0 ? z - 1 : 0;
                double gx = (a[IDX3(z, ip, j)] - a[IDX3(z, im, j)]) / 2.0;
                double gy = (a[IDX3(z, i, jp)] - a[IDX3(z, i, jm)]) / 2.0;
                double gz = (a[IDX3(zp, i, j)] - a[IDX3(zm, i, j)]) / 2.0;
                double m2 = gx * gx + gy * gy + gz * gz;
                double mag = (s == 2) ? m2 : sqrt(m2);
                g[IDX3(z, i, j)] = 1.0 / (1.0 + rho * mag);
            }
    free(k); free(a); free(b);
}

/* 3-D FFT of a D x M x N complex array: rows (j), columns (i), depth (z). */
int orc3_fft3(int D, int M, int N, double *re, double *im, int inverse)
{
    if (D < 1 || (D & (D - 1))) return -1;
    for (int z = 0; z < D; z++)
        if (orc_fft2(M, N, re + IDX3(z, 0, 0), im + IDX3(z, 0, 0), inverse)) return -1;
    #pragma omp parallel
    {
        double *cr = malloc(sizeof(double) * D), *ci = malloc(sizeof(double) * D);
        #pragma omp for schedule(static)
        for (int q = 0; q < M * N; q++) {
            for (int z = 0; z < D; z++) { cr[z] = re[(size_t)z * M * N + q]; ci[z] = im[(size_t)z * M * N + q]; }
            orc_fft(D, cr, ci, inverse);
            for (int z = 0; z < D; z++) { re[(size_t)z * M * N + q] = cr[z]; im[(size_t)z * M * N + q] = ci[z]; }
        }
        free(cr); free(ci);
    }
    return 0;
}

/* Eq. (32) in 3-D (Q10, Q26): 1 - tau mu (2cos z1 + 2cos z2 + 2cos z3 - 6). */
double orc3_symbol(int D, int M, int N, double tau, double mu, int k3, int k1, int k2)
{
    double z1 = 2.0 * M_PI * (double)k1 / (double)M;
    double z2 = 2.0 * M_PI * (double)k2 / (double)N;
    double z3 = 2.0 * M_PI * (double)k3 / (double)D;
    return 1.0 - tau * mu * (2.0 * cos(z1) + 2.0 * cos(z2) + 2.0 * cos(z3) - 6.0);
}

int orc3_solve(int D, int M, int N, double tau, double mu, const double *F, double *phi)
{
    size_t n = (size_t)D * M * N;
    double *re = malloc(sizeof(double) * n), *im = calloc(n, sizeof(double));
    memcpy(re, F, sizeof(double) * n);
    orc3_fft3(D, M, N, re, im, 0);
    for (int z = 0; z < D; z++)
        for (int k1 = 0; k1 < M; k1++)
            for (int k2 = 0; k2 < N; k2++) {
                double sg = orc3_symbol(D, M, N, tau, mu, z, k1, k2);
                re[IDX3(z, k1, k2)] /= sg;
                im[IDX3(z, k1, k2)] /= sg;
            }
    orc3_fft3(D, M, N, re, im, 1);
    double fmax = 0.0, imax = 0.0;
    for (size_t q = 0; q < n; q++) {
        if (fabs(F[q]) > fmax) fmax = fabs(F[q]);
        if (fabs(im[q]) > imax) imax = fabs(im[q]);
        phi[q] = re[q];
    }
    free(re); free(im);
    return imax > 1e-12 * (fmax > 0 ? fmax : 1.0) ? 1 : 0;
}

/* P:368 in 3-D: v(x) = sum over the ball p^2+q^2+r^2 <= R^2 (shape 0) or the cube (1) of
 * exp(-(p^2+q^2+r^2)/d^2) u(x + (p,q,r)); terms outside the volume are 0 (Q5). */
void orc3_window_sum(int D, int M, int N, int R, double d, int shape, const double *u1, const double *u2,
                     const double *u3, double *v1, double *v2, double *v3)
{
    #pragma omp parallel for schedule(static)
    for (int z = 0; z < D; z++)
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double a1 = 0.0, a2 = 0.0, a3 = 0.0;
                for (int r = -R; r <= R; r++)
                    for (int p = -R; p <= R; p++)
                        for (int q = -R; q <= R; q++) {
                            if (shape == 0 && p * p + q * q + r * r > R * R) continue;
                            int zz = z + r, ii = i + p, jj = j + q;
                            if (zz < 0 || zz >= D || ii < 0 || ii >= M || jj < 0 || jj >= N) continue;
                            double G = exp(-(double)(p * p + q * q + r * r) / (d * d));
                            size_t s = IDX3(zz, ii, jj);
                            a1 += G * u1[s]; a2 += G * u2[s]; a3 += G * u3[s];
                        }
                size_t o = IDX3(z, i, j);
                v1[o] = a1; v2[o] = a2; v3[o] = a3;
            }
}

/* Eq. (37) in 3-D. */
void orc3_rhs(int D, int M, int N, const orc_params *P, const double *psi, const double *w1, const double *w2,
              const double *w3, const double *b1, const double *b2, const double *b3, const double *g, double *F)
{
    size_t n = (size_t)D * M * N;
    double *u1 = malloc(sizeof(double) * n), *u2 = malloc(sizeof(double) * n), *u3 = malloc(sizeof(double) * n);
    double *v1 = malloc(sizeof(double) * n), *v2 = malloc(sizeof(double) * n), *v3 = malloc(sizeof(double) * n);
    double *c1 = malloc(sizeof(double) * n), *c2 = malloc(sizeof(double) * n), *c3 = malloc(sizeof(double) * n);
    double *dv = malloc(sizeof(double) * n);
    for (size_t q = 0; q < n; q++) {
        double hq = orc_h(psi[q], P->epsilon, P->l);
        u1[q] = hq * w1[q]; u2[q] = hq * w2[q]; u3[q] = hq * w3[q];
        c1[q] = b1[q] - w1[q]; c2[q] = b2[q] - w2[q]; c3[q] = b3[q] - w3[q];
    }
    orc3_window_sum(D, M, N, P->window, P->d, P->window_shape, u1, u2, u3, v1, v2, v3);
    orc3_div(D, M, N, c1, c2, c3, dv);
    #pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; q++) {
        double wn = sqrt(w1[q] * w1[q] + w2[q] * w2[q] + w3[q] * w3[q]);
        double t = -P->gamma * g[q] * wn * orc_delta_prime(psi[q], P->epsilon)
                 + P->alpha * g[q] * orc_delta(psi[q], P->epsilon)
                 + 2.0 * P->beta * orc_h_prime(psi[q], P->epsilon, P->l)
                       * (w1[q] * v1[q] + w2[q] * v2[q] + w3[q] * v3[q])
                 + P->mu * dv[q];
        F[q] = psi[q] + P->tau * t;
    }
    free(u1); free(u2); free(u3); free(v1); free(v2); free(v3); free(c1); free(c2); free(c3); free(dv);
}

/* Eq. (42) on 3-vectors. */
void orc3_shrink(const double *B, double t, double *o)
{
    double nb = sqrt(B[0] * B[0] + B[1] * B[1] + B[2] * B[2]);
    if (nb > 0.0) {
        double m = nb - t; if (m < 0.0) m = 0.0;
        for (int c = 0; c < 3; c++) o[c] = m * B[c] / nb;
    } else {
        o[0] = o[1] = o[2] = 0.0;
    }
}

/* Eq. (40) on 3-vectors, modes as Q1. */
void orc3_project(int mode, const double *a, double *o)
{
    double n = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    double s = 1.0;
    if (mode == 0) s = n > 1.0 ? n : 1.0;
    else if (mode == 1) s = n > 1e-4 ? n : 1.0;
    for (int c = 0; c < 3; c++) o[c] = a[c] / s;
}

/* w/b update (Eq. 41-42 or 38-39, 40, 23) in 3-D. */
void orc3_wb(int D, int M, int N, const orc_params *P, const double *phi, double *w1, double *w2, double *w3,
             double *b1, double *b2, double *b3, const double *g)
{
    size_t n = (size_t)D * M * N;
    double *gp[3], *u[3], *v[3], *nw[3];
    for (int c = 0; c < 3; c++) {
        gp[c] = malloc(sizeof(double) * n); u[c] = malloc(sizeof(double) * n);
        v[c] = malloc(sizeof(double) * n); nw[c] = malloc(sizeof(double) * n);
    }
    double *w[3] = {w1, w2, w3}, *b[3] = {b1, b2, b3};
    double *hh = malloc(sizeof(double) * n);
    orc3_grad(D, M, N, phi, gp[0], gp[1], gp[2]);
    for (size_t q = 0; q < n; q++) hh[q] = orc_h(phi[q], P->epsilon, P->l);
    if (P->w_mode == 0) {
        for (size_t q = 0; q < n; q++) for (int c = 0; c < 3; c++) u[c][q] = hh[q] * w[c][q];
        orc3_window_sum(D, M, N, P->window, P->d, P->window_shape, u[0], u[1], u[2], v[0], v[1], v[2]);
        for (size_t q = 0; q < n; q++) {
            double B[3], s[3], o[3];
            for (int c = 0; c < 3; c++) B[c] = gp[c][q] + b[c][q] + (2.0 * P->beta / P->mu) * hh[q] * v[c][q];
            double t = (P->gamma / P->mu) * g[q] * orc_delta(phi[q], P->epsilon);
            orc3_shrink(B, t, s);
            orc3_project(P->w_proj, s, o);
            for (int c = 0; c < 3; c++) nw[c][q] = o[c];
        }
    } else {
        for (int c = 0; c < 3; c++) memcpy(nw[c], w[c], sizeof(double) * n);
        for (int r = 0; r < P->w_iters; r++) {
            for (size_t q = 0; q < n; q++) for (int c = 0; c < 3; c++) u[c][q] = hh[q] * nw[c][q];
            orc3_window_sum(D, M, N, P->window, P->d, P->window_shape, u[0], u[1], u[2], v[0], v[1], v[2]);
            for (size_t q = 0; q < n; q++) {
                double den = P->gamma * g[q] * orc_delta(phi[q], P->epsilon) + P->mu;
                double a[3], o[3];
                for (int c = 0; c < 3; c++) a[c] = (P->mu * gp[c][q] + P->mu * b[c][q] + 2.0 * P->beta * hh[q] * v[c][q]) / den;
                orc3_project(P->w_proj, a, o);
                for (int c = 0; c < 3; c++) nw[c][q] = o[c];
            }
        }
    }
    for (size_t q = 0; q < n; q++)
        for (int c = 0; c < 3; c++) {
            b[c][q] = b[c][q] + gp[c][q] - nw[c][q];
            w[c][q] = nw[c][q];
        }
    for (int c = 0; c < 3; c++) { free(gp[c]); free(u[c]); free(v[c]); free(nw[c]); }
    free(hh);
}

void orc3_init(int D, int M, int N, const double *phi0, double *phi, double *w1, double *w2, double *w3,
               double *b1, double *b2, double *b3)
{
    size_t n = (size_t)D * M * N;
    memcpy(phi, phi0, sizeof(double) * n);
    orc3_grad(D, M, N, phi0, w1, w2, w3);
    memset(b1, 0, sizeof(double) * n); memset(b2, 0, sizeof(double) * n); memset(b3, 0, sizeof(double) * n);
}

/* Algorithm 1 in 3-D: K outer iterations of S FFT sweeps, clamp, w/b update. */
int orc3_iterate(int D, int M, int N, const orc_params *P, double *phi, double *w1, double *w2, double *w3,
                 double *b1, double *b2, double *b3, const double *g, int K)
{
    int bad = 0;
    size_t n = (size_t)D * M * N;
    double *F = malloc(sizeof(double) * n);
    for (int k = 0; k < K; k++) {
        for (int s = 0; s < P->S; s++) {
            orc3_rhs(D, M, N, P, phi, w1, w2, w3, b1, b2, b3, g, F);
            bad += orc3_solve(D, M, N, P->tau, P->mu, F, phi);
        }
        if (P->phi_clip > 0.0)
            for (size_t q = 0; q < n; q++) {
                if (phi[q] > P->phi_clip) phi[q] = P->phi_clip;
                if (phi[q] < -P->phi_clip) phi[q] = -P->phi_clip;
            }
        orc3_wb(D, M, N, P, phi, w1, w2, w3, b1, b2, b3, g);
    }
    free(F);
    return bad;
}
