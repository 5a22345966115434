// sr_kernels.h -- kernel function-pointer types and the per-size pickers (instantiated in
// fft_*.cu / stencil_r*.cu so the template instantiations compile in parallel).
#pragma once
#include "sr_fft.cuh"
#include "sr_stencil.cuh"
#include "sr_fused.cuh"

namespace srsb {

typedef void (*RowKernel)(const float*, float2*, const float2*, const float2*, FftRowArgs);
typedef void (*RowInvKernel)(const float2*, float*, const float2*, const float2*, FftRowArgs);
typedef void (*ColKernel)(float2*, const float2*, const float*, const float*, FftColArgs);
typedef void (*RhsKernel)(const float*, const float*, const float*, const float*, float*, StencilArgs);
typedef void (*RhsTmaKernel)(const RhsMaps, const float*, float*, StencilArgs);
typedef void (*WbTmaKernel)(const RhsMaps, float*, float*, int*, StencilArgs);
typedef void (*RhsR2cKernel)(const RhsMaps, const float*, float2*, const float2*, const float2*, StencilArgs, int);
typedef void (*WbKernel)(const float*, const float*, float*, float*, const float*, int*, StencilArgs);

RowKernel pick_row_fwd(int log2_h);       // fft_r2c.cu
RowInvKernel pick_row_inv(int log2_h);    // fft_c2r.cu
RowKernel pick_row_fwd_shape(int log2_h, int lg_rpc, int lg_G);      // specialised launch shapes, else generic
RowInvKernel pick_row_inv_shape(int log2_h, int lg_rpc, int lg_G);
ColKernel pick_col(int log2_m, bool contig, bool symt);   // fft_cols.cu; contig: whole image, G = 1; symt: symbol table
typedef void (*ColPKernel)(float2*, const float2*, const float*, const float*, FftColArgs, int, int);
ColPKernel pick_col_p(int log2_m, bool symt);      // fft_cols.cu: persistent prefetching solve, M >= 4096
typedef void (*LinesFftKernel)(float2*, const float2*, int, int);
LinesFftKernel pick_lines_fft(int log2_m, bool inverse);   // fft_lines.cu: batched complex FFT of contiguous lines, M = 8 .. 8192
// stencil_r<R>.cu; returns false if R is unsupported.  smem = dynamic shared bytes.
bool pick_stencil(int R, int shape, bool leq, RhsKernel& rhs, WbKernel (&wb)[2][2], WbKernel& wb_mon, int& smem);

bool pick_tma(int R, int shape, bool leq, RhsTmaKernel& k, WbTmaKernel (&wb)[2][2], WbTmaKernel& wb_mon,
              int& smem_rhs, int& smem_wb);

// k_rhs_r2c (sr_fused.cuh) for N = 2^(log2_h + 1) in 128 .. 1024; null if not instantiated
RhsR2cKernel pick_fused(int R, int shape, bool leq, int log2_h, int& smem);

#define SRSB_DECLARE_STENCIL(R) RhsR2cKernel pick_fused_r##R(int shape, bool leq, int log2_h, int& smem); \
 bool pick_stencil_r##R(int shape, bool leq, RhsKernel& rhs, WbKernel (&wb)[2][2], WbKernel& wb_mon, int& smem); \
    bool pick_tma_r##R(int shape, bool leq, RhsTmaKernel& k, WbTmaKernel (&wb)[2][2], WbTmaKernel& wb_mon, int& smem_rhs, int& smem_wb);
SRSB_DECLARE_STENCIL(0) SRSB_DECLARE_STENCIL(1) SRSB_DECLARE_STENCIL(2) SRSB_DECLARE_STENCIL(3)
SRSB_DECLARE_STENCIL(4) SRSB_DECLARE_STENCIL(5) SRSB_DECLARE_STENCIL(6) SRSB_DECLARE_STENCIL(7)
SRSB_DECLARE_STENCIL(8)
#undef SRSB_DECLARE_STENCIL

}  // namespace srsb
