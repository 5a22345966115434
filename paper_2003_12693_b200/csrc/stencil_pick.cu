// Dispatch on the window radius R (P:368 summation radius, 0..8).
#include "sr_kernels.h"
namespace srsb {
bool pick_stencil(int R, int shape, bool leq, RhsKernel& rhs, WbKernel (&wb)[2][2], WbKernel& wb_mon, int& smem) {
    switch (R) {
        case 0: return pick_stencil_r0(shape, leq, rhs, wb, wb_mon, smem);
        case 1: return pick_stencil_r1(shape, leq, rhs, wb, wb_mon, smem);
        case 2: return pick_stencil_r2(shape, leq, rhs, wb, wb_mon, smem);
        case 3: return pick_stencil_r3(shape, leq, rhs, wb, wb_mon, smem);
        case 4: return pick_stencil_r4(shape, leq, rhs, wb, wb_mon, smem);
        case 5: return pick_stencil_r5(shape, leq, rhs, wb, wb_mon, smem);
        case 6: return pick_stencil_r6(shape, leq, rhs, wb, wb_mon, smem);
        case 7: return pick_stencil_r7(shape, leq, rhs, wb, wb_mon, smem);
        case 8: return pick_stencil_r8(shape, leq, rhs, wb, wb_mon, smem);
    }
    return false;
}
RhsR2cKernel pick_fused(int R, int shape, bool leq, int log2_h, int& smem) {
    switch (R) {
        case 0: return pick_fused_r0(shape, leq, log2_h, smem);
        case 1: return pick_fused_r1(shape, leq, log2_h, smem);
        case 2: return pick_fused_r2(shape, leq, log2_h, smem);
        case 3: return pick_fused_r3(shape, leq, log2_h, smem);
        case 4: return pick_fused_r4(shape, leq, log2_h, smem);
        case 5: return pick_fused_r5(shape, leq, log2_h, smem);
        case 6: return pick_fused_r6(shape, leq, log2_h, smem);
        case 7: return pick_fused_r7(shape, leq, log2_h, smem);
        case 8: return pick_fused_r8(shape, leq, log2_h, smem);
    }
    return nullptr;
}
bool pick_tma(int R, int shape, bool leq, RhsTmaKernel& k, WbTmaKernel (&wb)[2][2], WbTmaKernel& wb_mon,
              int& smem_rhs, int& smem_wb) {
    switch (R) {
        case 0: return pick_tma_r0(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 1: return pick_tma_r1(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 2: return pick_tma_r2(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 3: return pick_tma_r3(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 4: return pick_tma_r4(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 5: return pick_tma_r5(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 6: return pick_tma_r6(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 7: return pick_tma_r7(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
        case 8: return pick_tma_r8(shape, leq, k, wb, wb_mon, smem_rhs, smem_wb);
    }
    return false;
}
}  // namespace srsb

#include "sr_vol3.h"
namespace srsb {
bool pick_vol(int R, int shape, bool leq, VolRhsKernel& rhs, VolWbKernel (&wb)[2][2], int& smem) {
    if (R < 0 || R > 4 || shape < 0 || shape > 1) return false;
    switch (R * 4 + shape * 2 + (leq ? 1 : 0)) {
        case 0: set_vol_r0_s0_l0(rhs, wb, smem); return true;
        case 1: set_vol_r0_s0_l1(rhs, wb, smem); return true;
        case 2: set_vol_r0_s1_l0(rhs, wb, smem); return true;
        case 3: set_vol_r0_s1_l1(rhs, wb, smem); return true;
        case 4: set_vol_r1_s0_l0(rhs, wb, smem); return true;
        case 5: set_vol_r1_s0_l1(rhs, wb, smem); return true;
        case 6: set_vol_r1_s1_l0(rhs, wb, smem); return true;
        case 7: set_vol_r1_s1_l1(rhs, wb, smem); return true;
        case 8: set_vol_r2_s0_l0(rhs, wb, smem); return true;
        case 9: set_vol_r2_s0_l1(rhs, wb, smem); return true;
        case 10: set_vol_r2_s1_l0(rhs, wb, smem); return true;
        case 11: set_vol_r2_s1_l1(rhs, wb, smem); return true;
        case 12: set_vol_r3_s0_l0(rhs, wb, smem); return true;
        case 13: set_vol_r3_s0_l1(rhs, wb, smem); return true;
        case 14: set_vol_r3_s1_l0(rhs, wb, smem); return true;
        case 15: set_vol_r3_s1_l1(rhs, wb, smem); return true;
        case 16: set_vol_r4_s0_l0(rhs, wb, smem); return true;
        case 17: set_vol_r4_s0_l1(rhs, wb, smem); return true;
        case 18: set_vol_r4_s1_l0(rhs, wb, smem); return true;
        case 19: set_vol_r4_s1_l1(rhs, wb, smem); return true;
    }
    return false;
}
}  // namespace srsb
