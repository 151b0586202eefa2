// fg_reg_inst.cu — one tile width (NW) and one direction of the register-blocked timed
// F / G kernels per object: build_lib.py compiles this file ten times with
// -DREG_NW=4..8 and -DREG_BWD=0|1 (each instantiates ~30 kernels; one translation unit
// for all of them took over five minutes).  The dispatchers live in fg_reg_fwd.cu.
//   forward: chunk-aligned van Herk / Gil-Werman (fg_cav.cuh) for K >= 17, the segmented
//            variant (fg_reg.cuh) for 2 <= K <= 16;
//   backward: LSE gather form, hard first-argmax runs, softmax (K >= 17).
#include "fg_cav.cuh"

#ifndef REG_NW
#error "compile with -DREG_NW=3..8 -DREG_BWD=0|1 (build_lib.py)"
#endif

namespace stlg {

#if REG_BWD == 0
template <int NW>
cudaError_t fwd_nw(int mode, int ek, FGParams& p, cudaStream_t st) {
  using C = RC<NW>;
  const int J = C::N - p.K + 1;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  const bool cav = p.K >= 17;
  cudaError_t e;
  if (mode == M_HARD) {
    const size_t smem = (size_t)C::NP * 4;
    if (cav && p.aux != nullptr) {  // keep every window's first arg-max for the backward
      REG_DISPATCH_EK(ek, e = reg_launch(k_cav_fwd<RK_HARDI, M_HARD, EK, NW>, grid, C::T, 2 * smem, p, st))
    } else if (cav) {
      REG_DISPATCH_EK(ek, e = reg_launch(k_cav_fwd<RK_HARD, M_HARD, EK, NW>, grid, C::T, smem, p, st))
    } else {
      REG_DISPATCH_EK(ek, e = reg_launch(k_reg_fwd<RK_HARD, M_HARD, EK, NW>, grid, C::T, smem, p, st))
    }
  } else if (mode == M_SOFT) {  // K >= 17 (reg_applicable)
    const size_t smem = (size_t)3 * C::NP * 4;
    REG_DISPATCH_EK(ek, e = reg_launch(k_cav_fwd<RK_SOFT, M_SOFT, EK, NW>, grid, C::T, smem, p, st))
  } else {
    const size_t smem = (size_t)2 * C::NP * 4;
    if (cav) {
      REG_DISPATCH_EK(ek, e = reg_launch(k_cav_fwd<RK_LSE, M_LSE, EK, NW>, grid, C::T, smem, p, st))
    } else {
      REG_DISPATCH_EK(ek, e = reg_launch(k_reg_fwd<RK_LSE, M_LSE, EK, NW>, grid, C::T, smem, p, st))
    }
  }
  return e;
}

template cudaError_t fwd_nw<REG_NW>(int, int, FGParams&, cudaStream_t);
#else
template <int NW>
cudaError_t bwd_nw(int mode, int ek, FGParams& p, cudaStream_t st) {
  using C = RC<NW>;
  const bool cav = p.K >= 17;
  cudaError_t e;
  if (mode == M_HARD) {
    const int J = C::N - 2 * p.K + 2;
    dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
    const size_t smem = (size_t)3 * C::NP * 4;
    if (cav) {
      if (p.aux_in != nullptr) {  // the forward's arg-max: no recomputation (two arrays)
        REG_DISPATCH_EK(ek, e = reg_launch(k_cav_bwd_hard<EK, NW, true>, grid, C::T, 2 * C::NP * 4, p, st))
      } else {
        REG_DISPATCH_EK(ek, e = reg_launch(k_cav_bwd_hard<EK, NW, false>, grid, C::T, smem, p, st))
      }
    } else {
      REG_DISPATCH_EK(ek, e = reg_launch(k_reg_bwd_hard<EK, NW>, grid, C::T, smem, p, st))
    }
  } else if (mode == M_SOFT) {  // K >= 17 (reg_applicable)
    const int J = C::N - p.K + 1;
    dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
    REG_DISPATCH_EK(ek, e = reg_launch(k_cav_bwd_soft<EK, NW>, grid, C::T, (size_t)3 * C::NP * 4, p, st))
  } else {
    const int J = C::N - p.K + 1;
    dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
    const size_t smem = (size_t)2 * C::NP * 4;
    if (cav) {
      REG_DISPATCH_EK(ek, e = reg_launch(k_cav_bwd_lse<EK, NW>, grid, C::T, smem, p, st))
    } else {
      REG_DISPATCH_EK(ek, e = reg_launch(k_reg_bwd_lse<EK, NW>, grid, C::T, smem, p, st))
    }
  }
  return e;
}

template cudaError_t bwd_nw<REG_NW>(int, int, FGParams&, cudaStream_t);
#endif

}  // namespace stlg
