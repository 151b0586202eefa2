// fg_reg_bwd.cu — backward launchers of the register-blocked timed F / G kernels
// (LSE gather form, hard first-argmax runs): chunk-aligned (fg_cav.cuh) for
// K >= 17, segmented (fg_reg.cuh) for 2 <= K <= 16.
#include "fg_cav.cuh"

namespace stlg {

template <int NW>
static cudaError_t bwd_nw(int mode, int ek, FGParams& p, cudaStream_t st) {
  using C = RC<NW>;
  const bool cav = p.K >= 17;
  cudaError_t e;
  if (mode == M_HARD) {
    const int J = C::N - 2 * p.K + 2;
    dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
    const size_t smem = (size_t)3 * C::NP * 4;
    if (cav) {
      REG_DISPATCH_EK(ek, e = reg_launch(k_cav_bwd_hard<EK, NW>, grid, C::T, smem, p, st))
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
    const size_t smem = (size_t)(cav ? 3 : 2) * C::NP * 4;
    if (cav) {
      REG_DISPATCH_EK(ek, e = reg_launch(k_cav_bwd_lse<EK, NW>, grid, C::T, smem, p, st))
    } else {
      REG_DISPATCH_EK(ek, e = reg_launch(k_reg_bwd_lse<EK, NW>, grid, C::T, smem, p, st))
    }
  }
  return e;
}

cudaError_t launch_reg_bwd(int mode, int ek, FGParams& p, cudaStream_t st) {
  cudaError_t e;
  REG_DISPATCH_NW(reg_pick_nw(p.L, p.K, mode == M_HARD), e = bwd_nw<NW>(mode, ek, p, st))
  return e;
}

}  // namespace stlg
