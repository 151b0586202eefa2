// fg_reg_fwd.cu — forward launchers of the register-blocked timed F / G kernels:
// chunk-aligned van Herk / Gil-Werman (fg_cav.cuh) for K >= 17, the segmented
// variant (fg_reg.cuh) for 2 <= K <= 16.  Also the dispatch predicates shared
// with the backward.
#include "fg_cav.cuh"

namespace stlg {

bool reg_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("STLG_REG");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool reg_applicable(int mode, const FGParams& p, bool bwd) {
  if (mode != M_HARD && mode != M_LSE && !(mode == M_SOFT && p.K >= 17)) return false;
  if (p.padmode || p.fill || p.K < 2 || p.L >= (1LL << 30) || p.B > 65535) return false;
  return reg_pick_nw(p.L, p.K, bwd && mode == M_HARD) > 0;
}

template <int NW>
static cudaError_t fwd_nw(int mode, int ek, FGParams& p, cudaStream_t st) {
  using C = RC<NW>;
  const int J = C::N - p.K + 1;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  const bool cav = p.K >= 17;
  cudaError_t e;
  if (mode == M_HARD) {
    const size_t smem = (size_t)C::NP * 4;
    if (cav) {
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

cudaError_t launch_reg_fwd(int mode, int ek, FGParams& p, cudaStream_t st) {
  cudaError_t e;
  REG_DISPATCH_NW(reg_pick_nw(p.L, p.K, false, mode != M_SOFT), e = fwd_nw<NW>(mode, ek, p, st))
  return e;
}

}  // namespace stlg
