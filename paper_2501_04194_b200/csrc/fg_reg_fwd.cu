// fg_reg_fwd.cu — dispatch of the register-blocked timed F / G kernels (forward and
// backward launchers pick the tile width NW; the kernels are instantiated per NW in
// fg_reg_inst.cu), and the dispatch predicates shared by both directions.
#include "fg_reg.cuh"

namespace stlg {

bool reg_applicable(int mode, const FGParams& p, bool bwd) {
  if (mode != M_HARD && mode != M_LSE && !(mode == M_SOFT && p.K >= 17)) return false;
  if (p.padmode || p.fill || p.K < 2 || p.L >= (1LL << 30) || p.B > 65535) return false;
  return reg_pick_nw(p.L, p.K, bwd && mode == M_HARD) > 0;
}

template <int NW>
cudaError_t fwd_nw(int mode, int ek, FGParams& p, cudaStream_t st);  // fg_reg_inst.cu
template <int NW>
cudaError_t bwd_nw(int mode, int ek, FGParams& p, cudaStream_t st);  // fg_reg_inst.cu

cudaError_t launch_reg_fwd(int mode, int ek, FGParams& p, cudaStream_t st) {
  cudaError_t e;
  REG_DISPATCH_NW(reg_pick_nw(p.L, p.K, false, mode != M_SOFT), e = fwd_nw<NW>(mode, ek, p, st))
  return e;
}

cudaError_t launch_reg_bwd(int mode, int ek, FGParams& p, cudaStream_t st) {
  cudaError_t e;
  REG_DISPATCH_NW(reg_pick_nw(p.L, p.K, mode == M_HARD), e = bwd_nw<NW>(mode, ek, p, st))
  return e;
}

}  // namespace stlg
