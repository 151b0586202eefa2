// kernels.cuh — parameter blocks and launch entry points of the stlg kernels.
#pragma once

#include "common.cuh"

namespace stlg {

// Eventually / Always (timed [a,b], untimed) and pointwise expression kernels.
struct FGParams {
  DExpr child;
  const float* out_in;  // backward: this node's forward trace (v-space)
  const float* aux_in;  // backward, softmax: window LSE L_t (u-space)
  const float* cot;     // backward: cotangent of this node's trace
  float* out;           // forward: trace (v-space); pointwise: output
  float* aux;           // forward, softmax: L_t
  float* gbuf;          // backward scratch [B, L] (hard untimed / brute force)
  long long B, L;
  int a, b, K, Kp, NB;
  float sg;       // +1 Eventually (max), -1 Always (min)
  int pad_last;   // PaddingPolicy('last')
  float pad_value;
  int canon;      // reproduce masking.py:192's `+ 0.0` (b > 0 and some window fits)
  int padmode;    // 1: windows read the padded child (smooth-interval hard path, no overrun rule)
  int fill;       // masked_fill compat: reduce sentinel-filled full columns (masking.py:195-202)
  float sent;     // SemanticsConfig.sentinel
  unsigned* lb;   // untimed scans: look-back slots [B][tiles][LB_WORDS] (lookback.cuh)
  ModeP mp;
};

// Until (timed [a,b] and untimed).
struct UParams {
  DExpr left, right;
  const float* out_in;
  const float* cot;
  float* out;
  float* gl;  // backward scratch: cotangent of the left child  [B, L]
  float* gr;  // backward scratch: cotangent of the right child [B, L]
  long long B, L;
  int a, b, K;
  int untimed;
  int pad_last;
  float pad_value;
  int canon;
  int fill;    // masked_fill compat: sentinel-filled columns, no overrun rule (masking.py:261-270)
  float sent;  // SemanticsConfig.sentinel
  float* scratch;  // backward: per-thread checkpoint slab of the persistent kernel (or null)
  unsigned long long* dacc;  // backward: reproducible accumulators [4][B, L] (detacc.cuh)
  int* dscale;               // backward: per-row grid exponents [B]
  unsigned* lb;              // untimed hard: look-back slots [B][tiles][LB_WORDS] (lookback.cuh)
  unsigned short* src;            // forward, hard timed (until_ht.cu): gradient source of every
  const unsigned short* src_in;   // output as (offset from t) | 0x8000 right child; 0xffff overrun
  int ht_nt, ht_ns;               // hard timed forward: outputs / staged positions per tile (host-set)
  ModeP mp;
};

// Smooth-interval F / G, LSE / softmax (weighted window of length L over the padded child).
struct SParams {
  DExpr child;
  const float* out_in;  // backward: this node's trace
  const float* aux_in;  // backward, softmax: weighted window LSE
  const float* cot;
  float* out;
  float* aux;          // forward, softmax
  const float* lw2;    // log2 w_i (fp32; -inf where w_i == 0), i = 0..L-1
  double* dw64;        // backward: d out / d w_i summed over rows and t [L] (fp64)
  double* dwpart;      // backward: per-row-tile partials of dw64 [smooth_dw_parts(B), L]
  float* gbuf;         // backward scratch: cotangent of the child [B, L]
  long long B, L;
  int i_lo, i_hi;      // kept index range {i : w_i > 0}
  float sg;
  int pad_last;
  float pad_value;
  ModeP mp;
};

// rows per CTA of the d/dw pass; each CTA writes one partial row of d out / d w_i and a
// second pass sums the partials in a fixed order (deterministic d(a, b, c))
// d/dw pass: one CTA (and one fp64 partial row) per ceil(B / parts) rows, parts = one
// wave of resident CTAs (148 SMs x 4) so the pass has no partial second wave
inline long long smooth_dw_parts(long long B) { return B < 592 ? B : 592; }

// timed softmax F / G in fp64 (fg_soft64.cu): applicability, forward, fused backward
bool sx_applicable(const FGParams& p);
cudaError_t launch_sx_fwd(FGParams& p, cudaStream_t st);
cudaError_t launch_sx_bwd(FGParams& p, cudaStream_t st);

// hard timed Until in O(T) (until_ht.cu): applicability, forward, backward into gl / gr
bool until_ht_applicable(const UParams& p);
cudaError_t launch_until_ht_fwd(UParams& p, cudaStream_t st);
cudaError_t launch_until_ht_bwd(UParams& p, cudaStream_t st);

// log2 weight table + log2 suffix sums [2L] of one smooth interval, on the device
cudaError_t launch_smooth_table(double a, double b, double c, double eps, long long L, int i_lo, int i_hi,
                                float* lw2, cudaStream_t st);

// fp64 weight table and its (a, b, c) partials -> d_abc (one smooth slot)
cudaError_t launch_smooth_abc(const double* dw64, const float* lw2, long long L, double a, double b,
                              double c, double eps, double* d_abc, cudaStream_t st);

// launchers (return cudaError_t)
cudaError_t launch_pointwise_fwd(int mode, const FGParams& p, cudaStream_t st);
cudaError_t launch_pointwise_vjp(int mode, const FGParams& p, const float* g, cudaStream_t st);
cudaError_t launch_fg_timed_fwd(int mode, FGParams& p, cudaStream_t st);
cudaError_t launch_fg_timed_bwd(int mode, FGParams& p, cudaStream_t st);
cudaError_t launch_fg_untimed_fwd(int mode, FGParams& p, cudaStream_t st);
cudaError_t launch_fg_untimed_bwd(int mode, FGParams& p, cudaStream_t st);
size_t until_bwd_scratch_bytes(int mode, int untimed, int fill, long long L, int b, int K);
// look-back slots of the multi-CTA untimed scans (lookback.cuh): tiles of >= 1024 samples
constexpr int LB_MIN_TILE = 1024;
inline size_t lb_slot_bytes(long long B, long long L) {  // + the ticket counter's slot
  return (size_t)B * (size_t)((L + LB_MIN_TILE - 1) / LB_MIN_TILE) * 32 + 32;
}
cudaError_t launch_mining_grid(int mode, const float* x, long long n, int L, long long rs, const double* a,
                               const double* b, long long npairs, double c, double eps, float tau,
                               double gamma, double* loss, double* dloss, cudaStream_t st);
cudaError_t launch_until_fwd(int mode, UParams& p, cudaStream_t st);
cudaError_t launch_until_bwd(int mode, UParams& p, cudaStream_t st);
cudaError_t launch_smooth_fwd(int mode, SParams& p, cudaStream_t st);
cudaError_t launch_smooth_bwd(int mode, SParams& p, cudaStream_t st);


cudaError_t launch_fill_strided(float* p, long long B, long long T, long long rs, long long es,
                                float v, cudaStream_t st);

// launch accounting (exec.cu)
void count_launch(int n = 1);

// register-blocked exact timed F / G (hard, LSE): fg_reg.cu
bool reg_applicable(int mode, const FGParams& p, bool bwd);
cudaError_t launch_reg_fwd(int mode, int ek, FGParams& p, cudaStream_t st);
cudaError_t launch_reg_bwd(int mode, int ek, FGParams& p, cudaStream_t st);
bool launch_unt_fwd(int mode, FGParams& p, cudaStream_t st, cudaError_t& err);  // fg_unt.cu
bool launch_unt_bwd(int mode, FGParams& p, cudaStream_t st, cudaError_t& err);

}  // namespace stlg
