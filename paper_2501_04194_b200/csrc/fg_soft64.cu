// fg_soft64.cu — timed softmax Eventually / Always in fp64 (masking.py:229-235, tape.py:381-386).
//
// Softmax gradients, sum_t g_t w_tj (1 + tau (u_j - M_t)), cancel terms of size
// tau |u - M| w down to O(w): in fp32 (values, window means M and LSEs L stored as
// fp32, ex2.approx weights, fp32 sums) they land at 1-5e-5 against the reference at
// tau = 10 on |x| ~ 8 signals.  These kernels keep everything that the cancellation
// touches in fp64:
//   * the child value u in fp64 (Ev::value64: the reference's x - c, sqrt(dx^2 + dy^2));
//   * per CTA one frame f = max u, e_i = exp(tau (u_i - f)) and e_i u_i in fp64 once per
//     staged sample (exp range 700 nat: a tile whose windows underflow takes the
//     per-window max-shifted path inside the same launch);
//   * window sums S_t = sum e, Q_t = sum e u (M_t = Q_t / S_t), fp64 adds, register
//     blocked: lane l of a warp owns outputs base + l + 32 o (o < SX_O), so every staged
//     element loaded by the warp feeds up to SX_O windows, conflict-free;
//   * backward (gather form, nothing stored by the forward): the CTA owning children
//     [j0, j0 + SX_N) recomputes S_t, M_t of the outputs t in [j0 - b, j0 + SX_N - a),
//     alpha_t = g_t / S_t, beta_t = alpha_t M_t, then per child the window sums
//     A_j = sum alpha, B_j = sum beta and  d c_j = e_j (A_j + tau (u_j A_j - B_j)).
// Work is O(K) fp64 adds per output (no O(K) exps), which at the C2 window (K = 91) costs
// about what the fp32 vHGW kernels cost; they remain for masked_fill / padded windows.
#include "fg_reg.cuh"

namespace stlg {

constexpr int SX_W = 4;            // warps per CTA
constexpr int SX_T = SX_W * 32;    // threads
constexpr int SX_O = 4;            // outputs per lane, 32 apart
constexpr int SX_N = SX_T * SX_O;  // outputs (forward) / children (backward) per CTA
constexpr int SX_KMAX = 2048;
constexpr double SX_TINY = 1e-290;  // smaller window sums: per-window frames

// S[o], Q[o] over staged elements [r0 + 32 o, r0 + 32 o + K) of (A, B)
__device__ __forceinline__ void sx_sums(const double* A, const double* B, int r0, int K, double S[SX_O],
                                        double Q[SX_O]) {
#pragma unroll
  for (int o = 0; o < SX_O; ++o) S[o] = Q[o] = 0.0;
  const int kend = K + 32 * (SX_O - 1);
#pragma unroll 4
  for (int k = 0; k < kend; ++k) {
    const double x = A[r0 + k], y = B[r0 + k];
#pragma unroll
    for (int o = 0; o < SX_O; ++o) {
      const int kk = k - 32 * o;  // warp-uniform
      if (kk >= 0 && kk < K) {
        S[o] += x;
        Q[o] += y;
      }
    }
  }
}

// block max of v (SX_T threads)
__device__ __forceinline__ double sx_bmax(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = red[0];
#pragma unroll
  for (int w = 1; w < SX_W; ++w) m = fmax(m, red[w]);
  __syncthreads();
  return m;
}

// stage u (fp64, max space) over positions [s0, s0 + n) (-inf past the signal), then the
// frame and e, e u; returns the frame
template <int EK>
__device__ __forceinline__ double sx_stage(const Ev<M_SOFT, EK>& ev, float sg, double tau, int s0, int n, int L,
                                           double* U, double* E, double* EU, double* red) {
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < n; i += SX_T) {
    const int pos = s0 + i;
    double u = -INFINITY;
    if (pos >= 0 && pos < L) u = (double)sg * ev.value64(pos, ev.load(pos));
    U[i] = u;
    mx = fmax(mx, u);
  }
  const double f = sx_bmax(mx, red);
  for (int i = threadIdx.x; i < n; i += SX_T) {
    const double u = U[i];
    const double e = (u > -INFINITY) ? exp(tau * (u - f)) : 0.0;
    E[i] = e;
    EU[i] = (e > 0.0) ? e * u : 0.0;
  }
  __syncthreads();
  return f;
}

// per-window max-shifted sums (tiles whose frame underflows a window)
__device__ __forceinline__ void sx_exact(const double* U, int r, int K, double tau, double& m, double& S, double& Q) {
  m = -INFINITY;
  for (int k = 0; k < K; ++k) m = fmax(m, U[r + k]);
  S = Q = 0.0;
  for (int k = 0; k < K; ++k) {
    const double e = exp(tau * (U[r + k] - m));
    S += e;
    Q += e * U[r + k];
  }
}

template <int EK>
__global__ void __launch_bounds__(SX_T) k_sx_fwd(const __grid_constant__ FGParams p) {
  extern __shared__ double sxs[];
  __shared__ double red[SX_W];
  const long long row = blockIdx.y;
  const int L = (int)p.L, K = p.K;
  const int t0 = blockIdx.x * SX_N;
  const int nvalid = L - p.b;  // outputs whose window lies inside the signal
  const float sg = p.sg;
  const double tau = p.mp.tau;
  Ev<M_SOFT, EK> ev(p.child, row, p.mp);
  float* outr = p.out + row * L;
  const float padv = p.pad_last ? ev.value(L - 1, ev.load(L - 1)) : p.pad_value;
  const float czero = p.canon ? 0.f : -0.f;  // x + (-0) == x: the `+ 0.0` rule is one add
  const int tend = min(t0 + SX_N, L);
  if (t0 >= nvalid) {
    for (int t = t0 + (int)threadIdx.x; t < tend; t += SX_T) outr[t] = __fadd_rn(padv, czero);
    return;
  }
  const int NS = SX_N + K + 32 * SX_O;  // staged (+ slack read by the blocked sums)
  double* U = sxs;
  double* E = U + NS;
  double* EU = E + NS;
  sx_stage<EK>(ev, sg, tau, t0 + p.a, NS, L, U, E, EU, red);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = warp * 32 * SX_O + lane;  // staged index of the lane's first window
  double S[SX_O], Q[SX_O];
  sx_sums(E, EU, r0, K, S, Q);
  bool fb = false;
#pragma unroll
  for (int o = 0; o < SX_O; ++o) fb |= (t0 + r0 + 32 * o < nvalid) && !(S[o] > SX_TINY);
  fb = __syncthreads_or(fb);
#pragma unroll
  for (int o = 0; o < SX_O; ++o) {
    const int t = t0 + r0 + 32 * o;
    if (t >= tend) continue;
    float v = padv;
    if (t < nvalid) {
      double s = S[o], q = Q[o];
      if (fb) {
        double m;
        sx_exact(U, r0 + 32 * o, K, tau, m, s, q);
      }
      v = (float)((double)sg * (q / s));
    }
    outr[t] = __fadd_rn(v, czero);
  }
}

template <int EK>
__global__ void __launch_bounds__(SX_T) k_sx_bwd(const __grid_constant__ FGParams p) {
  extern __shared__ double sxs[];
  __shared__ double red[SX_W];
  const long long row = blockIdx.y;
  const int L = (int)p.L, K = p.K, b = p.b;
  const int j0 = blockIdx.x * SX_N;
  const int nvalid = L - b;
  const float sg = p.sg;
  const double tau = p.mp.tau;
  Ev<M_SOFT, EK> ev(p.child, row, p.mp);
  const float* cot = p.cot + row * L;
  const int tb = j0 - b;                       // first output whose window can reach j0
  const int NO = SX_N + K - 1;                 // outputs [tb, tb + NO)
  const int NOR = ((NO + SX_N - 1) / SX_N) * SX_N;  // rounded to whole blocked groups
  const int NS = NOR + K + 32 * SX_O;          // staged positions [tb + a, tb + a + NS)
  double* U = sxs;
  double* E = U + NS;
  double* EU = E + NS;
  double* AL = EU + NS;                        // alpha_t (or L_t on per-window frames)
  double* BE = AL + NOR + K + 32 * SX_O;       // beta_t  (or M_t)
  sx_stage<EK>(ev, sg, tau, tb + p.a, NS, L, U, E, EU, red);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // phase 1: window sums of the outputs
  bool fb = false;
  for (int g0 = 0; g0 < NOR; g0 += SX_N) {
    const int r0 = g0 + warp * 32 * SX_O + lane;
    double S[SX_O], Q[SX_O];
    sx_sums(E, EU, r0, K, S, Q);
#pragma unroll
    for (int o = 0; o < SX_O; ++o) {
      const int r = r0 + 32 * o, t = tb + r;
      const bool live = r < NO && t >= 0 && t < nvalid;
      const float g = live ? cot[t] : 0.f;
      fb |= live && g != 0.f && !(S[o] > SX_TINY);
      AL[r] = live ? (double)g / S[o] : 0.0;
      BE[r] = live ? ((double)g / S[o]) * (Q[o] / S[o]) : 0.0;
    }
  }
  for (int r = NOR + (int)threadIdx.x; r < NOR + K + 32 * SX_O; r += SX_T) AL[r] = BE[r] = 0.0;
  fb = __syncthreads_or(fb);
  if (fb) {  // per-window frames: AL <- L_t (window LSE), BE <- M_t, per-pair exps below
    for (int r = threadIdx.x; r < NOR; r += SX_T) {
      const int t = tb + r;
      if (r < NO && t >= 0 && t < nvalid) {
        double m, s, q;
        sx_exact(U, r, K, tau, m, s, q);
        AL[r] = m + log(s) / tau;
        BE[r] = q / s;
      } else {
        AL[r] = INFINITY;  // exp(tau (u - inf)) = 0: no contribution
        BE[r] = 0.0;
      }
    }
    __syncthreads();
  }
  // phase 2: child j = j0 + c receives from outputs t in [j - b, j - a]: r in [c, c + K)
  const int r0 = warp * 32 * SX_O + lane;
  double A[SX_O], Bs[SX_O];
  if (!fb) sx_sums(AL, BE, r0, K, A, Bs);
#pragma unroll
  for (int o = 0; o < SX_O; ++o) {
    const int c = r0 + 32 * o, j = j0 + c;
    if (j >= L) continue;
    const int iu = c + K - 1;  // staged index of j (staged base tb + a = j0 - (K - 1))
    const double u = U[iu];
    double G;
    if (!fb) {
      G = E[iu] * (A[o] + tau * (u * A[o] - Bs[o]));
    } else {
      G = 0.0;
      for (int k = 0; k < K; ++k) {
        const int r = c + k, t = tb + r;
        if (t < 0 || t >= nvalid) continue;
        const double g = (double)cot[t];
        if (g == 0.0) continue;
        G += g * exp(tau * (u - AL[r])) * (1.0 + tau * (u - BE[r]));
      }
    }
    if (j == L - 1 && p.pad_last)  // overrun outputs take the pad value c[L-1] ('last')
      for (int t = max(nvalid, 0); t < L; ++t) G += (double)cot[t];
    ev.grad(j, ev.load(j), (float)G);
  }
}

static size_t sx_fwd_smem(int K) { return sizeof(double) * 3 * (size_t)(SX_N + K + 32 * SX_O); }
static size_t sx_bwd_smem(int K) {
  const int NO = SX_N + K - 1;
  const int NOR = ((NO + SX_N - 1) / SX_N) * SX_N;
  const size_t NS = (size_t)NOR + K + 32 * SX_O;
  return sizeof(double) * (3 * NS + 2 * NS);
}

bool sx_applicable(const FGParams& p) {
  return !p.fill && !p.padmode && p.K >= 1 && p.K <= SX_KMAX && p.L < (1LL << 30) &&
         p.B <= 65535 && sx_bwd_smem(p.K) <= 200 * 1024;
}

template <typename KernT>
static cudaError_t sx_launch(KernT k, const FGParams& p, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + SX_N - 1) / SX_N), (unsigned)p.B);
  k<<<grid, SX_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sx_fwd(FGParams& p, cudaStream_t st) {
  cudaError_t e;
  REG_DISPATCH_EK(expr_kind(p.child), e = sx_launch(k_sx_fwd<EK>, p, sx_fwd_smem(p.K), st))
  return e;
}

// writes every child gradient element through the fused child VJP
cudaError_t launch_sx_bwd(FGParams& p, cudaStream_t st) {
  cudaError_t e;
  REG_DISPATCH_EK(expr_kind(p.child), e = sx_launch(k_sx_bwd<EK>, p, sx_bwd_smem(p.K), st))
  return e;
}

}  // namespace stlg
