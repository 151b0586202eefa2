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
//   * window sums S_t = sum e, Q_t = sum e u (M_t = Q_t / S_t) in fp64 without
//     subtraction: 32-sample blocks carry warp-scanned prefixes / suffixes and totals,
//     a window is suffix + whole blocks + prefix (about K / 32 + 2 adds per output);
//   * backward (gather form, nothing stored by the forward): the CTA owning children
//     [j0, j0 + SX_N) recomputes S_t, M_t of the outputs t in [j0 - b, j0 + SX_N - a),
//     alpha_t = g_t / S_t, beta_t = alpha_t M_t, then per child the window sums
//     A_j = sum alpha, B_j = sum beta and  d c_j = e_j (A_j + tau (u_j A_j - B_j)).
// One fp64 exp per staged sample, O(K / 32) adds per output; the fp32 vHGW kernels
// remain for masked_fill / padded windows.
#include "fg_reg.cuh"

namespace stlg {

constexpr int SX_W = 4;            // warps per CTA
constexpr int SX_T = SX_W * 32;    // threads
constexpr int SX_N = 512;          // outputs (forward) / children (backward) per CTA
constexpr int SX_KMAX = 2048;
constexpr double SX_TINY = 1e-290;  // smaller window sums: per-window frames

// Window sums without subtraction (no cancellation, fixed order): 32-sample blocks carry
// their inclusive prefix P and suffix Q (warp shuffle scans) and their total; a window of
// K >= 33 samples is Q[start] + (whole blocks) + P[end].  K <= 32: a direct sum.
struct SxBlk {
  double *PX, *QX, *PY, *QY, *BX, *BY;
};

__device__ __forceinline__ SxBlk sx_carve(double* base, int n) {
  const int nb = (n + 31) / 32 + 1;
  return SxBlk{base, base + n, base + 2 * n, base + 3 * n, base + 4 * n, base + 4 * n + nb};
}
__host__ __device__ constexpr int sx_blk_doubles(int n) { return 4 * n + 2 * ((n + 31) / 32 + 1); }

__device__ __forceinline__ void sx_blockify(const double* X, const double* Y, int n, const SxBlk& b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (n + 31) >> 5;
  for (int bk = warp; bk < nb; bk += SX_W) {
    const int i = bk * 32 + lane;
    const double x = i < n ? X[i] : 0.0, y = i < n ? Y[i] : 0.0;
    double px = x, py = y, qx = x, qy = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ax = __shfl_up_sync(0xffffffffu, px, o), ay = __shfl_up_sync(0xffffffffu, py, o);
      const double cx = __shfl_down_sync(0xffffffffu, qx, o), cy = __shfl_down_sync(0xffffffffu, qy, o);
      if (lane >= o) {
        px += ax;
        py += ay;
      }
      if (lane + o < 32) {
        qx += cx;
        qy += cy;
      }
    }
    if (i < n) {
      b.PX[i] = px;
      b.QX[i] = qx;
      b.PY[i] = py;
      b.QY[i] = qy;
    }
    if (lane == 0) {
      b.BX[bk] = qx;
      b.BY[bk] = qy;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void sx_win(const double* X, const double* Y, const SxBlk& b, int r, int K, double& s,
                                       double& q) {
  if (K <= 32) {
    s = q = 0.0;
    for (int k = 0; k < K; ++k) {
      s += X[r + k];
      q += Y[r + k];
    }
    return;
  }
  const int e = r + K - 1, qa = r >> 5, qb = e >> 5;
  s = b.QX[r];
  q = b.QY[r];
  for (int m = qa + 1; m < qb; ++m) {
    s += b.BX[m];
    q += b.BY[m];
  }
  s += b.PX[e];
  q += b.PY[e];
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

// stage u (fp64, max space) over positions [s0, s0 + n) (-inf outside the signal), then
// the frame f = max u and e = exp(tau (u - f)), e u
template <int EK>
__device__ __forceinline__ void sx_stage(const Ev<M_SOFT, EK>& ev, float sg, double tau, int s0, int n, int L,
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
  const int NS = SX_N + K - 1;  // staged positions [t0 + a, t0 + a + NS): output t's window at t - t0
  double* U = sxs;
  double* E = U + NS;
  double* EU = E + NS;
  const SxBlk bl = sx_carve(EU + NS, NS);
  sx_stage<EK>(ev, sg, tau, t0 + p.a, NS, L, U, E, EU, red);
  sx_blockify(E, EU, NS, bl);
  bool fb = false;
  for (int r = threadIdx.x; r < tend - t0; r += SX_T) {
    if (t0 + r >= nvalid) continue;
    double s, q;
    sx_win(E, EU, bl, r, K, s, q);
    fb |= !(s > SX_TINY);
  }
  fb = __syncthreads_or(fb);
  for (int r = threadIdx.x; r < tend - t0; r += SX_T) {
    const int t = t0 + r;
    float v = padv;
    if (t < nvalid) {
      double s, q, m;
      if (fb) sx_exact(U, r, K, tau, m, s, q);
      else sx_win(E, EU, bl, r, K, s, q);
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
  const int tb = j0 - b;         // first output whose window can reach j0
  const int NO = SX_N + K - 1;   // outputs [tb, tb + NO); output r's window at staged r
  const int NS = NO + K - 1;     // staged positions [tb + a, tb + a + NS)
  double* U = sxs;
  double* E = U + NS;
  double* EU = E + NS;
  double* AL = EU + NS;          // alpha_t = g_t / S_t   (L_t on per-window frames)
  double* BE = AL + NO;          // beta_t = alpha_t M_t  (M_t on per-window frames)
  const SxBlk bl = sx_carve(BE + NO, NS);
  sx_stage<EK>(ev, sg, tau, tb + p.a, NS, L, U, E, EU, red);
  sx_blockify(E, EU, NS, bl);
  bool fb = false;
  for (int r = threadIdx.x; r < NO; r += SX_T) {
    const int t = tb + r;
    const bool live = t >= 0 && t < nvalid;
    const float g = live ? cot[t] : 0.f;
    double s = 1.0, q = 0.0;
    if (live && g != 0.f) sx_win(E, EU, bl, r, K, s, q);
    fb |= live && g != 0.f && !(s > SX_TINY);
    const double al = (live && g != 0.f) ? (double)g / s : 0.0;
    AL[r] = al;
    BE[r] = al * (q / s);
  }
  fb = __syncthreads_or(fb);
  if (fb) {  // per-window frames: AL <- L_t (window LSE), BE <- M_t, per-pair exps below
    for (int r = threadIdx.x; r < NO; r += SX_T) {
      const int t = tb + r;
      if (t >= 0 && t < nvalid) {
        double m, s, q;
        sx_exact(U, r, K, tau, m, s, q);
        AL[r] = m + log(s) / tau;
        BE[r] = q / s;
      } else {
        AL[r] = INFINITY;  // exp(tau (u - inf)) = 0: no contribution
        BE[r] = 0.0;
      }
    }
  } else {
    sx_blockify(AL, BE, NO, bl);  // (the staged blocks are no longer needed)
  }
  __syncthreads();
  // child j = j0 + c receives from outputs t in [j - b, j - a]: r in [c, c + K)
  for (int c = threadIdx.x; c < SX_N; c += SX_T) {
    const int j = j0 + c;
    if (j >= L) break;
    const int iu = c + K - 1;  // staged index of j (staged base tb + a = j0 - (K - 1))
    const double u = U[iu];
    double G;
    if (!fb) {
      double A, Bs;
      sx_win(AL, BE, bl, c, K, A, Bs);
      G = E[iu] * (A + tau * (u * A - Bs));
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

static size_t sx_fwd_smem(int K) {
  const int NS = SX_N + K - 1;
  return sizeof(double) * (size_t)(3 * NS + sx_blk_doubles(NS));
}
static size_t sx_bwd_smem(int K) {
  const int NO = SX_N + K - 1, NS = NO + K - 1;
  return sizeof(double) * (size_t)(3 * NS + 2 * NO + sx_blk_doubles(NS));
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
