// smooth.cu — smooth-interval Eventually / Always, LSE and softmax modes
// (masking.py:207-215, 300-305; smoothing.py:85-109; tape.py:360-387).
//
//   w_i = relu(sigmoid(c (i - a L)) - sigmoid(c (i - b L)) - eps),  i = 0..L-1
//   padded = child ++ [pad] * (L - 1)
//   LSE:     out[t] = sg * log(sum_{w_i > 0} w_i exp(tau u_{t+i})) / tau
//   softmax: out[t] = sg * sum w_i u e / sum w_i e,  e = exp(tau u_{t+i})
// with u = sg * padded (max space).  The reference shifts by the hard max of
// the kept entries; here the shift is the running max of the log-weighted
// scores v_i = tau u_{t+i} + ln w_i (the same value in exact arithmetic, and
// it keeps tail weights down to 1e-300 representable: ln w is stored, never w).
// The kept range {i : w_i > 0} is contiguous (a difference of two sigmoids is
// unimodal) and is computed on the host in fp64 together with log2(w_i).
// Hard mode does not come here: it is the vHGW window kernel over the kept
// range with padded-window semantics (fg.cu, padmode).
//
// Backward (gather form, weights recomputed, nothing stored per pair):
//   g_child[j] = sum_{t = j - i} g_t * d out_t / d u_j        (thread per j)
//   d out / d w_i summed over rows and t (thread per i, fp64 atomics), then
//   d_a, d_b, d_c = sum_i dW_i * d w_i / d(a, b, c)            (fp64)
#include "kernels.cuh"

namespace stlg {

constexpr int S_T = 256;    // outputs (or child elements) per CTA
constexpr int S_CH = 1024;  // window offsets staged per chunk
constexpr int S_RP = 8;     // rows per CTA in the d/dw pass

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_fwd(const __grid_constant__ SParams p) {
  __shared__ float U[S_T + S_CH];
  __shared__ float LW[S_CH];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int t0 = blockIdx.x * S_T;
  const int K = p.i_hi - p.i_lo + 1;
  const float sg = p.sg, tau2 = p.mp.tau2;
  const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  const int t = t0 + threadIdx.x;
  float m = -INFINITY, s = 0.f, d = 0.f, u0 = 0.f;
  bool first = true;
  for (int k0 = 0; k0 < K; k0 += S_CH) {
    const int kc = min(S_CH, K - k0);
    const int base = t0 + p.i_lo + k0;
    for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
      int idx = base + q;
      U[q] = sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
    }
    for (int q = threadIdx.x; q < kc; q += S_T) LW[q] = p.lw2[p.i_lo + k0 + q];
    __syncthreads();
    if (t < L) {
      for (int k = 0; k < kc; ++k) {
        float u = U[threadIdx.x + k];
        float v = fmaf(tau2, u, LW[k]);  // log2 of w_i e^{tau u}
        if (first) {
          m = v;
          s = 1.f;
          u0 = u;
          d = 0.f;
          first = false;
          continue;
        }
        if (MODE == M_LSE) {
          lse_add(m, s, v, 1.f);
        } else {
          // online softmax; payload centred on the current top-scoring sample u0
          float dv = v - m;
          float e = ex2f(-fabsf(dv));
          bool up = dv > 0.f;
          float du = u - u0;
          float s_up = fmaf(s, e, 1.f), d_up = e * fmaf(-du, s, d);
          float s_dn = s + e, d_dn = fmaf(du, e, d);
          s = up ? s_up : s_dn;
          d = up ? d_up : d_dn;
          u0 = up ? u : u0;
          m = up ? v : m;
        }
      }
    }
    __syncthreads();
  }
  if (t < L) {
    float lse = (m + lg2f(s)) * p.mp.inv_tau2;  // log(sum w e^{tau u}) / tau, u units
    if (MODE == M_LSE) {
      p.out[row * L + t] = sg * lse;
    } else {
      p.out[row * L + t] = sg * (u0 + d / s);
      p.aux[row * L + t] = lse;
    }
  }
}

// ---------------------------------------------------------------------------
// backward 1: child cotangent, thread per child element j (incl. virtual pad
// positions j >= L, which sum into c[L-1] for 'last' padding)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_bwd_child(const __grid_constant__ SParams p) {
  __shared__ float Gt[S_T + S_CH];
  __shared__ float Mt[S_T + S_CH];
  __shared__ float Lt[(MODE == M_SOFT) ? S_T + S_CH : 1];
  __shared__ float LW[S_CH];
  __shared__ float red[S_T / 32];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int j0 = blockIdx.x * S_T;
  const int K = p.i_hi - p.i_lo + 1;
  const float sg = p.sg, tau2 = p.mp.tau2, tau = p.mp.tau;
  const int j = j0 + threadIdx.x;
  const int jmax = L - 1 + p.i_hi;  // last position any window reaches
  const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  float uj = 0.f;
  if (j <= jmax) uj = sg * (j < L ? expr_eval<MODE>(p.child, row, j, p.mp) : padv);
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  float acc = 0.f;
  // offsets i in [i_lo + k0, i_lo + k0 + kc): t = j - i in [j0 - i_lo - k0 - kc + 1, j0 + S_T - 1 - i_lo - k0]
  for (int k0 = 0; k0 < K; k0 += S_CH) {
    const int kc = min(S_CH, K - k0);
    const int tlo = j0 - p.i_lo - k0 - (kc - 1);
    for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
      int tt = tlo + q;
      bool v = tt >= 0 && tt < L;
      float g = v ? cot[tt] : 0.f;
      Gt[q] = g;
      Mt[q] = (v && g != 0.f) ? sg * outr[tt] : 0.f;
      if (MODE == M_SOFT) Lt[q] = (v && g != 0.f) ? p.aux_in[row * L + tt] : 0.f;
    }
    for (int q = threadIdx.x; q < kc; q += S_T) LW[q] = p.lw2[p.i_lo + k0 + q];
    __syncthreads();
    if (j <= jmax) {
      // t = j - i_lo - k0 - k  ->  index into the staged range: (kc - 1 - k) + threadIdx.x
      for (int k = 0; k < kc; ++k) {
        int q = threadIdx.x + kc - 1 - k;
        float g = Gt[q];
        if (g == 0.f) continue;
        if (MODE == M_LSE) {
          acc = fmaf(g, ex2f(fmaf(tau2, uj - Mt[q], LW[k])), acc);
        } else {
          float w = ex2f(fmaf(tau2, uj - Lt[q], LW[k]));
          acc = fmaf(g * w, fmaf(tau, uj - Mt[q], 1.f), acc);
        }
      }
    }
    __syncthreads();
  }
  float* gb = p.gbuf + row * L;
  if (j < L) {
    if (j == L - 1) atomicAdd(gb + j, acc);
    else gb[j] = acc;
  }
  // virtual pad positions: sum into c[L-1] ('last'); dropped for const padding
  float v = (j >= L && j <= jmax && p.pad_last) ? acc : 0.f;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.f;
    for (int w = 0; w < S_T / 32; ++w) sum += red[w];
    if (sum != 0.f) atomicAdd(gb + (L - 1), sum);
  }
}

// ---------------------------------------------------------------------------
// backward 2: d out / d w_i summed over t and rows (thread per offset i)
//   LSE:  exp(tau (u_{t+i} - M_t)) / tau        softmax: exp(tau (u - L_t)) (u - M_t)
// (zero where w_i == 0: the reference masks those entries before exp, tape.py:372)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_bwd_w(const __grid_constant__ SParams p) {
  __shared__ float U[S_T + S_CH];
  __shared__ float Gt[S_T], Mt[S_T], Lt[S_T];
  const int L = (int)p.L;
  const int t0 = blockIdx.x * S_T;
  const int K = p.i_hi - p.i_lo + 1;
  const float sg = p.sg, tau2 = p.mp.tau2, itau = 1.f / p.mp.tau;
  const long long r0 = (long long)blockIdx.y * S_RP;
  const long long r1 = min(r0 + S_RP, p.B);
  const int nt = min(S_T, L - t0);
  for (int k0 = 0; k0 < K; k0 += S_CH) {
    const int kc = min(S_CH, K - k0);
    // each thread owns offsets i = i_lo + k0 + k, k = threadIdx.x + S_T * c
    float acc[S_CH / S_T];
#pragma unroll
    for (int c = 0; c < S_CH / S_T; ++c) acc[c] = 0.f;
    for (long long row = r0; row < r1; ++row) {
      const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
      const int base = t0 + p.i_lo + k0;
      for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
        int idx = base + q;
        U[q] = sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
      }
      if (threadIdx.x < S_T) {
        int tt = t0 + threadIdx.x;
        bool v = tt < L;
        float g = v ? p.cot[row * L + tt] : 0.f;
        Gt[threadIdx.x] = g;
        Mt[threadIdx.x] = v ? sg * p.out_in[row * L + tt] : 0.f;
        Lt[threadIdx.x] = (MODE == M_SOFT && v) ? p.aux_in[row * L + tt] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < S_CH / S_T; ++c) {
        int k = threadIdx.x + S_T * c;
        if (k >= kc) break;
        float a = 0.f;
        for (int q = 0; q < nt; ++q) {
          float g = Gt[q];
          if (g == 0.f) continue;
          float u = U[q + k];
          if (MODE == M_LSE) a = fmaf(g, ex2f(tau2 * (u - Mt[q])), a);
          else a = fmaf(g * ex2f(tau2 * (u - Lt[q])), u - Mt[q], a);
        }
        acc[c] += a;
      }
      __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < S_CH / S_T; ++c) {
      int k = threadIdx.x + S_T * c;
      if (k >= kc) break;
      int i = p.i_lo + k0 + k;
      if (p.lw2[i] == -INFINITY) continue;
      double v = (double)(sg * acc[c]) * (MODE == M_LSE ? (double)itau : 1.0);
      if (v != 0.0) atomicAdd(p.dw64 + i, v);
    }
  }
}

// ---------------------------------------------------------------------------
// d(a, b, c) from d/dw_i (fp64): w_i = relu(lo - hi - eps),
//   lo = sigmoid(c (i - a L)), hi = sigmoid(c (i - b L))   (masking.py:300-305)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sigmoid_d(double z) {
  if (z >= 0) return 1.0 / (1.0 + exp(-z));
  double ez = exp(z);
  return ez / (1.0 + ez);
}

__global__ void k_smooth_abc(const double* __restrict__ dw64, long long L, double a, double b,
                             double c, double eps, double* d_abc) {
  __shared__ double red[3][32];
  double da = 0, db = 0, dc = 0;
  const double Lf = (double)L;
  for (long long i = threadIdx.x; i < L; i += blockDim.x) {
    double g = dw64[i];
    if (g == 0.0) continue;
    double lo = sigmoid_d((i - a * Lf) * c);
    double hi = sigmoid_d((i - b * Lf) * c);
    if (!(lo - hi - eps > 0)) continue;  // relu gradient is 0 where the clamp is active
    double slo = lo * (1.0 - lo), shi = hi * (1.0 - hi);
    da += g * (-slo * c * Lf);
    db += g * (shi * c * Lf);
    dc += g * (slo * (i - a * Lf) - shi * (i - b * Lf));
  }
  for (int o = 16; o > 0; o >>= 1) {
    da += __shfl_xor_sync(0xffffffffu, da, o);
    db += __shfl_xor_sync(0xffffffffu, db, o);
    dc += __shfl_xor_sync(0xffffffffu, dc, o);
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = da;
    red[1][w] = db;
    red[2][w] = dc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0, s2 = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      s0 += red[0][k];
      s1 += red[1][k];
      s2 += red[2][k];
    }
    d_abc[0] += s0;
    d_abc[1] += s1;
    d_abc[2] += s2;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_smooth_fwd(int mode, SParams& p, cudaStream_t st) {
  dim3 grid((unsigned)((p.L + S_T - 1) / S_T), (unsigned)p.B);
  if (mode == M_LSE) k_smooth_fwd<M_LSE><<<grid, S_T, 0, st>>>(p);
  else k_smooth_fwd<M_SOFT><<<grid, S_T, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_smooth_bwd(int mode, SParams& p, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.gbuf, 0, sizeof(float) * p.B * p.L, st)) != cudaSuccess) return e;
  long long span = p.L + p.i_hi;  // child positions incl. virtual pad positions
  dim3 g1((unsigned)((span + S_T - 1) / S_T), (unsigned)p.B);
  if (mode == M_LSE) k_smooth_bwd_child<M_LSE><<<g1, S_T, 0, st>>>(p);
  else k_smooth_bwd_child<M_SOFT><<<g1, S_T, 0, st>>>(p);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (p.dw64 != nullptr) {
    dim3 g2((unsigned)((p.L + S_T - 1) / S_T), (unsigned)((p.B + S_RP - 1) / S_RP));
    if (mode == M_LSE) k_smooth_bwd_w<M_LSE><<<g2, S_T, 0, st>>>(p);
    else k_smooth_bwd_w<M_SOFT><<<g2, S_T, 0, st>>>(p);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  FGParams q;
  memset(&q, 0, sizeof(q));
  q.B = p.B;
  q.L = p.L;
  q.mp = p.mp;
  q.child = p.child;
  return launch_pointwise_vjp(mode, q, p.gbuf, st);
}

cudaError_t launch_smooth_abc(const double* dw64, long long L, double a, double b, double c,
                              double eps, double* d_abc, cudaStream_t st) {
  k_smooth_abc<<<1, 1024, 0, st>>>(dw64, L, a, b, c, eps, d_abc);
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
