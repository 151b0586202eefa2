// fg.cu — Eventually / Always kernels (timed [a, b] and untimed) plus the
// pointwise expression kernels.
//
// Reference semantics (masking.py:205-235, tape.py:338-391, 475-535):
//   timed:    out[t] = R_{i=a..b} c[t+i]           if t + b <= L-1
//             out[t] = pad (c[L-1] | const v)       otherwise    (masking.py:180-192)
//   untimed:  out[t] = R_{j=t..L-1} c[j]
// with R = hard max (first arg-max), log-sum-exp or softmax mean under
// temperature tau, and Always = -Eventually(-c).  Everything runs in
// "max space" u = sg * c; the output is sg * R(u).
//
// Timed windows use the van Herk / Gil-Werman decomposition: the child
// sequence is cut into blocks of K = b - a + 1 samples; every window of
// length K is (suffix of block q) (+) (prefix of block q+1), so each output
// costs O(1) monoid combines regardless of K.  One thread owns one block:
// it writes its block's prefix scan to shared memory, then walks the block
// backwards building the suffix on the fly and combining it with the next
// block's prefix.  The monoids carry the reference's detached max shift
// (LSE / softmax are computed exactly as m + log(sum e^{tau (u - m)}) / tau
// with m the window's hard max), so the only approximation is fp32 + MUFU.
//
// The backward is in gather form: the CTA that owns child element j
// computes g_child[j] = sum_t g_t d out_t / d c_j over t in [j-b, j-a] as a
// second sliding-window reduction over the cotangent sequence (LSE /
// softmax) or by scattering each g_t to its recomputed arg-max in shared
// memory (hard), then runs the child expression's VJP at j — so the
// cotangent of an elementwise child is never materialised.
#include "kernels.cuh"

namespace stlg {

// ===========================================================================
// pointwise expression kernels (root formula / materialised sub-formulas)
// ===========================================================================
template <int MODE>
__global__ void __launch_bounds__(256) k_pointwise_fwd(const __grid_constant__ FGParams p) {
  const long long n = p.B * p.L;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long row = i / p.L, t = i - row * p.L;
    p.out[i] = expr_eval<MODE>(p.child, row, t, p.mp);
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_pointwise_vjp(const __grid_constant__ FGParams p,
                                                       const float* __restrict__ g) {
  const long long n = p.B * p.L;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long row = i / p.L, t = i - row * p.L;
    expr_vjp<MODE>(p.child, row, t, g[i], p.mp);
  }
}

static int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  long long cap = 148LL * 16;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

cudaError_t launch_pointwise_fwd(int mode, const FGParams& p, cudaStream_t st) {
  int grid = grid_for(p.B * p.L, 256);
  if (mode == M_HARD) k_pointwise_fwd<M_HARD><<<grid, 256, 0, st>>>(p);
  else if (mode == M_LSE) k_pointwise_fwd<M_LSE><<<grid, 256, 0, st>>>(p);
  else k_pointwise_fwd<M_SOFT><<<grid, 256, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pointwise_vjp(int mode, const FGParams& p, const float* g, cudaStream_t st) {
  int grid = grid_for(p.B * p.L, 256);
  if (mode == M_HARD) k_pointwise_vjp<M_HARD><<<grid, 256, 0, st>>>(p, g);
  else if (mode == M_LSE) k_pointwise_vjp<M_LSE><<<grid, 256, 0, st>>>(p, g);
  else k_pointwise_vjp<M_SOFT><<<grid, 256, 0, st>>>(p, g);
  count_launch();
  return cudaGetLastError();
}

// ===========================================================================
// timed F / G — forward (vHGW)
// ===========================================================================
// shared layout: NB blocks, row stride Kp (odd => conflict-free per-thread walks)
//   u[NB*Kp]                 child in max space; overwritten in place by outputs
//   P0, P1 [, P2]            prefix states (hard: value, index; lse: m, s; soft: m, s, d)
//   AX (soft)                window LSE (aux output)
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_fwd(const __grid_constant__ FGParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float padv_sh;
  const int NB = p.NB, K = p.K, Kp = p.Kp;
  const long long row = blockIdx.y, L = p.L;
  const long long J = (long long)(NB - 1) * K;
  const long long t0 = (long long)blockIdx.x * J;
  const long long nvalid = L - p.b;
  const long long s0 = t0 + p.a;
  const int nsm = NB * Kp;
  float* u = sm;
  float* P0 = sm + nsm;
  float* P1 = sm + 2 * nsm;
  float* P2 = sm + 3 * nsm;
  float* AX = sm + 4 * nsm;
  const float tau2 = p.mp.tau2;
  const bool any = t0 < nvalid;

  if (threadIdx.x == 0)
    padv_sh = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  if (any) {
    const int n = NB * K;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int blk = i / K, off = i - blk * K;
      long long idx = s0 + i;
      u[blk * Kp + off] = idx < L ? p.sg * expr_eval<MODE>(p.child, row, idx, p.mp) : -INFINITY;
    }
  }
  __syncthreads();
  if (any && threadIdx.x < NB) {  // prefix scan of own block
    const int base = threadIdx.x * Kp;
    if (MODE == M_HARD) {
      float bv = u[base];
      P0[base] = bv;
      for (int i = 1; i < K; ++i) {
        float x = u[base + i];
        if (x > bv) bv = x;
        P0[base + i] = bv;
      }
    } else if (MODE == M_LSE) {
      LseAcc a = {u[base], 1.f};
      P0[base] = a.m;
      P1[base] = a.s;
      for (int i = 1; i < K; ++i) {
        a = lse_push(a, u[base + i], tau2);
        P0[base + i] = a.m;
        P1[base + i] = a.s;
      }
    } else {
      SoftAcc a = {u[base], 1.f, 0.f};
      P0[base] = a.m;
      P1[base] = a.s;
      P2[base] = a.d;
      for (int i = 1; i < K; ++i) {
        a = soft_push(a, u[base + i], tau2);
        P0[base + i] = a.m;
        P1[base + i] = a.s;
        P2[base + i] = a.d;
      }
    }
  }
  __syncthreads();
  if (any && threadIdx.x < NB - 1) {  // suffix walk + combine with next block's prefix
    const int base = threadIdx.x * Kp, nb = base + Kp;
    if (MODE == M_HARD) {
      float acc = -INFINITY;
      for (int i = K - 1; i >= 0; --i) {
        float x = u[base + i];
        if (x >= acc) acc = x;  // value only; ties keep the earlier element (same value)
        float r = acc;
        if (i > 0) {
          float pv = P0[nb + i - 1];
          if (pv > r) r = pv;
        }
        u[base + i] = r;
      }
    } else if (MODE == M_LSE) {
      LseAcc acc = {0.f, 0.f};
      for (int i = K - 1; i >= 0; --i) {
        acc = lse_push(acc, u[base + i], tau2);
        LseAcc r = acc;
        if (i > 0) r = lse_comb(acc, LseAcc{P0[nb + i - 1], P1[nb + i - 1]}, tau2);
        u[base + i] = fmaf(lg2f(r.s), p.mp.inv_tau2, r.m);
      }
    } else {
      SoftAcc acc = {0.f, 0.f, 0.f};
      for (int i = K - 1; i >= 0; --i) {
        acc = soft_push(acc, u[base + i], tau2);
        SoftAcc r = acc;
        if (i > 0) r = soft_comb(acc, SoftAcc{P0[nb + i - 1], P1[nb + i - 1], P2[nb + i - 1]}, tau2);
        u[base + i] = r.m + r.d / r.s;
        AX[base + i] = fmaf(lg2f(r.s), p.mp.inv_tau2, r.m);
      }
    }
  }
  __syncthreads();
  const long long tend = t0 + J < L ? t0 + J : L;
  const float padv = padv_sh;
  for (long long t = t0 + threadIdx.x; t < tend; t += blockDim.x) {
    int i = (int)(t - t0);
    int blk = i / K, off = i - blk * K;
    float v = (t < nvalid) ? p.sg * u[blk * Kp + off] : padv;
    if (p.canon) v = __fadd_rn(v, 0.f);
    p.out[row * L + t] = v;
    if (MODE == M_SOFT && t < nvalid) p.aux[row * L + t] = AX[blk * Kp + off];
  }
}

// ===========================================================================
// timed F / G — backward, LSE and softmax (window sum over the cotangent)
// ===========================================================================
// CTA owns child elements j in [j0, j0 + J); it needs outputs t in
// [j0 - b, j0 + J - 1 - a] (NB blocks of K).  h_t = (mu_t, g_t [, Bc]) with
//   LSE:  mu_t = M_t (u-space output);           g_child[j] = A e^{tau (u_j - mu)}
//   soft: mu_t = L_t (window LSE), c_t = M_t;     g_child[j] = e^{tau (u_j - mu)} (A (1 + tau (u_j - c)) - tau Bc)
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_bwd_smooth(const __grid_constant__ FGParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red_sh[32];
  __shared__ float padsum_sh;
  const int NB = p.NB, K = p.K, Kp = p.Kp;
  const long long row = blockIdx.y, L = p.L;
  const long long J = (long long)(NB - 1) * K;
  const long long j0 = (long long)blockIdx.x * J;
  const long long tb = j0 - p.b;
  const long long nvalid = L - p.b;
  const int nsm = NB * Kp;
  const int NW = (MODE == M_SOFT) ? 4 : 2;  // words per state
  float* H = sm;                 // NW arrays of nsm
  float* P = sm + NW * nsm;      // NW arrays of nsm
  const float tau2 = p.mp.tau2;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;

  {
    const int n = NB * K;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int blk = i / K, off = i - blk * K, pos = blk * Kp + off;
      long long t = tb + i;
      float g = 0.f;
      if (t >= 0 && t < nvalid) g = cot[t];
      if (MODE == M_LSE) {
        H[pos] = g != 0.f ? p.sg * outr[t] : 0.f;
        H[nsm + pos] = g;
      } else {
        if (g != 0.f) {
          H[pos] = p.aux_in[row * L + t];
          H[2 * nsm + pos] = 0.f;
          H[3 * nsm + pos] = p.sg * outr[t];
        } else {
          H[pos] = 0.f;
          H[2 * nsm + pos] = 0.f;
          H[3 * nsm + pos] = 0.f;
        }
        H[nsm + pos] = g;
      }
    }
  }
  // pad contribution: overrun outputs route their cotangent to c[L-1] (last pad)
  const bool own_last = p.pad_last && (L - 1 >= j0) && (L - 1 < j0 + J);
  if (own_last) {
    float s = 0.f;
    long long t_lo = nvalid > 0 ? nvalid : 0;
    for (long long t = t_lo + threadIdx.x; t < L; t += blockDim.x) s += cot[t];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red_sh[threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (own_last && threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red_sh[w];
    padsum_sh = s;
  }
  if (threadIdx.x < NB) {  // prefix scans
    const int base = threadIdx.x * Kp;
    if (MODE == M_LSE) {
      GLse a = {0.f, 0.f};
      for (int i = 0; i < K; ++i) {
        a = glse_comb(a, GLse{H[base + i], H[nsm + base + i]}, tau2);
        P[base + i] = a.mu;
        P[nsm + base + i] = a.A;
      }
    } else {
      GSoft a = {0.f, 0.f, 0.f, 0.f};
      for (int i = 0; i < K; ++i) {
        int q = base + i;
        a = gsoft_comb(a, GSoft{H[q], H[nsm + q], H[2 * nsm + q], H[3 * nsm + q]}, tau2);
        P[q] = a.mu;
        P[nsm + q] = a.A;
        P[2 * nsm + q] = a.Bc;
        P[3 * nsm + q] = a.c;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < NB - 1) {  // suffix walk + combine, result in place into H
    const int base = threadIdx.x * Kp, nb = base + Kp;
    if (MODE == M_LSE) {
      GLse acc = {0.f, 0.f};
      for (int i = K - 1; i >= 0; --i) {
        acc = glse_comb(GLse{H[base + i], H[nsm + base + i]}, acc, tau2);
        GLse r = acc;
        if (i > 0) r = glse_comb(acc, GLse{P[nb + i - 1], P[nsm + nb + i - 1]}, tau2);
        H[base + i] = r.mu;
        H[nsm + base + i] = r.A;
      }
    } else {
      GSoft acc = {0.f, 0.f, 0.f, 0.f};
      for (int i = K - 1; i >= 0; --i) {
        int q = base + i;
        acc = gsoft_comb(GSoft{H[q], H[nsm + q], H[2 * nsm + q], H[3 * nsm + q]}, acc, tau2);
        GSoft r = acc;
        if (i > 0) {
          int pq = nb + i - 1;
          r = gsoft_comb(acc, GSoft{P[pq], P[nsm + pq], P[2 * nsm + pq], P[3 * nsm + pq]}, tau2);
        }
        H[q] = r.mu;
        H[nsm + q] = r.A;
        H[2 * nsm + q] = r.Bc;
        H[3 * nsm + q] = r.c;
      }
    }
  }
  __syncthreads();
  const long long jend = j0 + J < L ? j0 + J : L;
  for (long long j = j0 + threadIdx.x; j < jend; j += blockDim.x) {
    int i = (int)(j - j0);
    int blk = i / K, off = i - blk * K, q = blk * Kp + off;
    float g = 0.f;
    float A = H[nsm + q];
    if (MODE == M_LSE) {
      if (A != 0.f) {
        float uj = p.sg * expr_eval<MODE>(p.child, row, j, p.mp);
        g = A * ex2f(tau2 * (uj - H[q]));
      }
    } else {
      float Bc = H[2 * nsm + q];
      if (A != 0.f || Bc != 0.f) {
        float uj = p.sg * expr_eval<MODE>(p.child, row, j, p.mp);
        float c = H[3 * nsm + q];
        g = ex2f(tau2 * (uj - H[q])) * (A * fmaf(p.mp.tau, uj - c, 1.f) - p.mp.tau * Bc);
      }
    }
    if (own_last && j == L - 1) g += padsum_sh;
    expr_vjp<MODE>(p.child, row, j, g, p.mp);
  }
}

// ===========================================================================
// timed F / G — backward, hard (recompute arg-max, scatter in shared memory)
// ===========================================================================
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_bwd_hard(const __grid_constant__ FGParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red_sh[32];
  __shared__ float padsum_sh;
  const int NB = p.NB, K = p.K, Kp = p.Kp;
  const int NBi = NB + 1;  // input blocks
  const long long row = blockIdx.y, L = p.L;
  const long long J = (long long)(NB - 1) * K;
  const long long j0 = (long long)blockIdx.x * J;
  const long long s0 = j0 - K + 1;  // first input index (start of window of t = j0 - b)
  const long long nvalid = L - p.b;
  const int nsm = NBi * Kp;
  float* u = sm;
  float* PV = sm + nsm;
  int* PI = reinterpret_cast<int*>(sm + 2 * nsm);
  float* G = sm + 3 * nsm;  // J accumulators
  const float* cot = p.cot + row * L;

  {
    const int n = NBi * K;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int blk = i / K, off = i - blk * K;
      long long idx = s0 + i;
      u[blk * Kp + off] =
          (idx >= 0 && idx < L) ? p.sg * expr_eval<MODE>(p.child, row, idx, p.mp) : -INFINITY;
    }
    for (int i = threadIdx.x; i < (int)J; i += blockDim.x) G[i] = 0.f;
  }
  const bool own_last = p.pad_last && (L - 1 >= j0) && (L - 1 < j0 + J);
  if (own_last) {
    float s = 0.f;
    long long t_lo = nvalid > 0 ? nvalid : 0;
    for (long long t = t_lo + threadIdx.x; t < L; t += blockDim.x) s += cot[t];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red_sh[threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (own_last && threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red_sh[w];
    padsum_sh = s;
  }
  if (threadIdx.x < NBi) {  // prefix (value, first arg-max)
    const int base = threadIdx.x * Kp;
    float bv = u[base];
    int bi = threadIdx.x * K;
    PV[base] = bv;
    PI[base] = bi;
    for (int i = 1; i < K; ++i) {
      float x = u[base + i];
      if (x > bv) {
        bv = x;
        bi = threadIdx.x * K + i;
      }
      PV[base + i] = bv;
      PI[base + i] = bi;
    }
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    const int qb = threadIdx.x;
    const int base = qb * Kp, nb = base + Kp;
    HardAcc acc = {-INFINITY, 0};
    for (int i = K - 1; i >= 0; --i) {
      float x = u[base + i];
      if (x >= acc.v) acc = {x, qb * K + i};  // walking backwards: the new element is earlier
      HardAcc r = acc;
      if (i > 0) {
        float pv = PV[nb + i - 1];
        if (pv > r.v) r = {pv, PI[nb + i - 1]};
      }
      long long s = s0 + (long long)qb * K + i;
      long long t = s - p.a;
      if (t >= 0 && t < nvalid) {
        float g = cot[t];
        long long jj = s0 + r.i;
        if (g != 0.f && jj >= j0 && jj < j0 + J) atomicAdd(&G[jj - j0], g);
      }
    }
  }
  __syncthreads();
  const long long jend = j0 + J < L ? j0 + J : L;
  for (long long j = j0 + threadIdx.x; j < jend; j += blockDim.x) {
    float g = G[j - j0];
    if (own_last && j == L - 1) g += padsum_sh;
    expr_vjp<MODE>(p.child, row, j, g, p.mp);
  }
}

// ===========================================================================
// brute-force timed F / G (tiny or huge windows): direct O(K) per output
// ===========================================================================
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_fwd_direct(const __grid_constant__ FGParams p) {
  const long long row = blockIdx.y, L = p.L;
  const long long nvalid = L - p.b;
  const float tau2 = p.mp.tau2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < L;
       t += (long long)gridDim.x * blockDim.x) {
    float v;
    if (t < nvalid) {
      if (MODE == M_HARD) {
        float m = -INFINITY;
        for (int k = 0; k < p.K; ++k) {
          float x = p.sg * expr_eval<MODE>(p.child, row, t + p.a + k, p.mp);
          if (x > m) m = x;
        }
        v = p.sg * m;
      } else if (MODE == M_LSE) {
        LseAcc a = {0.f, 0.f};
        for (int k = 0; k < p.K; ++k)
          a = lse_push(a, p.sg * expr_eval<MODE>(p.child, row, t + p.a + k, p.mp), tau2);
        v = p.sg * fmaf(lg2f(a.s), p.mp.inv_tau2, a.m);
      } else {
        SoftAcc a = {0.f, 0.f, 0.f};
        for (int k = 0; k < p.K; ++k)
          a = soft_push(a, p.sg * expr_eval<MODE>(p.child, row, t + p.a + k, p.mp), tau2);
        v = p.sg * (a.m + a.d / a.s);
        p.aux[row * L + t] = fmaf(lg2f(a.s), p.mp.inv_tau2, a.m);
      }
    } else {
      v = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
    }
    if (p.canon) v = __fadd_rn(v, 0.f);
    p.out[row * L + t] = v;
  }
}

// backward: cotangent of the child into gbuf (atomics), then a pointwise VJP
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_bwd_direct(const __grid_constant__ FGParams p) {
  const long long row = blockIdx.y, L = p.L;
  const long long nvalid = L - p.b;
  const float tau2 = p.mp.tau2;
  float* gb = p.gbuf + row * L;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < L;
       t += (long long)gridDim.x * blockDim.x) {
    float g = p.cot[row * L + t];
    if (g == 0.f) continue;
    if (t >= nvalid) {
      if (p.pad_last) atomicAdd(gb + (L - 1), g);
      continue;
    }
    if (MODE == M_HARD) {
      float m = -INFINITY;
      int am = 0;
      for (int k = 0; k < p.K; ++k) {
        float x = p.sg * expr_eval<MODE>(p.child, row, t + p.a + k, p.mp);
        if (x > m) {
          m = x;
          am = k;
        }
      }
      atomicAdd(gb + t + p.a + am, g);
    } else {
      float M = p.sg * p.out_in[row * L + t];
      float Lt = (MODE == M_SOFT) ? p.aux_in[row * L + t] : M;
      for (int k = 0; k < p.K; ++k) {
        float x = p.sg * expr_eval<MODE>(p.child, row, t + p.a + k, p.mp);
        float w = ex2f(tau2 * (x - Lt));
        if (MODE == M_SOFT) w *= fmaf(p.mp.tau, x - M, 1.f);
        atomicAdd(gb + t + p.a + k, g * w);
      }
    }
  }
}

// ===========================================================================
// launchers for timed F / G
// ===========================================================================
static int odd_stride(int K) { return K | 1; }

template <typename KernT>
static cudaError_t set_smem(KernT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static const size_t kSmemBudget = 72 * 1024;   // per CTA target (3 CTAs / SM)
static const size_t kSmemMax = 200 * 1024;

// words per element of each kernel's shared layout
static int fwd_words(int mode) { return mode == M_SOFT ? 5 : 3; }
static int bwd_words(int mode) { return mode == M_HARD ? 4 : (mode == M_SOFT ? 8 : 4); }

static int pick_nb(int K, int words, int extra_blocks) {
  int Kp = odd_stride(K);
  long long per_block = (long long)words * Kp * 4;
  long long nb = (long long)(kSmemBudget / per_block) - extra_blocks;
  if (nb > 256 - extra_blocks) nb = 256 - extra_blocks;
  if (nb < 2) nb = 2;
  return (int)nb;
}

static bool use_direct(int K, int mode) {
  if (K < 4) return true;
  int Kp = odd_stride(K);
  // two blocks (+1 input block for hard backward) must fit
  size_t need = (size_t)bwd_words(mode) * 3 * Kp * 4;
  return need > kSmemMax;
}

cudaError_t launch_fg_timed_fwd(int mode, FGParams& p, cudaStream_t st) {
  if (use_direct(p.K, mode)) {
    dim3 grid((unsigned)((p.L + 255) / 256), (unsigned)p.B);
    if (mode == M_HARD) k_fg_timed_fwd_direct<M_HARD><<<grid, 256, 0, st>>>(p);
    else if (mode == M_LSE) k_fg_timed_fwd_direct<M_LSE><<<grid, 256, 0, st>>>(p);
    else k_fg_timed_fwd_direct<M_SOFT><<<grid, 256, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  p.Kp = odd_stride(p.K);
  p.NB = pick_nb(p.K, fwd_words(mode), 0);
  long long J = (long long)(p.NB - 1) * p.K;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  int threads = ((p.NB + 31) / 32) * 32;
  if (threads < 128) threads = 128;
  if (threads > 256) threads = 256;
  size_t smem = (size_t)fwd_words(mode) * p.NB * p.Kp * 4;
  cudaError_t e;
  if (mode == M_HARD) {
    if ((e = set_smem(k_fg_timed_fwd<M_HARD>, smem)) != cudaSuccess) return e;
    k_fg_timed_fwd<M_HARD><<<grid, threads, smem, st>>>(p);
  } else if (mode == M_LSE) {
    if ((e = set_smem(k_fg_timed_fwd<M_LSE>, smem)) != cudaSuccess) return e;
    k_fg_timed_fwd<M_LSE><<<grid, threads, smem, st>>>(p);
  } else {
    if ((e = set_smem(k_fg_timed_fwd<M_SOFT>, smem)) != cudaSuccess) return e;
    k_fg_timed_fwd<M_SOFT><<<grid, threads, smem, st>>>(p);
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fg_timed_bwd(int mode, FGParams& p, cudaStream_t st) {
  cudaError_t e;
  if (use_direct(p.K, mode)) {
    if ((e = cudaMemsetAsync(p.gbuf, 0, sizeof(float) * p.B * p.L, st)) != cudaSuccess) return e;
    dim3 grid((unsigned)((p.L + 255) / 256), (unsigned)p.B);
    if (mode == M_HARD) k_fg_timed_bwd_direct<M_HARD><<<grid, 256, 0, st>>>(p);
    else if (mode == M_LSE) k_fg_timed_bwd_direct<M_LSE><<<grid, 256, 0, st>>>(p);
    else k_fg_timed_bwd_direct<M_SOFT><<<grid, 256, 0, st>>>(p);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_pointwise_vjp(mode, p, p.gbuf, st);
  }
  p.Kp = odd_stride(p.K);
  const int words = bwd_words(mode);
  if (mode == M_HARD) {
    // (NB+1) input blocks * 3 words + J accumulators
    int nb = pick_nb(p.K, 4, 1);
    p.NB = nb;
    size_t smem = (size_t)3 * (nb + 1) * p.Kp * 4 + (size_t)(nb - 1) * p.K * 4;
    long long J = (long long)(nb - 1) * p.K;
    dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
    int threads = ((nb + 1 + 31) / 32) * 32;
    if (threads < 128) threads = 128;
    if (threads > 256) threads = 256;
    if ((e = set_smem(k_fg_timed_bwd_hard<M_HARD>, smem)) != cudaSuccess) return e;
    k_fg_timed_bwd_hard<M_HARD><<<grid, threads, smem, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  int nb = pick_nb(p.K, words, 0);
  p.NB = nb;
  size_t smem = (size_t)words * nb * p.Kp * 4;
  long long J = (long long)(nb - 1) * p.K;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  int threads = ((nb + 31) / 32) * 32;
  if (threads < 128) threads = 128;
  if (threads > 256) threads = 256;
  if (mode == M_LSE) {
    if ((e = set_smem(k_fg_timed_bwd_smooth<M_LSE>, smem)) != cudaSuccess) return e;
    k_fg_timed_bwd_smooth<M_LSE><<<grid, threads, smem, st>>>(p);
  } else {
    if ((e = set_smem(k_fg_timed_bwd_smooth<M_SOFT>, smem)) != cudaSuccess) return e;
    k_fg_timed_bwd_smooth<M_SOFT><<<grid, threads, smem, st>>>(p);
  }
  count_launch();
  return cudaGetLastError();
}

// ===========================================================================
// untimed F / G: one CTA per row, chunks of UT_CH samples, block scans
// ===========================================================================
constexpr int UT_T = 256;          // threads
constexpr int UT_E = 8;            // samples per thread per chunk
constexpr int UT_CH = UT_T * UT_E;
constexpr int UT_S = UT_E + 1;     // padded per-thread stride in shared memory

__device__ __forceinline__ int upos(int k) { return (k >> 3) * UT_S + (k & 7); }

// block-wide inclusive scan over per-thread states in shared memory.
// SUFFIX: x_i <- x_i (+) x_{i+1} (+) ...   ; PREFIX: x_i <- ... (+) x_{i-1} (+) x_i
template <typename S, typename F, bool SUFFIX>
__device__ __forceinline__ void block_scan(S* buf, F comb) {
  const int i = threadIdx.x;
  for (int off = 1; off < UT_T; off <<= 1) {
    S x = buf[i];
    if (SUFFIX) {
      if (i + off < UT_T) x = comb(x, buf[i + off]);
    } else {
      if (i >= off) x = comb(buf[i - off], x);
    }
    __syncthreads();
    buf[i] = x;
    __syncthreads();
  }
}

template <int MODE>
__global__ void __launch_bounds__(UT_T) k_fg_untimed_fwd(const __grid_constant__ FGParams p) {
  __shared__ float u[UT_T * UT_S];
  __shared__ float ax[(MODE == M_SOFT) ? UT_T * UT_S : 1];
  const long long row = blockIdx.x, L = p.L;
  const float tau2 = p.mp.tau2;
  const int tid = threadIdx.x;
  if (MODE == M_HARD) {
    __shared__ float sb[UT_T];
    float carry = -INFINITY;
    auto comb = [](float e, float l) { return l > e ? l : e; };
    for (long long c0 = ((L - 1) / UT_CH) * UT_CH; c0 >= 0; c0 -= UT_CH) {
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        u[upos(k)] = t < L ? p.sg * expr_eval<MODE>(p.child, row, t, p.mp) : -INFINITY;
      }
      __syncthreads();
      float agg = -INFINITY;
      for (int e = UT_E - 1; e >= 0; --e) agg = comb(u[tid * UT_S + e], agg);
      sb[tid] = agg;
      __syncthreads();
      block_scan<float, decltype(comb), true>(sb, comb);
      float acc = comb(tid + 1 < UT_T ? sb[tid + 1] : -INFINITY, carry);
      for (int e = UT_E - 1; e >= 0; --e) {
        acc = comb(u[tid * UT_S + e], acc);
        u[tid * UT_S + e] = acc;
      }
      float nc = comb(sb[0], carry);
      __syncthreads();
      carry = nc;
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        if (t < L) p.out[row * L + t] = p.sg * u[upos(k)];
      }
      __syncthreads();
    }
  } else if (MODE == M_LSE) {
    __shared__ LseAcc sb[UT_T];
    LseAcc carry = {0.f, 0.f};
    auto comb = [tau2](LseAcc e, LseAcc l) { return lse_comb(e, l, tau2); };
    for (long long c0 = ((L - 1) / UT_CH) * UT_CH; c0 >= 0; c0 -= UT_CH) {
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        u[upos(k)] = t < L ? p.sg * expr_eval<MODE>(p.child, row, t, p.mp) : 0.f;
      }
      __syncthreads();
      LseAcc agg = {0.f, 0.f};
      for (int e = UT_E - 1; e >= 0; --e)
        if (c0 + tid * UT_E + e < L) agg = lse_push(agg, u[tid * UT_S + e], tau2);
      sb[tid] = agg;
      __syncthreads();
      block_scan<LseAcc, decltype(comb), true>(sb, comb);
      LseAcc acc = comb(tid + 1 < UT_T ? sb[tid + 1] : LseAcc{0.f, 0.f}, carry);
      for (int e = UT_E - 1; e >= 0; --e) {
        if (c0 + tid * UT_E + e >= L) continue;
        acc = lse_push(acc, u[tid * UT_S + e], tau2);
        u[tid * UT_S + e] = fmaf(lg2f(acc.s), p.mp.inv_tau2, acc.m);
      }
      LseAcc nc = comb(sb[0], carry);
      __syncthreads();
      carry = nc;
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        if (t < L) p.out[row * L + t] = p.sg * u[upos(k)];
      }
      __syncthreads();
    }
  } else {
    __shared__ SoftAcc sb[UT_T];
    SoftAcc carry = {0.f, 0.f, 0.f};
    auto comb = [tau2](SoftAcc e, SoftAcc l) { return soft_comb(e, l, tau2); };
    for (long long c0 = ((L - 1) / UT_CH) * UT_CH; c0 >= 0; c0 -= UT_CH) {
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        u[upos(k)] = t < L ? p.sg * expr_eval<MODE>(p.child, row, t, p.mp) : 0.f;
      }
      __syncthreads();
      SoftAcc agg = {0.f, 0.f, 0.f};
      for (int e = UT_E - 1; e >= 0; --e)
        if (c0 + tid * UT_E + e < L) agg = soft_push(agg, u[tid * UT_S + e], tau2);
      sb[tid] = agg;
      __syncthreads();
      block_scan<SoftAcc, decltype(comb), true>(sb, comb);
      SoftAcc acc = comb(tid + 1 < UT_T ? sb[tid + 1] : SoftAcc{0.f, 0.f, 0.f}, carry);
      for (int e = UT_E - 1; e >= 0; --e) {
        if (c0 + tid * UT_E + e >= L) continue;
        acc = soft_push(acc, u[tid * UT_S + e], tau2);
        u[tid * UT_S + e] = acc.m + acc.d / acc.s;
        ax[tid * UT_S + e] = fmaf(lg2f(acc.s), p.mp.inv_tau2, acc.m);
      }
      SoftAcc nc = comb(sb[0], carry);
      __syncthreads();
      carry = nc;
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        if (t < L) {
          p.out[row * L + t] = p.sg * u[upos(k)];
          p.aux[row * L + t] = ax[upos(k)];
        }
      }
      __syncthreads();
    }
  }
}

// LSE / softmax backward: prefix scan over t of the cotangent states (fused VJP)
template <int MODE>
__global__ void __launch_bounds__(UT_T) k_fg_untimed_bwd_smooth(const __grid_constant__ FGParams p) {
  constexpr int NW = (MODE == M_SOFT) ? 4 : 2;
  __shared__ float h[NW][UT_T * UT_S];
  const long long row = blockIdx.x, L = p.L;
  const float tau2 = p.mp.tau2;
  const int tid = threadIdx.x;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  if (MODE == M_LSE) {
    __shared__ GLse sb[UT_T];
    GLse carry = {0.f, 0.f};
    auto comb = [tau2](GLse x, GLse y) { return glse_comb(x, y, tau2); };
    for (long long c0 = 0; c0 < L; c0 += UT_CH) {
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        float g = t < L ? cot[t] : 0.f;
        h[0][upos(k)] = g != 0.f ? p.sg * outr[t] : 0.f;
        h[1][upos(k)] = g;
      }
      __syncthreads();
      GLse agg = {0.f, 0.f};
      for (int e = 0; e < UT_E; ++e) agg = comb(agg, GLse{h[0][tid * UT_S + e], h[1][tid * UT_S + e]});
      sb[tid] = agg;
      __syncthreads();
      block_scan<GLse, decltype(comb), false>(sb, comb);
      GLse acc = comb(carry, tid > 0 ? sb[tid - 1] : GLse{0.f, 0.f});
      for (int e = 0; e < UT_E; ++e) {
        acc = comb(acc, GLse{h[0][tid * UT_S + e], h[1][tid * UT_S + e]});
        h[0][tid * UT_S + e] = acc.mu;
        h[1][tid * UT_S + e] = acc.A;
      }
      GLse nc = comb(carry, sb[UT_T - 1]);
      __syncthreads();
      carry = nc;
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        if (t >= L) continue;
        float A = h[1][upos(k)];
        float g = 0.f;
        if (A != 0.f) {
          float uj = p.sg * expr_eval<MODE>(p.child, row, t, p.mp);
          g = A * ex2f(tau2 * (uj - h[0][upos(k)]));
        }
        expr_vjp<MODE>(p.child, row, t, g, p.mp);
      }
      __syncthreads();
    }
  } else {
    __shared__ GSoft sb[UT_T];
    GSoft carry = {0.f, 0.f, 0.f, 0.f};
    auto comb = [tau2](GSoft x, GSoft y) { return gsoft_comb(x, y, tau2); };
    for (long long c0 = 0; c0 < L; c0 += UT_CH) {
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        float g = t < L ? cot[t] : 0.f;
        bool on = g != 0.f;
        h[0][upos(k)] = on ? p.aux_in[row * L + t] : 0.f;
        h[1][upos(k)] = g;
        h[2][upos(k)] = 0.f;
        h[3][upos(k)] = on ? p.sg * outr[t] : 0.f;
      }
      __syncthreads();
      GSoft agg = {0.f, 0.f, 0.f, 0.f};
      for (int e = 0; e < UT_E; ++e) {
        int q = tid * UT_S + e;
        agg = comb(agg, GSoft{h[0][q], h[1][q], h[2][q], h[3][q]});
      }
      sb[tid] = agg;
      __syncthreads();
      block_scan<GSoft, decltype(comb), false>(sb, comb);
      GSoft acc = comb(carry, tid > 0 ? sb[tid - 1] : GSoft{0.f, 0.f, 0.f, 0.f});
      for (int e = 0; e < UT_E; ++e) {
        int q = tid * UT_S + e;
        acc = comb(acc, GSoft{h[0][q], h[1][q], h[2][q], h[3][q]});
        h[0][q] = acc.mu;
        h[1][q] = acc.A;
        h[2][q] = acc.Bc;
        h[3][q] = acc.c;
      }
      GSoft nc = comb(carry, sb[UT_T - 1]);
      __syncthreads();
      carry = nc;
      for (int k = tid; k < UT_CH; k += UT_T) {
        long long t = c0 + k;
        if (t >= L) continue;
        int q = upos(k);
        float A = h[1][q], Bc = h[2][q];
        float g = 0.f;
        if (A != 0.f || Bc != 0.f) {
          float uj = p.sg * expr_eval<MODE>(p.child, row, t, p.mp);
          g = ex2f(tau2 * (uj - h[0][q])) * (A * fmaf(p.mp.tau, uj - h[3][q], 1.f) - p.mp.tau * Bc);
        }
        expr_vjp<MODE>(p.child, row, t, g, p.mp);
      }
      __syncthreads();
    }
  }
}

// hard backward: recompute the suffix first-arg-max, scatter g_t into gbuf
template <int MODE>
__global__ void __launch_bounds__(UT_T) k_fg_untimed_bwd_hard(const __grid_constant__ FGParams p) {
  __shared__ float u[UT_T * UT_S];
  __shared__ HardAcc sb[UT_T];
  const long long row = blockIdx.x, L = p.L;
  const int tid = threadIdx.x;
  const float* cot = p.cot + row * L;
  float* gb = p.gbuf + row * L;
  auto comb = [](HardAcc e, HardAcc l) { return hard_comb(e, l); };
  HardAcc carry = {-INFINITY, 0x7fffffff};
  for (long long c0 = ((L - 1) / UT_CH) * UT_CH; c0 >= 0; c0 -= UT_CH) {
    for (int k = tid; k < UT_CH; k += UT_T) {
      long long t = c0 + k;
      u[upos(k)] = t < L ? p.sg * expr_eval<MODE>(p.child, row, t, p.mp) : -INFINITY;
    }
    __syncthreads();
    HardAcc agg = {-INFINITY, 0x7fffffff};
    for (int e = UT_E - 1; e >= 0; --e) {
      long long t = c0 + tid * UT_E + e;
      if (t < L) agg = comb(HardAcc{u[tid * UT_S + e], (int)t}, agg);
    }
    sb[tid] = agg;
    __syncthreads();
    block_scan<HardAcc, decltype(comb), true>(sb, comb);
    HardAcc acc = comb(tid + 1 < UT_T ? sb[tid + 1] : HardAcc{-INFINITY, 0x7fffffff}, carry);
    // walk backwards; arg-max is non-decreasing in t, so equal targets form runs
    int run_idx = -1;
    float run_sum = 0.f;
    for (int e = UT_E - 1; e >= 0; --e) {
      long long t = c0 + tid * UT_E + e;
      if (t >= L) continue;
      acc = comb(HardAcc{u[tid * UT_S + e], (int)t}, acc);
      float g = cot[t];
      if (acc.i != run_idx) {
        if (run_idx >= 0 && run_sum != 0.f) atomicAdd(gb + run_idx, run_sum);
        run_idx = acc.i;
        run_sum = 0.f;
      }
      run_sum += g;
    }
    if (run_idx >= 0 && run_sum != 0.f) atomicAdd(gb + run_idx, run_sum);
    HardAcc nc = comb(sb[0], carry);
    __syncthreads();
    carry = nc;
  }
}

cudaError_t launch_fg_untimed_fwd(int mode, FGParams& p, cudaStream_t st) {
  dim3 grid((unsigned)p.B);
  if (mode == M_HARD) k_fg_untimed_fwd<M_HARD><<<grid, UT_T, 0, st>>>(p);
  else if (mode == M_LSE) k_fg_untimed_fwd<M_LSE><<<grid, UT_T, 0, st>>>(p);
  else k_fg_untimed_fwd<M_SOFT><<<grid, UT_T, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fg_untimed_bwd(int mode, FGParams& p, cudaStream_t st) {
  dim3 grid((unsigned)p.B);
  if (mode == M_HARD) {
    cudaError_t e = cudaMemsetAsync(p.gbuf, 0, sizeof(float) * p.B * p.L, st);
    if (e != cudaSuccess) return e;
    k_fg_untimed_bwd_hard<M_HARD><<<grid, UT_T, 0, st>>>(p);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_pointwise_vjp(mode, p, p.gbuf, st);
  }
  if (mode == M_LSE) k_fg_untimed_bwd_smooth<M_LSE><<<grid, UT_T, 0, st>>>(p);
  else k_fg_untimed_bwd_smooth<M_SOFT><<<grid, UT_T, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
