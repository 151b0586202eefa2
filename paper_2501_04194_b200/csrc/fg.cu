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
#include <cstdlib>

#include "kernels.cuh"

namespace stlg {

// ===========================================================================
// pointwise expression kernels (root formula / materialised sub-formulas)
// ===========================================================================
// grid (t tiles of 1024, rows): 4 samples per thread, 32-bit time index, no division
constexpr int PW_T = 256, PW_E = 4, PW_N = PW_T * PW_E;

// NS > 0: expressions of exactly NS steps in registers (expr_eval_n); 0: the generic walk
template <int MODE, int NS>
__device__ __forceinline__ float pw_eval(const DExpr& e, long long row, int t, const ModeP& mp) {
  if (NS > 0) return expr_eval_n<MODE, (NS > 0 ? NS : 1)>(e, row, t, mp);
  return expr_eval<MODE>(e, row, t, mp);
}
template <int MODE, int NS>
__device__ __forceinline__ void pw_vjp(const DExpr& e, long long row, int t, float g, const ModeP& mp) {
  if (NS > 0) expr_vjp_n<MODE, (NS > 0 ? NS : 1)>(e, row, t, g, mp);
  else expr_vjp<MODE>(e, row, t, g, mp);
}

// UNIT: every leaf is a constant, trace or affine predicate over unit-stride planes
// (pw_unit): the leaves are resolved once per row (RowLeaves)
template <int MODE, int NS, bool UNIT>
__global__ void __launch_bounds__(PW_T) k_pointwise_fwd(const __grid_constant__ FGParams p) {
  const int L = (int)p.L;
  for (long long row = blockIdx.y; row < p.B; row += gridDim.y) {
    float* out = p.out + row * L;
    if constexpr (UNIT && NS > 0) {
      const RowLeaves<NS> R(p.child, row, false);
#pragma unroll
      for (int e = 0; e < PW_E; ++e) {
        const int t = blockIdx.x * PW_N + e * PW_T + threadIdx.x;
        if (t < L) out[t] = expr_eval_rn<MODE, NS>(p.child, R, t, p.mp);
      }
    } else {
#pragma unroll
      for (int e = 0; e < PW_E; ++e) {
        const int t = blockIdx.x * PW_N + e * PW_T + threadIdx.x;
        if (t < L) out[t] = pw_eval<MODE, NS>(p.child, row, t, p.mp);
      }
    }
  }
}

template <int MODE, int NS, bool UNIT>
__global__ void __launch_bounds__(PW_T) k_pointwise_vjp(const __grid_constant__ FGParams p,
                                                       const float* __restrict__ g) {
  const int L = (int)p.L;
  for (long long row = blockIdx.y; row < p.B; row += gridDim.y) {
    const float* gr = g + row * L;
    if constexpr (UNIT && NS > 0) {
      const RowLeaves<NS> R(p.child, row, true);
#pragma unroll
      for (int e = 0; e < PW_E; ++e) {
        const int t = blockIdx.x * PW_N + e * PW_T + threadIdx.x;
        if (t < L) expr_vjp_rn<MODE, NS>(p.child, R, t, gr[t], p.mp);
      }
    } else {
#pragma unroll
      for (int e = 0; e < PW_E; ++e) {
        const int t = blockIdx.x * PW_N + e * PW_T + threadIdx.x;
        if (t < L) pw_vjp<MODE, NS>(p.child, row, t, gr[t], p.mp);
      }
    }
  }
}

// host: every leaf a constant / trace / affine predicate with unit element strides
static bool pw_unit(const DExpr& e) {
  for (int i = 0; i < e.n_leaf; ++i) {
    const DLeaf& L = e.leaf[i];
    if (L.kind == LEAF_CONST) continue;
    if (L.kind != LEAF_SRC && L.kind != LEAF_AFFINE) return false;
    if (e.src[L.src].es != 1) return false;
    if (e.dst[L.src].p != nullptr && e.dst[L.src].es != 1) return false;
  }
  return true;
}

// Binary root over two trace / affine leaves (And / Or of two sub-formulas — the usual
// pointwise root): both leaves resolved into registers once per thread.
struct PwLeaf {
  const float* p;
  long long es;
  float* gp;
  long long ges;
  int gst, src;  // src: 1 trace (LEAF_SRC), 0 affine
  float s_in, c, s_out;
  __device__ __forceinline__ PwLeaf(const DExpr& e, const DLeaf& L, long long row) {
    const DSrc& sr = e.src[L.src];
    p = sr.p + row * sr.rs;
    es = sr.es;
    const DDst& d = e.dst[L.src];
    gp = d.p ? d.p + row * d.rs : nullptr;
    ges = d.es;
    gst = L.st1;
    src = L.kind == LEAF_SRC;
    s_in = L.s_in;
    c = L.c;
    s_out = L.s_out;
  }
  __device__ __forceinline__ float value(long long j) const { return apply(raw(j)); }
  // the load and the transform apart: a thread issues all its loads before the first store
  // (the output may alias nothing the compiler can prove, so it would not hoist them)
  __device__ __forceinline__ float raw(long long j) const { return __ldg(p + j * es); }
  __device__ __forceinline__ float apply(float x) const { return src ? s_out * x : s_out * __fadd_rn(s_in * x, c); }
  __device__ __forceinline__ void grad(long long j, float g) const {
    if (gp == nullptr || (g == 0.f && !gst)) return;
    const float v = src ? g * s_out : g * s_out * s_in;
    float* q = gp + j * ges;
    if (gst) *q = v;
    else *q += v;
  }
};

template <int MODE>
__global__ void __launch_bounds__(PW_T) k_pointwise2_fwd(const __grid_constant__ FGParams p) {
  const int L = (int)p.L;
  const DExpr& e = p.child;
  const float sg = e.step[2].op == ST_MAX ? 1.f : -1.f;
  for (long long row = blockIdx.y; row < p.B; row += gridDim.y) {
    const PwLeaf a(e, e.leaf[e.step[0].a], row), b(e, e.leaf[e.step[1].a], row);
    float* out = p.out + row * L;
    float xa[PW_E], xb[PW_E];
#pragma unroll
    for (int k = 0; k < PW_E; ++k) {
      const int t = blockIdx.x * PW_N + k * PW_T + threadIdx.x;
      const int tc = t < L ? t : L - 1;
      xa[k] = a.raw(tc);
      xb[k] = b.raw(tc);
    }
#pragma unroll
    for (int k = 0; k < PW_E; ++k) {
      const int t = blockIdx.x * PW_N + k * PW_T + threadIdx.x;
      if (t < L) {
        float w1, w2;
        out[t] = pair_red<MODE>(a.apply(xa[k]), b.apply(xb[k]), sg, p.mp, w1, w2);
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(PW_T) k_pointwise2_vjp(const __grid_constant__ FGParams p,
                                                        const float* __restrict__ g) {
  const int L = (int)p.L;
  const DExpr& e = p.child;
  const float sg = e.step[2].op == ST_MAX ? 1.f : -1.f;
  for (long long row = blockIdx.y; row < p.B; row += gridDim.y) {
    const PwLeaf a(e, e.leaf[e.step[0].a], row), b(e, e.leaf[e.step[1].a], row);
    const float* gr = g + row * L;
    float xa[PW_E], xb[PW_E], xg[PW_E];
#pragma unroll
    for (int k = 0; k < PW_E; ++k) {
      const int t = blockIdx.x * PW_N + k * PW_T + threadIdx.x;
      const int tc = t < L ? t : L - 1;
      xa[k] = a.raw(tc);
      xb[k] = b.raw(tc);
      xg[k] = gr[tc];
    }
#pragma unroll
    for (int k = 0; k < PW_E; ++k) {
      const int t = blockIdx.x * PW_N + k * PW_T + threadIdx.x;
      if (t < L) {
        float w1, w2;
        pair_red<MODE>(a.apply(xa[k]), b.apply(xb[k]), sg, p.mp, w1, w2);
        const float gv = xg[k];
        b.grad(t, 0.f + gv * w2);  // expr_vjp order (the later step first) and its 0 + adj
        a.grad(t, 0.f + gv * w1);
      }
    }
  }
}

static bool pw_binary(const DExpr& e) {
  if (e.n_step != 3 || e.step[0].op != ST_LEAF || e.step[1].op != ST_LEAF || e.step[2].op == ST_LEAF ||
      e.step[2].a != 0 || e.step[2].b != 1)
    return false;
  const DLeaf &l0 = e.leaf[e.step[0].a], &l1 = e.leaf[e.step[1].a];
  auto fast = [](const DLeaf& L) { return L.kind == LEAF_SRC || L.kind == LEAF_AFFINE; };
  return fast(l0) && fast(l1);
}

#define PW_DISPATCH(NSV, ...)                                    \
  switch (NSV) {                                                 \
    case 1: { constexpr int NS = 1; __VA_ARGS__; } break;        \
    case 3: { constexpr int NS = 3; __VA_ARGS__; } break;        \
    case 5: { constexpr int NS = 5; __VA_ARGS__; } break;        \
    case 7: { constexpr int NS = 7; __VA_ARGS__; } break;        \
    default: { constexpr int NS = 0; __VA_ARGS__; } break;       \
  }

static dim3 pw_grid(const FGParams& p) {
  return dim3((unsigned)((p.L + PW_N - 1) / PW_N), (unsigned)(p.B < 65535 ? p.B : 65535));
}

__global__ void k_fill_strided(float* p, long long B, long long T, long long rs, long long es,
                               float v) {
  const long long n = B * T;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long b = i / T, t = i - b * T;
    p[b * rs + t * es] = v;
  }
}

static int grid_for(long long n, int threads);

cudaError_t launch_fill_strided(float* p, long long B, long long T, long long rs, long long es,
                                float v, cudaStream_t st) {
  k_fill_strided<<<grid_for(B * T, 256), 256, 0, st>>>(p, B, T, rs, es, v);
  count_launch();
  return cudaGetLastError();
}

static int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  long long cap = 148LL * 16;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

cudaError_t launch_pointwise_fwd(int mode, const FGParams& p, cudaStream_t st) {
  const dim3 grid = pw_grid(p);
  if (pw_binary(p.child)) {
    if (mode == M_HARD) k_pointwise2_fwd<M_HARD><<<grid, PW_T, 0, st>>>(p);
    else if (mode == M_LSE) k_pointwise2_fwd<M_LSE><<<grid, PW_T, 0, st>>>(p);
    else k_pointwise2_fwd<M_SOFT><<<grid, PW_T, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  if (pw_unit(p.child)) {
    PW_DISPATCH(p.child.n_step,
                if (mode == M_HARD) k_pointwise_fwd<M_HARD, NS, true><<<grid, PW_T, 0, st>>>(p);
                else if (mode == M_LSE) k_pointwise_fwd<M_LSE, NS, true><<<grid, PW_T, 0, st>>>(p);
                else k_pointwise_fwd<M_SOFT, NS, true><<<grid, PW_T, 0, st>>>(p))
  } else {
    PW_DISPATCH(p.child.n_step,
                if (mode == M_HARD) k_pointwise_fwd<M_HARD, NS, false><<<grid, PW_T, 0, st>>>(p);
                else if (mode == M_LSE) k_pointwise_fwd<M_LSE, NS, false><<<grid, PW_T, 0, st>>>(p);
                else k_pointwise_fwd<M_SOFT, NS, false><<<grid, PW_T, 0, st>>>(p))
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pointwise_vjp(int mode, const FGParams& p, const float* g, cudaStream_t st) {
  const dim3 grid = pw_grid(p);
  if (pw_binary(p.child)) {
    if (mode == M_HARD) k_pointwise2_vjp<M_HARD><<<grid, PW_T, 0, st>>>(p, g);
    else if (mode == M_LSE) k_pointwise2_vjp<M_LSE><<<grid, PW_T, 0, st>>>(p, g);
    else k_pointwise2_vjp<M_SOFT><<<grid, PW_T, 0, st>>>(p, g);
    count_launch();
    return cudaGetLastError();
  }
  if (pw_unit(p.child)) {
    PW_DISPATCH(p.child.n_step,
                if (mode == M_HARD) k_pointwise_vjp<M_HARD, NS, true><<<grid, PW_T, 0, st>>>(p, g);
                else if (mode == M_LSE) k_pointwise_vjp<M_LSE, NS, true><<<grid, PW_T, 0, st>>>(p, g);
                else k_pointwise_vjp<M_SOFT, NS, true><<<grid, PW_T, 0, st>>>(p, g))
  } else {
    PW_DISPATCH(p.child.n_step,
                if (mode == M_HARD) k_pointwise_vjp<M_HARD, NS, false><<<grid, PW_T, 0, st>>>(p, g);
                else if (mode == M_LSE) k_pointwise_vjp<M_LSE, NS, false><<<grid, PW_T, 0, st>>>(p, g);
                else k_pointwise_vjp<M_SOFT, NS, false><<<grid, PW_T, 0, st>>>(p, g))
  }
  count_launch();
  return cudaGetLastError();
}

// ===========================================================================
// timed F / G — forward (vHGW)
// ===========================================================================
// Shared layout: NB blocks of K samples, row stride Kp = K | 1 (odd, so the
// per-thread block walks are bank-conflict free); flat index i of the tile
// lives at i + (i / K) * (Kp - K):
//   U  child in max space; overwritten in place by the outputs
//   P1 prefix state: hard = running max; lse = log-domain prefix LSE;
//      soft = prefix softmax value M
//   P2 soft: prefix LSE L
//   AX soft: window LSE (aux output for the backward)
// Loads / stores are flat and coalesced (4 independent loads in flight per
// thread); the scans run one thread per block.
constexpr int FG_THREADS = 256;

template <int MODE, int EK>
__global__ void __launch_bounds__(FG_THREADS) k_fgt_fwd(const __grid_constant__ FGParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float padv_sh;
  const int NB = p.NB, K = p.K, Kp = p.Kp, dK = Kp - K;
  const int nsm = NB * Kp;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = (NB - 1) * K;
  const int t0 = blockIdx.x * J;
  const int nvalid = p.padmode ? L : L - p.b;  // padded windows: every output reduces a window
  const int s0 = t0 + p.a;
  const float invK = 1.f / (float)K;
  float* U = sm;
  float* P1 = sm + nsm;
  float* P2 = sm + 2 * nsm;
  float* AX = sm + 3 * nsm;
  const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2, sg = p.sg;
  Ev<MODE, EK> ev(p.child, row, p.mp);
  const bool any = t0 < nvalid;
  const float padv0 = p.pad_last ? ev.value(L - 1, ev.load(L - 1)) : p.pad_value;
  const float ufill = p.padmode ? sg * padv0 : -INFINITY;  // samples past the end

  if (threadIdx.x == 0) padv_sh = padv0;
  if (any) {
    const int n = NB * K;
    for (int i0 = threadIdx.x; i0 < n; i0 += 4 * FG_THREADS) {
      typename Ev<MODE, EK>::Raw r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = i0 + u * FG_THREADS;
        if (i < n && s0 + i < L) r[u] = ev.load(s0 + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = i0 + u * FG_THREADS;
        if (i < n) {
          int idx = s0 + i;
          U[i + div_k(i, K, invK) * dK] = idx < L ? sg * ev.value(idx, r[u]) : ufill;
        }
      }
    }
  }
  __syncthreads();
  if (any && threadIdx.x < NB) {  // prefix scan of own block
    const float* u = U + threadIdx.x * Kp;
    float* q1 = P1 + threadIdx.x * Kp;
    if (MODE == M_HARD) {
      float bv = u[0];
      q1[0] = bv;
#pragma unroll 4
      for (int i = 1; i < K; ++i) {
        float x = u[i];
        bv = (x > bv) ? x : bv;
        q1[i] = bv;
      }
    } else if (MODE == M_LSE) {
      float m = u[0], s = 1.f;
      q1[0] = m;
#pragma unroll 4
      for (int i = 1; i < K; ++i) {
        lse_add(m, s, u[i], tau2);
        q1[i] = fmaf(lg2f(s), itau2, m);
      }
    } else {
      float* q2 = P2 + threadIdx.x * Kp;
      float m = u[0], s = 1.f, q = 0.f;
      q1[0] = m;
      q2[0] = m;
#pragma unroll 2
      for (int i = 1; i < K; ++i) {
        soft_add(m, s, q, u[i], tau2);
        q1[i] = m + q / s;
        q2[i] = fmaf(lg2f(s), itau2, m);
      }
    }
  }
  __syncthreads();
  if (any && threadIdx.x < NB - 1) {  // suffix walk + combine with the next block's prefix
    float* u = U + threadIdx.x * Kp;
    const float* n1 = P1 + (threadIdx.x + 1) * Kp - 1;  // n1[i] = next block prefix at i-1
    if (MODE == M_HARD) {
      float acc = u[K - 1];
#pragma unroll 4
      for (int i = K - 1; i >= 0; --i) {
        float x = u[i];
        acc = (x >= acc) ? x : acc;  // walking backwards: ties keep the earlier sample
        float r = acc;
        if (i > 0) {
          float pv = n1[i];
          r = (pv > r) ? pv : r;
        }
        u[i] = r;
      }
    } else if (MODE == M_LSE) {
      float m = u[K - 1], s = 1.f;
#pragma unroll 4
      for (int i = K - 1; i >= 0; --i) {
        if (i < K - 1) lse_add(m, s, u[i], tau2);
        float mm = m, ss = s;
        if (i > 0) lse_merge(mm, ss, n1[i], 1.f, tau2);
        u[i] = fmaf(lg2f(ss), itau2, mm);
      }
    } else {
      const float* n2 = P2 + (threadIdx.x + 1) * Kp - 1;
      float* ax = AX + threadIdx.x * Kp;
      float m = u[K - 1], s = 1.f, q = 0.f;
#pragma unroll 2
      for (int i = K - 1; i >= 0; --i) {
        if (i < K - 1) soft_add(m, s, q, u[i], tau2);
        float mm = m, ss = s, qq = q;
        if (i > 0) {
          float Lp = n2[i];
          soft_merge(mm, ss, qq, Lp, 1.f, n1[i] - Lp, tau2);
        }
        u[i] = mm + qq / ss;
        ax[i] = fmaf(lg2f(ss), itau2, mm);
      }
    }
  }
  __syncthreads();
  const float padv = padv_sh;
  float* outr = p.out + row * L;
  float* auxr = (MODE == M_SOFT) ? p.aux + row * L : nullptr;
  const int tend = (t0 + J < L ? t0 + J : L) - t0;
  for (int i = threadIdx.x; i < tend; i += FG_THREADS) {
    int t = t0 + i;
    int q = i + div_k(i, K, invK) * dK;
    float v;
    if (t < nvalid) {
      float M = U[q];
      float lse = (MODE == M_SOFT) ? AX[q] : 0.f;
      if (p.fill)  // columns of L + b rows: K kept, the rest sentinel (t + a of them first)
        fill_merge<MODE>(M, lse, (float)(L + p.b - K), p.sent, t + p.a > 0, tau2, itau2);
      v = sg * M;
      if (MODE == M_SOFT) auxr[t] = lse;
    } else {
      v = padv;
    }
    if (p.canon) v = __fadd_rn(v, 0.f);
    outr[t] = v;
  }
}

// ===========================================================================
// timed F / G — backward, LSE and softmax (window sum over the cotangent)
// ===========================================================================
// The CTA owns child elements j in [j0, j0 + J), J = (NB-1) K; element j
// receives from outputs t in [j - b, j - a], a window of K over the output
// sequence starting at tb = j0 - b.  Shared layout (stride Kp):
//   LSE:  HM = M_t (u-space output), HG = g_t; prefix PM, PA
//   soft: HM = L_t (window LSE), HG = g_t, HC = M_t, HB (result Bc); prefix PM, PA, PB, PC
// Gradient: LSE  g_child[j] = sum_t g_t exp(tau (u_j - M_t))
//           soft g_child[j] = sum_t g_t exp(tau (u_j - L_t)) (1 + tau (u_j - M_t))
__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

template <int MODE, int EK>
__global__ void __launch_bounds__(FG_THREADS) k_fgt_bwd_sm(const __grid_constant__ FGParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red_sh[32];
  const int NB = p.NB, K = p.K, Kp = p.Kp, dK = Kp - K;
  const int nsm = NB * Kp;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = (NB - 1) * K;
  const int j0 = blockIdx.x * J;
  const int tb = j0 - p.b;
  const int nvalid = L - p.b;
  const float invK = 1.f / (float)K;
  float* HM = sm;
  float* HG = sm + nsm;
  float* HC = sm + 2 * nsm;  // soft only
  float* HB = sm + 3 * nsm;  // soft only
  float* PM = sm + (MODE == M_SOFT ? 4 : 2) * nsm;
  float* PA = PM + nsm;
  float* PB = PA + nsm;  // soft only
  float* PC = PB + nsm;  // soft only
  const float tau2 = p.mp.tau2, tau = p.mp.tau, sg = p.sg;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  const float* auxr = (MODE == M_SOFT) ? p.aux_in + row * L : nullptr;

  {
    const int n = NB * K;
    for (int i0 = threadIdx.x; i0 < n; i0 += 2 * FG_THREADS) {
      float gv[2], ov[2], av[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        int i = i0 + u * FG_THREADS;
        int t = tb + i;
        bool v = i < n && t >= 0 && t < nvalid;
        gv[u] = v ? cot[t] : 0.f;
        ov[u] = v ? outr[t] : 0.f;
        av[u] = (MODE == M_SOFT && v) ? auxr[t] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        int i = i0 + u * FG_THREADS;
        if (i >= n) continue;
        int q = i + div_k(i, K, invK) * dK;
        HG[q] = gv[u];
        if (MODE == M_LSE) {
          HM[q] = sg * ov[u];
        } else {
          HM[q] = av[u];
          HC[q] = sg * ov[u];
        }
      }
    }
  }
  // pad contribution: overrun outputs route their cotangent to c[L-1] ('last' padding)
  const bool own_last = p.pad_last && (L - 1 >= j0) && (L - 1 < j0 + J);
  float padsum = 0.f;
  if (own_last) {  // block-uniform branch
    float s = 0.f;
    int t_lo = nvalid > 0 ? nvalid : 0;
    for (int t = t_lo + threadIdx.x; t < L; t += blockDim.x) s += cot[t];
    padsum = block_sum(s, red_sh);
  }
  __syncthreads();
  if (threadIdx.x < NB) {  // prefix scans
    const int b0 = threadIdx.x * Kp;
    if (MODE == M_LSE) {
      float mu = HM[b0], A = HG[b0];
      PM[b0] = mu;
      PA[b0] = A;
#pragma unroll 4
      for (int i = 1; i < K; ++i) {
        gl_add(mu, A, HM[b0 + i], HG[b0 + i], tau2);
        PM[b0 + i] = mu;
        PA[b0 + i] = A;
      }
    } else {
      float mu = HM[b0], A = HG[b0], Bc = 0.f, c = HC[b0];
      PM[b0] = mu;
      PA[b0] = A;
      PB[b0] = Bc;
      PC[b0] = c;
#pragma unroll 2
      for (int i = 1; i < K; ++i) {
        int q = b0 + i;
        gs_add(mu, A, Bc, c, HM[q], HG[q], 0.f, HC[q], tau2);
        PM[q] = mu;
        PA[q] = A;
        PB[q] = Bc;
        PC[q] = c;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < NB - 1) {  // suffix walk + combine; results in place into H*
    const int b0 = threadIdx.x * Kp, nb = b0 + Kp - 1;  // nb + i = next block prefix at i - 1
    if (MODE == M_LSE) {
      float mu = HM[b0 + K - 1], A = HG[b0 + K - 1];
#pragma unroll 4
      for (int i = K - 1; i >= 0; --i) {
        if (i < K - 1) gl_add(mu, A, HM[b0 + i], HG[b0 + i], tau2);
        float m2 = mu, a2 = A;
        if (i > 0) gl_add(m2, a2, PM[nb + i], PA[nb + i], tau2);
        HM[b0 + i] = m2;
        HG[b0 + i] = a2;
      }
    } else {
      int q = b0 + K - 1;
      float mu = HM[q], A = HG[q], Bc = 0.f, c = HC[q];
#pragma unroll 2
      for (int i = K - 1; i >= 0; --i) {
        q = b0 + i;
        if (i < K - 1) gs_add(mu, A, Bc, c, HM[q], HG[q], 0.f, HC[q], tau2);
        float m2 = mu, a2 = A, b2 = Bc, c2 = c;
        if (i > 0) gs_add(m2, a2, b2, c2, PM[nb + i], PA[nb + i], PB[nb + i], PC[nb + i], tau2);
        HM[q] = m2;
        HG[q] = a2;
        HC[q] = c2;
        HB[q] = b2;
      }
    }
  }
  __syncthreads();
  Ev<MODE, EK> ev(p.child, row, p.mp);
  const int jn = (j0 + J < L ? j0 + J : L) - j0;
  for (int i0 = threadIdx.x; i0 < jn; i0 += 2 * FG_THREADS) {
    typename Ev<MODE, EK>::Raw r[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int i = i0 + u * FG_THREADS;
      if (i < jn) r[u] = ev.load(j0 + i);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int i = i0 + u * FG_THREADS;
      if (i >= jn) continue;
      int j = j0 + i;
      int q = i + div_k(i, K, invK) * dK;
      float A = HG[q];
      float g = 0.f;
      if (MODE == M_LSE) {
        if (A != 0.f) {
          float uj = sg * ev.value(j, r[u]);
          g = A * ex2f(tau2 * (uj - HM[q]));
        }
      } else {
        float Bc = HB[q];
        if (A != 0.f || Bc != 0.f) {
          float uj = sg * ev.value(j, r[u]);
          g = ex2f(tau2 * (uj - HM[q])) * (A * fmaf(tau, uj - HC[q], 1.f) - tau * Bc);
        }
      }
      if (own_last && j == L - 1) g += padsum;
      ev.grad(j, r[u], g);
    }
  }
}

// ===========================================================================
// timed F / G — backward, hard (recompute the first arg-max, scatter in smem)
// ===========================================================================
// Inputs cover NB+1 blocks from s0 = j0 - K + 1 (the start of the window of
// output t = j0 - b); outputs t = s - a for starts s in blocks 0..NB-1.
//   U [(NB+1)Kp] child, PV/PI prefix (value, tile-local index),
//   GT [NB*Kp] cotangent by start, G [2][J] accumulated child cotangent: thread qb's
//   windows reach blocks qb and qb+1 only, so even and odd threads each own their
//   targets in one of the two copies (plain adds in program order, summed in a fixed
//   order at the end: reproducible, no atomics); padded targets ('last') are summed per
//   thread and folded in thread order
template <int EK>
__global__ void __launch_bounds__(FG_THREADS) k_fgt_bwd_hard(const __grid_constant__ FGParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red_sh[32];
  const int NB = p.NB, K = p.K, Kp = p.Kp, dK = Kp - K;
  const int NBi = NB + 1;
  const int nsi = NBi * Kp;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = (NB - 1) * K;
  const int j0 = blockIdx.x * J;
  const int s0 = j0 - K + 1;
  // padded windows: outputs whose window lies wholly past the end route to c[L-1] via padsum
  const int nvalid = p.padmode ? L - p.a : L - p.b;
  const float invK = 1.f / (float)K;
  float* U = sm;
  float* PV = sm + nsi;
  int* PI = reinterpret_cast<int*>(sm + 2 * nsi);
  float* GT = sm + 3 * nsi;
  float* G = GT + NB * Kp;
  float* G2 = G + J;
  __shared__ float PADG[256];
  const float sg = p.sg;
  const float* cot = p.cot + row * L;
  Ev<M_HARD, EK> ev(p.child, row, p.mp);
  const float ufill =
      p.padmode ? sg * (p.pad_last ? ev.value(L - 1, ev.load(L - 1)) : p.pad_value) : -INFINITY;

  {
    const int n = NBi * K;
    for (int i0 = threadIdx.x; i0 < n; i0 += 4 * FG_THREADS) {
      typename Ev<M_HARD, EK>::Raw r[4];
      float gv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = i0 + u * FG_THREADS;
        int idx = s0 + i;
        if (i < n && idx >= 0 && idx < L) r[u] = ev.load(idx);
        int t = idx - p.a;
        gv[u] = (i < NB * K && t >= 0 && t < nvalid) ? cot[t] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i = i0 + u * FG_THREADS;
        if (i >= n) continue;
        int idx = s0 + i;
        int q = i + div_k(i, K, invK) * dK;
        U[q] = (idx >= 0 && idx < L) ? sg * ev.value(idx, r[u]) : (idx >= L ? ufill : -INFINITY);
        if (i < NB * K) GT[q] = gv[u];
      }
    }
  }
  for (int i = threadIdx.x; i < 2 * J; i += FG_THREADS) G[i] = 0.f;
  // all-pad windows route to c[L-1]; in fill mode only if the pad beats the sentinel
  const bool own_last = p.pad_last && (L - 1 >= j0) && (L - 1 < j0 + J) &&
                        !(p.fill && ufill <= -p.sent);
  float padsum = 0.f;
  if (own_last) {
    float s = 0.f;
    int t_lo = nvalid > 0 ? nvalid : 0;
    for (int t = t_lo + threadIdx.x; t < L; t += blockDim.x) s += cot[t];
    padsum = block_sum(s, red_sh);
  }
  __syncthreads();
  if (threadIdx.x < NBi) {  // prefix (value, first arg-max)
    const int b0 = threadIdx.x * Kp;
    const int l0 = threadIdx.x * K;
    float bv = U[b0];
    int bi = l0;
    PV[b0] = bv;
    PI[b0] = bi;
#pragma unroll 4
    for (int i = 1; i < K; ++i) {
      float x = U[b0 + i];
      bool up = x > bv;
      bv = up ? x : bv;
      bi = up ? l0 + i : bi;
      PV[b0 + i] = bv;
      PI[b0 + i] = bi;
    }
  }
  __syncthreads();
  if (threadIdx.x < NB) {
    const int qb = threadIdx.x;
    const int b0 = qb * Kp, nb = b0 + Kp - 1;
    float* Gw = (qb & 1) ? G2 : G;
    float padg = 0.f;
    float av = U[b0 + K - 1];
    int ai = qb * K + K - 1;
#pragma unroll 4
    for (int i = K - 1; i >= 0; --i) {
      float x = U[b0 + i];
      bool up = x >= av;  // walking backwards: the new sample is earlier
      av = up ? x : av;
      ai = up ? qb * K + i : ai;
      int ri = ai;
      float rv = av;
      if (i > 0 && PV[nb + i] > av) {
        ri = PI[nb + i];
        rv = PV[nb + i];
      }
      float g = GT[b0 + i];
      if (p.fill) {  // the sentinel wins: no gradient (mask_fill cuts it, tape.py:229-234)
        float lse0 = 0.f;
        if (!fill_merge<M_HARD>(rv, lse0, (float)(L + p.b - K), p.sent, s0 + qb * K + i > 0, 0.f, 0.f))
          g = 0.f;
      }
      const int jj = s0 + ri;
      if (jj >= L) {  // padded samples route to c[L-1] ('last')
        if (p.pad_last) padg += g;
      } else if (g != 0.f && jj >= j0 && jj < j0 + J) {
        Gw[jj - j0] += g;
      }
    }
    PADG[qb] = padg;
  }
  __syncthreads();
  if (threadIdx.x == 0 && p.pad_last && L - 1 >= j0 && L - 1 < j0 + J) {
    float s = 0.f;
    for (int q = 0; q < NB; ++q) s += PADG[q];
    G[L - 1 - j0] += s;
  }
  __syncthreads();
  const int jn = (j0 + J < L ? j0 + J : L) - j0;
  for (int i0 = threadIdx.x; i0 < jn; i0 += 2 * FG_THREADS) {
    typename Ev<M_HARD, EK>::Raw r[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int i = i0 + u * FG_THREADS;
      if (i < jn) r[u] = ev.load(j0 + i);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int i = i0 + u * FG_THREADS;
      if (i >= jn) continue;
      int j = j0 + i;
      float g = G[i] + G2[i];
      if (own_last && j == L - 1) g += padsum;
      ev.grad(j, r[u], g);
    }
  }
}

// ===========================================================================
// brute-force timed F / G (tiny or huge windows): direct O(K) per output
// ===========================================================================
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_fwd_direct(const __grid_constant__ FGParams p) {
  const long long row = blockIdx.y, L = p.L;
  const long long nvalid = p.padmode ? L : L - p.b;
  const float tau2 = p.mp.tau2;
  const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  auto uval = [&](long long idx) {
    return p.sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
  };
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < L;
       t += (long long)gridDim.x * blockDim.x) {
    float v;
    if (t < nvalid) {
      if (MODE == M_HARD) {
        float m = -INFINITY;
        for (int k = 0; k < p.K; ++k) {
          float x = uval(t + p.a + k);
          if (x > m) m = x;
        }
        v = p.sg * m;
      } else if (MODE == M_LSE) {
        LseAcc a = {0.f, 0.f};
        for (int k = 0; k < p.K; ++k) a = lse_push(a, uval(t + p.a + k), tau2);
        v = p.sg * fmaf(lg2f(a.s), p.mp.inv_tau2, a.m);
      } else {
        SoftAcc a = {0.f, 0.f, 0.f};
        for (int k = 0; k < p.K; ++k) a = soft_push(a, uval(t + p.a + k), tau2);
        v = p.sg * (a.m + a.d / a.s);
        p.aux[row * L + t] = fmaf(lg2f(a.s), p.mp.inv_tau2, a.m);
      }
    } else {
      v = padv;
    }
    if (p.fill && t < nvalid) {
      float M = p.sg * v, lse = (MODE == M_SOFT) ? p.aux[row * L + t] : 0.f;
      fill_merge<MODE>(M, lse, (float)(L + p.b - p.K), p.sent, t + p.a > 0, tau2, p.mp.inv_tau2);
      v = p.sg * M;
      if (MODE == M_SOFT) p.aux[row * L + t] = lse;
    }
    if (p.canon) v = __fadd_rn(v, 0.f);
    p.out[row * L + t] = v;
  }
}

// backward: cotangent of the child into gbuf (atomics), then a pointwise VJP
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_bwd_direct(const __grid_constant__ FGParams p) {
  const long long row = blockIdx.y, L = p.L;
  const long long nvalid = p.padmode ? L : L - p.b;
  const float tau2 = p.mp.tau2;
  const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  auto uval = [&](long long idx) {
    return p.sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
  };
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
      long long am = 0;
      for (int k = 0; k < p.K; ++k) {
        float x = uval(t + p.a + k);
        if (x > m) {
          m = x;
          am = t + p.a + k;
        }
      }
      if (am >= L) am = p.pad_last ? L - 1 : -1;
      if (p.fill) {
        float lse0 = 0.f;
        if (!fill_merge<M_HARD>(m, lse0, (float)(L + p.b - p.K), p.sent, t + p.a > 0, 0.f, 0.f))
          am = -1;
      }
      if (am >= 0) atomicAdd(gb + am, g);
    } else {
      float M = p.sg * p.out_in[row * L + t];
      float Lt = (MODE == M_SOFT) ? p.aux_in[row * L + t] : M;
      for (int k = 0; k < p.K; ++k) {
        long long idx = t + p.a + k;
        float x = uval(idx);
        float w = ex2f(tau2 * (x - Lt));
        if (MODE == M_SOFT) w *= fmaf(p.mp.tau, x - M, 1.f);
        if (idx >= L) idx = p.pad_last ? L - 1 : -1;
        if (idx >= 0) atomicAdd(gb + idx, g * w);
      }
    }
  }
}

// backward for windows of K < 4 samples in gather form: thread j sums the contributions
// of the (at most 3) outputs whose window holds j, recomputing each window — every
// element written once, no atomics, so the sum order is fixed.  Element L-1 also
// collects the padded samples of 'last' padding and the overrun outputs.
template <int MODE>
__global__ void __launch_bounds__(256) k_fg_timed_bwd_gather(const __grid_constant__ FGParams p) {
  const long long row = blockIdx.y, L = p.L;
  const long long nvalid = p.padmode ? L : L - p.b;
  const float tau2 = p.mp.tau2;
  const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  auto uval = [&](long long idx) {
    return p.sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
  };
  const float* cot = p.cot + row * L;
  float* gb = p.gbuf + row * L;
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= L) return;
  const bool last = j == L - 1;
  // outputs whose window reaches j (or, for L-1 with 'last' padding, any padded sample)
  long long t_lo = j - p.b, t_hi = last ? L - 1 : j - p.a;
  if (t_lo < 0) t_lo = 0;
  float acc = 0.f;
  for (long long t = t_lo; t <= t_hi; ++t) {
    const float g = cot[t];
    if (g == 0.f) continue;
    if (t >= nvalid) {  // overrun output: the whole cotangent to the pad source
      if (last && p.pad_last) acc += g;
      continue;
    }
    if (MODE == M_HARD) {
      float m = -INFINITY;
      long long am = 0;
      for (int k = 0; k < p.K; ++k) {
        const float x = uval(t + p.a + k);
        if (x > m) {
          m = x;
          am = t + p.a + k;
        }
      }
      if (am >= L) am = p.pad_last ? L - 1 : -1;
      if (p.fill) {
        float lse0 = 0.f;
        if (!fill_merge<M_HARD>(m, lse0, (float)(L + p.b - p.K), p.sent, t + p.a > 0, 0.f, 0.f)) am = -1;
      }
      if (am == j) acc += g;
    } else {
      const float M = p.sg * p.out_in[row * L + t];
      const float Lt = (MODE == M_SOFT) ? p.aux_in[row * L + t] : M;
      for (int k = 0; k < p.K; ++k) {
        long long idx = t + p.a + k;
        if (idx >= L) idx = p.pad_last ? L - 1 : -1;
        if (idx != j) continue;
        const float x = uval(t + p.a + k);
        float w = ex2f(tau2 * (x - Lt));
        if (MODE == M_SOFT) w *= fmaf(p.mp.tau, x - M, 1.f);
        acc += g * w;
      }
    }
  }
  gb[j] = acc;
}

// ===========================================================================
// launchers for timed F / G
// ===========================================================================
static int odd_stride(int K) { return K | 1; }

// raise the dynamic shared-memory limit once per (kernel, size)
template <typename KernT>
static cudaError_t set_smem(KernT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static thread_local const void* done_fn[64];
  static thread_local size_t done_sz[64];
  static thread_local int n_done = 0;
  for (int i = 0; i < n_done; ++i)
    if (done_fn[i] == (const void*)k && done_sz[i] >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && n_done < 64) {
    done_fn[n_done] = (const void*)k;
    done_sz[n_done++] = bytes;
  }
  return e;
}

static const size_t kSmemBudget = 56 * 1024;  // per CTA: 4 CTAs x 256 threads per SM
static const size_t kSmemMax = 200 * 1024;

static int fwd_words(int mode) { return mode == M_SOFT ? 4 : 2; }
static int bwd_words(int mode) { return mode == M_SOFT ? 8 : (mode == M_HARD ? 5 : 4); }

// blocks per CTA: a multiple of 32 when it fits (full warps in the scans)
static int pick_nb(int K, int words) {
  long long per_block = (long long)words * odd_stride(K) * 4;
  long long nb = (long long)(kSmemBudget / per_block);
  if (nb >= 32) nb = (nb / 32) * 32;
  if (nb > 224) nb = 224;
  if (nb < 2) nb = 2;
  return (int)nb;
}

static bool use_direct(int K, int mode) {
  if (K < 4) return true;
  size_t need = (size_t)bwd_words(mode) * 3 * odd_stride(K) * 4;
  return need > kSmemMax;
}

#define DISPATCH_EK(EKV, ...)          \
  if ((EKV) == EK_AFF || (EKV) == EK_AFF1) { \
    constexpr int EK = EK_AFF;         \
    __VA_ARGS__;                       \
  } else if ((EKV) == EK_NORM) {       \
    constexpr int EK = EK_NORM;        \
    __VA_ARGS__;                       \
  } else if ((EKV) == EK_SRC) {        \
    constexpr int EK = EK_SRC;         \
    __VA_ARGS__;                       \
  } else if ((EKV) == EK_PAIR) {       \
    constexpr int EK = EK_PAIR;        \
    __VA_ARGS__;                       \
  } else {                             \
    constexpr int EK = EK_GEN;         \
    __VA_ARGS__;                       \
  }

template <int MODE, int EK>
static cudaError_t fwd_v2(FGParams& p, size_t smem, dim3 grid, cudaStream_t st) {
  cudaError_t e = set_smem(k_fgt_fwd<MODE, EK>, smem);
  if (e != cudaSuccess) return e;
  k_fgt_fwd<MODE, EK><<<grid, FG_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fg_timed_fwd(int mode, FGParams& p, cudaStream_t st) {
  if (mode == M_SOFT && sx_applicable(p)) return launch_sx_fwd(p, st);  // fp64 softmax (fg_soft64.cu)
  if (reg_applicable(mode, p, false)) return launch_reg_fwd(mode, expr_kind(p.child), p, st);
  if (use_direct(p.K, mode)) {
    dim3 grid((unsigned)((p.L + 255) / 256), (unsigned)p.B);
    if (mode == M_HARD) k_fg_timed_fwd_direct<M_HARD><<<grid, 256, 0, st>>>(p);
    else if (mode == M_LSE) k_fg_timed_fwd_direct<M_LSE><<<grid, 256, 0, st>>>(p);
    else k_fg_timed_fwd_direct<M_SOFT><<<grid, 256, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  const int ek = expr_kind(p.child);
  cudaError_t e;
  p.Kp = odd_stride(p.K);
  p.NB = pick_nb(p.K, fwd_words(mode));
  long long J = (long long)(p.NB - 1) * p.K;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  size_t smem = (size_t)fwd_words(mode) * p.NB * p.Kp * 4;
  if (mode == M_HARD) {
    DISPATCH_EK(ek, e = (fwd_v2<M_HARD, EK>(p, smem, grid, st)))
  } else if (mode == M_LSE) {
    DISPATCH_EK(ek, e = (fwd_v2<M_LSE, EK>(p, smem, grid, st)))
  } else {
    DISPATCH_EK(ek, e = (fwd_v2<M_SOFT, EK>(p, smem, grid, st)))
  }
  count_launch();
  return e;
}

template <int MODE, int EK>
static cudaError_t bwd_sm_v2(FGParams& p, size_t smem, dim3 grid, cudaStream_t st) {
  cudaError_t e = set_smem(k_fgt_bwd_sm<MODE, EK>, smem);
  if (e != cudaSuccess) return e;
  k_fgt_bwd_sm<MODE, EK><<<grid, FG_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

template <int EK>
static cudaError_t bwd_hard_v2(FGParams& p, size_t smem, dim3 grid, cudaStream_t st) {
  cudaError_t e = set_smem(k_fgt_bwd_hard<EK>, smem);
  if (e != cudaSuccess) return e;
  k_fgt_bwd_hard<EK><<<grid, FG_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fg_timed_bwd(int mode, FGParams& p, cudaStream_t st) {
  cudaError_t e;
  if (mode == M_SOFT && sx_applicable(p)) return launch_sx_bwd(p, st);
  if (reg_applicable(mode, p, true)) return launch_reg_bwd(mode, expr_kind(p.child), p, st);
  if (use_direct(p.K, mode)) {
    dim3 grid((unsigned)((p.L + 255) / 256), (unsigned)p.B);
    if (p.K < 4) {  // gather form: reproducible (K > ~3000 windows keep the scatter below)
      if (mode == M_HARD) k_fg_timed_bwd_gather<M_HARD><<<grid, 256, 0, st>>>(p);
      else if (mode == M_LSE) k_fg_timed_bwd_gather<M_LSE><<<grid, 256, 0, st>>>(p);
      else k_fg_timed_bwd_gather<M_SOFT><<<grid, 256, 0, st>>>(p);
    } else {
      if ((e = cudaMemsetAsync(p.gbuf, 0, sizeof(float) * p.B * p.L, st)) != cudaSuccess) return e;
      if (mode == M_HARD) k_fg_timed_bwd_direct<M_HARD><<<grid, 256, 0, st>>>(p);
      else if (mode == M_LSE) k_fg_timed_bwd_direct<M_LSE><<<grid, 256, 0, st>>>(p);
      else k_fg_timed_bwd_direct<M_SOFT><<<grid, 256, 0, st>>>(p);
    }
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_pointwise_vjp(mode, p, p.gbuf, st);
  }
  p.Kp = odd_stride(p.K);
  const int ek = expr_kind(p.child);
  if (mode == M_HARD) {
    // U, PV, PI over NB+1 blocks + GT over NB blocks + 2 x J accumulators
    int nb = pick_nb(p.K, 6);
    if (nb > 254) nb = 254;
    p.NB = nb;
    size_t smem = (size_t)3 * (nb + 1) * p.Kp * 4 + (size_t)nb * p.Kp * 4 + (size_t)2 * (nb - 1) * p.K * 4;
    long long J = (long long)(nb - 1) * p.K;
    dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
    DISPATCH_EK(ek, e = (bwd_hard_v2<EK>(p, smem, grid, st)))
    count_launch();
    return e;
  }
  const int words = bwd_words(mode);
  int nb = pick_nb(p.K, words);
  p.NB = nb;
  size_t smem = (size_t)words * nb * p.Kp * 4;
  long long J = (long long)(nb - 1) * p.K;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  if (mode == M_LSE) {
    DISPATCH_EK(ek, e = (bwd_sm_v2<M_LSE, EK>(p, smem, grid, st)))
  } else {
    DISPATCH_EK(ek, e = (bwd_sm_v2<M_SOFT, EK>(p, smem, grid, st)))
  }
  count_launch();
  return e;
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
        if (t < L) {
          float M = u[upos(k)], lse0 = 0.f;
          if (p.fill) fill_merge<M_HARD>(M, lse0, (float)t, p.sent, t > 0, 0.f, 0.f);
          p.out[row * L + t] = p.sg * M;
        }
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
        if (t < L) {
          float M = u[upos(k)], lse0 = 0.f;
          if (p.fill) fill_merge<M_LSE>(M, lse0, (float)t, p.sent, t > 0, tau2, p.mp.inv_tau2);
          p.out[row * L + t] = p.sg * M;
        }
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
          float M = u[upos(k)], lse = ax[upos(k)];
          if (p.fill) fill_merge<M_SOFT>(M, lse, (float)t, p.sent, t > 0, tau2, p.mp.inv_tau2);
          p.out[row * L + t] = p.sg * M;
          p.aux[row * L + t] = lse;
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
      if (p.fill) {
        float M = acc.v, lse0 = 0.f;
        if (!fill_merge<M_HARD>(M, lse0, (float)t, p.sent, t > 0, 0.f, 0.f)) g = 0.f;
      }
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
  cudaError_t err;
  if (launch_unt_fwd(mode, p, st, err)) return err;
  dim3 grid((unsigned)p.B);
  if (mode == M_HARD) k_fg_untimed_fwd<M_HARD><<<grid, UT_T, 0, st>>>(p);
  else if (mode == M_LSE) k_fg_untimed_fwd<M_LSE><<<grid, UT_T, 0, st>>>(p);
  else k_fg_untimed_fwd<M_SOFT><<<grid, UT_T, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fg_untimed_bwd(int mode, FGParams& p, cudaStream_t st) {
  {
    cudaError_t err;
    if (launch_unt_bwd(mode, p, st, err)) return err;
  }
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
