// until.cu — Until kernels (masking.py:238-293).
//
// Reference semantics, per start t (K = b - a + 1 timed; untimed a = 0 and
// k runs over the remaining signal):
//   pm_k(t)   = R^min l[t .. t+a+k]          (incremental for hard / LSE,
//                                            one application per k for softmax)
//   term_k(t) = R^min(pm_k(t), r[t+a+k])     (two-element reduction)
//   out[t]    = R^max_k term_k(t)
// timed: t + b > L-1  ->  hard min(pad_l, pad_r) in every mode, plus the
// `+ 0.0` canonicalisation of _replace_overrun (masking.py:180-192).
// Hard tie rules: pm keeps the earlier element, term ties go to pm, the outer
// max picks the smallest k (first arg-max).
//
// Kernels
//   * k_until_fwd / k_until_bwd: one thread per output t, child values staged
//     in shared memory.  The backward runs the k loop twice: forward to find
//     the output-level weights, then backwards from checkpoints (every CB
//     steps) to form the suffix sums over k that the gradient of pm_k needs.
//     The scattered cotangents (output t touches l[t..t+b], r[t+a..t+b]) are
//     accumulated warp-systolically: at step k lane i's contribution lands on
//     element t0 + a + k + i, which is owned by lane (i + k) mod 32, so a
//     shuffle replaces the atomic and each element is flushed once per warp.
//   * untimed hard: the O(T) clamp recurrence out[t] = max(min(l_t, r_t),
//     min(l_t, out[t+1])) as a chunked block scan of clamp functions; the
//     backward finds each output's gradient source locally (terminator test
//     with the stored out[t+1]) and sums cotangents over runs — no atomics,
//     the child VJPs are fused.
#include "kernels.cuh"

namespace stlg {

constexpr int U_THREADS = 128;
constexpr int U_CB = 64;  // checkpoint interval of the backward's reverse pass

// ---------------------------------------------------------------------------
// shared staging of the two child traces
// ---------------------------------------------------------------------------
// rows of the left / right child in "value space" over [lo, lo + n)
template <int MODE>
__device__ __forceinline__ void stage_children(const UParams& p, long long row, long long lo, int n,
                                               float* Ls, float* Rs) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    long long j = lo + i;
    if (j < p.L) {
      Ls[i] = expr_eval<MODE>(p.left, row, j, p.mp);
      Rs[i] = expr_eval<MODE>(p.right, row, j, p.mp);
    } else if (p.pad_last) {  // padded rows (read by masked_fill windows only)
      Ls[i] = expr_eval<MODE>(p.left, row, p.L - 1, p.mp);
      Rs[i] = expr_eval<MODE>(p.right, row, p.L - 1, p.mp);
    } else {
      Ls[i] = p.pad_value;
      Rs[i] = p.pad_value;
    }
  }
}

__device__ __forceinline__ float hard_min_first(float x, float y) { return (x <= y) ? x : y; }

// ---------------------------------------------------------------------------
// per-output forward (all modes, timed; untimed LSE / softmax)
// ---------------------------------------------------------------------------
// State of the running pm over x = -l ("max space"):
//   hard: value;  lse: (m, s);  soft: (m, s, q)
template <int MODE>
struct PmState {
  float m, s, q;
  int i;  // hard: index (tile-local) of the first arg-min
  __device__ __forceinline__ void init(float l, int idx) {
    m = -l;
    s = 1.f;
    q = 0.f;
    i = idx;
  }
  __device__ __forceinline__ void push(float l, int idx, float tau2) {
    float x = -l;
    if (MODE == M_HARD) {
      if (x > m) {  // strictly smaller l: the earlier minimum keeps ties
        m = x;
        i = idx;
      }
    } else if (MODE == M_LSE) {
      lse_add(m, s, x, tau2);
    } else {
      soft_add(m, s, q, x, tau2);
    }
  }
  // pm value (l space)
  __device__ __forceinline__ float value(float itau2) const {
    if (MODE == M_HARD) return -m;
    if (MODE == M_LSE) return -fmaf(lg2f(s), itau2, m);
    return -(m + q / s);
  }
};

// term = R^min(pm, r) as the reference's 2-element reduction (stack + reduce)
template <int MODE>
__device__ __forceinline__ float term_of(float pm, float r, const ModeP& mp, float& p1, float& p2) {
  return pair_red<MODE>(pm, r, -1.f, mp, p1, p2);
}

// masked_fill (masking.py:261-270): pm_k and the right operand are reductions over
// FULL columns of `rows` entries, the kept rows plus sentinel fills (+sent for a min,
// i.e. -sent in max space).  (MX, lse): the kept part's reduction in max space (and
// its LSE for softmax).  Returns the filled l-space value; lse becomes the filled LSE;
// `kept` is false when a sentinel wins the hard min (then no gradient flows).
template <int MODE>
__device__ __forceinline__ float fill_min(float MX, float& lse, float nu, float sent, bool sent_first,
                                          float tau2, float itau2, bool& kept) {
  kept = fill_merge<MODE>(MX, lse, nu, sent, sent_first, tau2, itau2);
  if (MODE == M_LSE) lse = MX;
  return -MX;
}
// (max-space value, LSE) of a PmState
template <int MODE>
__device__ __forceinline__ void pm_mx(const PmState<MODE>& pm, float itau2, float& MX, float& lse) {
  if (MODE == M_HARD) {
    MX = pm.m;
    lse = pm.m;
  } else if (MODE == M_LSE) {
    MX = fmaf(lg2f(pm.s), itau2, pm.m);
    lse = MX;
  } else {
    MX = pm.m + pm.q / pm.s;
    lse = fmaf(lg2f(pm.s), itau2, pm.m);
  }
}
// d(filled min)/d(element) for an element x (l space) of that column
template <int MODE>
__device__ __forceinline__ float fill_weight(float x, float vfill, float lse, float tau, float tau2, bool kept) {
  if (MODE == M_HARD) return kept ? 1.f : 0.f;
  const float w = ex2f(tau2 * (-x - lse));
  if (MODE == M_LSE) return w;
  return w * fmaf(tau, vfill - x, 1.f);
}

template <int MODE>
__global__ void __launch_bounds__(U_THREADS) k_until_fwd(const __grid_constant__ UParams p) {
  extern __shared__ __align__(16) float sm[];
  const long long row = blockIdx.y, L = p.L;
  const long long t0 = (long long)blockIdx.x * U_THREADS;
  const long long nvalid = (p.untimed || p.fill) ? L : L - p.b;
  const int span = p.untimed ? (int)(L - t0) : U_THREADS + p.b;
  const int nst = (int)((t0 + span <= L || p.fill) ? span : (L - t0));
  const long long rows = p.untimed ? L : L + p.b;  // column height (masked_fill)
  float* Ls = sm;
  float* Rs = sm + nst;
  if (t0 < nvalid) stage_children<MODE>(p, row, t0, nst, Ls, Rs);
  __syncthreads();
  const long long t = t0 + threadIdx.x;
  if (t >= L) return;
  float v;
  if (t >= nvalid) {
    float pl = p.pad_last ? expr_eval<MODE>(p.left, row, L - 1, p.mp) : p.pad_value;
    float pr = p.pad_last ? expr_eval<MODE>(p.right, row, L - 1, p.mp) : p.pad_value;
    v = hard_min_first(pl, pr);
  } else {
    const int i0 = threadIdx.x;
    const int K = p.untimed ? (int)(L - t) : p.K;
    const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2;
    PmState<MODE> pm;
    pm.init(Ls[i0], i0);
    for (int i = 1; i <= p.a; ++i) pm.push(Ls[i0 + i], i0 + i, tau2);
    // outer max over k, in max space of the terms
    float M = 0.f, S = 0.f, Q = 0.f;
    for (int k = 0; k < K; ++k) {
      int e = i0 + p.a + k;
      if (k > 0) pm.push(Ls[e], e, tau2);
      float w1, w2;
      float pmv, rv = Rs[e];
      if (p.fill) {
        float MX, lse;
        bool kept;
        pm_mx<MODE>(pm, itau2, MX, lse);
        pmv = fill_min<MODE>(MX, lse, (float)(rows - (p.a + k + 1)), p.sent, t > 0, tau2, itau2, kept);
        float lr = -rv;
        rv = fill_min<MODE>(-rv, lr, (float)(rows - 1), p.sent, t + p.a + k > 0, tau2, itau2, kept);
      } else {
        pmv = pm.value(itau2);
      }
      float term = term_of<MODE>(pmv, rv, p.mp, w1, w2);
      if (MODE == M_HARD) {
        if (k == 0 || term > M) M = term;  // first k wins ties
      } else if (MODE == M_LSE) {
        if (k == 0) {
          M = term;
          S = 1.f;
        } else {
          lse_add(M, S, term, tau2);
        }
      } else {
        if (k == 0) {
          M = term;
          S = 1.f;
          Q = 0.f;
        } else {
          soft_add(M, S, Q, term, tau2);
        }
      }
    }
    if (MODE == M_HARD) v = M;
    else if (MODE == M_LSE) v = fmaf(lg2f(S), itau2, M);
    else v = M + Q / S;
    if (p.fill && p.untimed && t > 0) {  // slices past the end: -sentinel terms (masking.py:271-273)
      float lse = (MODE == M_SOFT) ? fmaf(lg2f(S), itau2, M) : v;
      fill_merge<MODE>(v, lse, (float)t, p.sent, false, tau2, itau2);
    }
  }
  if (p.canon) v = __fadd_rn(v, 0.f);
  p.out[row * L + t] = v;
}

// ---------------------------------------------------------------------------
// warp-systolic scatter: lane i contributes `val` to element base + k + i;
// owner lane o = (i + k) mod 32 accumulates element base + k + ((o - k) mod 32)
// ---------------------------------------------------------------------------
struct Systolic {
  float acc;
  long long cur;  // element currently accumulated by this lane (-1 none)
  __device__ __forceinline__ void reset() {
    acc = 0.f;
    cur = -1;
  }
  // called by all 32 lanes with the same k (warp-uniform); dst = row base pointer
  __device__ __forceinline__ void step(float val, long long base, int k, float* dst, long long L) {
    const int lane = threadIdx.x & 31;
    int src = (lane - k) & 31;
    float got = __shfl_sync(0xffffffffu, val, src);
    long long j = base + k + ((lane - k) & 31);
    if (j != cur) {
      put(dst, L);
      cur = j;
      acc = 0.f;
    }
    acc += got;
  }
  // padded positions (masked_fill windows past the end) feed element L - 1 under
  // 'last' padding (pad_last is set by the caller) and nothing under a constant pad
  int pad_last = 0;
  __device__ __forceinline__ void put(float* dst, long long L) {
    if (cur >= 0 && acc != 0.f) {
      if (cur < L) atomicAdd(dst + cur, acc);
      else if (pad_last) atomicAdd(dst + L - 1, acc);
    }
  }
  __device__ __forceinline__ void flush(float* dst, long long L) {
    put(dst, L);
    reset();
  }
};

// ---------------------------------------------------------------------------
// per-output backward (timed all modes; untimed LSE / softmax)
// ---------------------------------------------------------------------------
// Writes the child cotangents into p.gl / p.gr (zero-initialised, atomics);
// the child VJPs run afterwards as pointwise kernels.
//
// Hard: one source per output (pm's first arg-min or r at the winning k).
// LSE (reference VJP of the incremental pair LSEs, equal to the flat form):
//   dr[e_k]  += g exp(tau (2 term_k - out - r_e))
//   dl[j]    += g exp(tau (pm_k0 - l_j)) * SA_k0,  k0 = max(0, j - t - a)
//   SA_k      = sum_{k' >= k} exp(tau (2 term_k' - out - pm_k))   (suffix, stable)
// Softmax: out = softmax_k(term_k) (weights W_k (1 + tau (term_k - out))),
//   term_k = 2-element softmin(pm_k, r), pm_k = softmin(l[t..t+a+k]).
template <int MODE>
__global__ void __launch_bounds__(U_THREADS) k_until_bwd(const __grid_constant__ UParams p) {
  extern __shared__ __align__(16) float sm[];
  const long long row = blockIdx.y, L = p.L;
  const long long t0 = (long long)blockIdx.x * U_THREADS;
  const long long nvalid = (p.untimed || p.fill) ? L : L - p.b;
  const int span = p.untimed ? (int)(L - t0) : U_THREADS + p.b;
  const int nst = (int)((t0 + span <= L || p.fill) ? span : (L - t0));
  const long long rows = p.untimed ? L : L + p.b;  // column height (masked_fill)
  const int Kmax = p.untimed ? (int)(L - t0) : p.K;
  const int nck = (Kmax + U_CB - 1) / U_CB;
  float* Ls = sm;
  float* Rs = sm + nst;
  float* CK = Rs + nst;                         // checkpoints [nck][3][U_THREADS]
  float* BUF = CK + (size_t)nck * 3 * U_THREADS;  // block buffer [U_CB][2][U_THREADS]
  const int tid = threadIdx.x;
  const long long t = t0 + tid;
  const bool active = t < nvalid;
  float* gl = p.gl + row * L;
  float* gr = p.gr + row * L;
  const float* cot = p.cot + row * L;
  if (t0 < L) {
    // overrun outputs route to the pad sources (last padding): left if pl <= pr
    if (t < L && !active && p.pad_last) {
      float g = cot[t];
      if (g != 0.f) {
        float pl = expr_eval<MODE>(p.left, row, L - 1, p.mp);
        float pr = expr_eval<MODE>(p.right, row, L - 1, p.mp);
        atomicAdd((pl <= pr ? gl : gr) + (L - 1), g);
      }
    }
  }
  if (t0 >= nvalid) return;  // whole tile overruns (uniform)
  stage_children<MODE>(p, row, t0, nst, Ls, Rs);
  __syncthreads();
  const float tau = p.mp.tau, tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2;
  const int K = active ? (p.untimed ? (int)(L - t) : p.K) : 0;
  const float g = active ? cot[t] : 0.f;
  const float out_t = active ? p.out_in[row * L + t] : 0.f;

  // warp-uniform loop bound
  int Kw = K;
  for (int o = 16; o > 0; o >>= 1) Kw = max(Kw, __shfl_xor_sync(0xffffffffu, Kw, o));

  if (MODE == M_HARD) {
    if (!active || g == 0.f) return;
    PmState<M_HARD> pm;
    pm.init(Ls[tid], tid);
    for (int i = 1; i <= p.a; ++i) pm.push(Ls[tid + i], tid + i, tau2);
    float best = 0.f;
    int bsrc = 0;  // tile-local index; bit 30 set: right child; -1: a sentinel won
    for (int k = 0; k < K; ++k) {
      int e = tid + p.a + k;
      if (k > 0) pm.push(Ls[e], e, tau2);
      float pmv = -pm.m, r = Rs[e];
      bool kl = true, kr = true;
      if (p.fill) {
        float lse = pm.m;
        pmv = fill_min<M_HARD>(pm.m, lse, (float)(rows - (p.a + k + 1)), p.sent, t > 0, tau2, itau2, kl);
        float lr = -r;
        r = fill_min<M_HARD>(-r, lr, (float)(rows - 1), p.sent, t + p.a + k > 0, tau2, itau2, kr);
      }
      bool use_l = pmv <= r;
      float term = use_l ? pmv : r;
      if (k == 0 || term > best) {
        best = term;
        bsrc = use_l ? (kl ? pm.i : -1) : (kr ? (e | (1 << 30)) : -1);
      }
    }
    if (p.fill && p.untimed && t > 0 && best < -p.sent) bsrc = -1;  // -sentinel terms win
    if (bsrc < 0) return;
    long long j = t0 + (bsrc & ~(1 << 30));
    if (j >= L) {  // padded row: 'last' padding reads element L - 1
      if (!p.pad_last) return;
      j = L - 1;
    }
    atomicAdd(((bsrc & (1 << 30)) ? gr : gl) + j, g);
    return;
  }

  // ---- pass 1: forward over k, checkpoints of the pm state; outer LSE ------------
  PmState<MODE> pm;
  pm.init(Ls[tid], tid);
  for (int i = 1; i <= p.a; ++i) pm.push(Ls[tid + i], tid + i, tau2);
  float Lout = 0.f;  // LSE over the terms (softmax needs it; LSE: equals out)
  {
    float M = 0.f, S = 0.f;
    for (int k = 0; k < K; ++k) {
      int e = tid + p.a + k;
      if (k > 0) pm.push(Ls[e], e, tau2);
      if (k % U_CB == 0) {
        float* c = CK + (size_t)(k / U_CB) * 3 * U_THREADS;
        c[tid] = pm.m;
        c[U_THREADS + tid] = pm.s;
        c[2 * U_THREADS + tid] = pm.q;
      }
      if (MODE == M_SOFT) {
        float w1, w2;
        float pmv = pm.value(itau2), rv = Rs[e];
        if (p.fill) {
          float MX, lse;
          bool kept;
          pm_mx<MODE>(pm, itau2, MX, lse);
          pmv = fill_min<MODE>(MX, lse, (float)(rows - (p.a + k + 1)), p.sent, t > 0, tau2, itau2, kept);
          float lr = -rv;
          rv = fill_min<MODE>(-rv, lr, (float)(rows - 1), p.sent, t + p.a + k > 0, tau2, itau2, kept);
        }
        float term = term_of<MODE>(pmv, rv, p.mp, w1, w2);
        if (k == 0) {
          M = term;
          S = 1.f;
        } else {
          lse_add(M, S, term, tau2);
        }
      }
    }
    if (MODE == M_SOFT && p.fill && p.untimed && t > 0 && K > 0) lse_merge(M, S, -p.sent, (float)t, tau2);
    Lout = (MODE == M_SOFT) ? fmaf(lg2f(S), itau2, M) : out_t;
  }
  // ---- pass 2: backwards over checkpoint blocks -------------------------------
  Systolic accL, accR;
  accL.reset();
  accR.reset();
  accL.pad_last = accR.pad_last = p.pad_last;
  const long long base = t0 + p.a;  // lane i, step k -> element base + k + i (within the warp's t0)
  const int lane = tid & 31;
  const long long wbase = t0 + (tid & ~31) + p.a;
  // suffix accumulators
  float SA = 0.f, SB = 0.f;   // LSE: SA (ref pm_k); soft: SA = sum A, SB = sum A (pm' - pm_k)
  float prev_ref = 0.f;       // reference of the accumulators (pm_{k+1} for LSE, L_pm_{k+1} for soft)
  float prev_pm = 0.f;
  bool have = false;
  float pm0 = 0.f, Lpm0 = 0.f;
  for (int cb = (Kw + U_CB - 1) / U_CB - 1; cb >= 0; --cb) {
    const int k_lo = cb * U_CB;
    const int k_hi = min(k_lo + U_CB, Kw);
    // recompute the block forward from its checkpoint into BUF
    if (k_lo < K) {
      float* c = CK + (size_t)cb * 3 * U_THREADS;
      PmState<MODE> st;
      st.m = c[tid];
      st.s = c[U_THREADS + tid];
      st.q = c[2 * U_THREADS + tid];
      st.i = 0;
      for (int k = k_lo; k < min(k_hi, K); ++k) {
        int e = tid + p.a + k;
        if (k > k_lo) st.push(Ls[e], e, tau2);
        float* bb = BUF + (size_t)(k - k_lo) * 2 * U_THREADS;
        if (p.fill) {  // the filled column's min and LSE
          float MX, lse;
          bool kept;
          pm_mx<MODE>(st, itau2, MX, lse);
          bb[tid] = fill_min<MODE>(MX, lse, (float)(rows - (p.a + k + 1)), p.sent, t > 0, tau2, itau2, kept);
          bb[U_THREADS + tid] = lse;
        } else {
          bb[tid] = st.value(itau2);                                          // pm_k
          bb[U_THREADS + tid] = (MODE == M_SOFT) ? fmaf(lg2f(st.s), itau2, st.m) : 0.f;  // L_pm (x space)
        }
      }
    }
    for (int k = k_hi - 1; k >= k_lo; --k) {
      float vr = 0.f, vl = 0.f;
      if (k < K) {
        int e = tid + p.a + k;
        float* bb = BUF + (size_t)(k - k_lo) * 2 * U_THREADS;
        float pmk = bb[tid];
        float r = Rs[e];
        float dr = 1.f;  // d(filled right operand) / d r
        if (p.fill) {
          float lr = -r;
          bool kept;
          const float rf = fill_min<MODE>(-r, lr, (float)(rows - 1), p.sent, t + p.a + k > 0, tau2, itau2, kept);
          dr = fill_weight<MODE>(r, rf, lr, tau, tau2, kept);
          r = rf;
        }
        float w1, w2;
        float term = term_of<MODE>(pmk, r, p.mp, w1, w2);
        if (MODE == M_LSE) {
          // dr: g exp(tau (term - out)) * w2 ; dpm: g exp(tau (term - out)) * w1
          float wk = ex2f(tau2 * (term - out_t));
          vr = g * wk * w2 * dr;
          float c_pm = g * wk * w1;  // = g exp(tau (2 term - out - pm))
          // SA_k = c_pm_k / g-scale + exp(-tau (pm_k - pm_{k+1})) SA_{k+1}   (ref pm_k)
          SA = have ? fmaf(SA, ex2f(-tau2 * (pmk - prev_ref)), c_pm) : c_pm;
          prev_ref = pmk;
          have = true;
          // element e = t + a + k receives dpm via exp(tau (pm_k - l_e)) (k >= 1;
          // k == 0 elements are the a-prefix, handled after the loop)
          if (k > 0) vl = SA * ex2f(tau2 * (pmk - Ls[e]));
          if (k == 0) pm0 = pmk;
        } else {
          float Wk = ex2f(tau2 * (term - Lout)) * fmaf(tau, term - out_t, 1.f);
          vr = g * Wk * w2 * dr;
          float c_pm = g * Wk * w1;
          float Lpm = bb[U_THREADS + tid];
          // dl_j = exp(tau (-l_j - Lpm_k0)) [ (1 + tau (pm_k0 - l_j)) SA + tau SB ]
          //   SA = sum_{k'>=k0} c_pm_k' exp(-tau (Lpm_k' - Lpm_k0)),
          //   SB = sum_{k'>=k0} c_pm_k' exp(...) (pm_k' - pm_k0)
          if (have) {
            float f = ex2f(-tau2 * (prev_ref - Lpm));
            SB = f * fmaf(prev_pm - pmk, SA, SB);
            SA = fmaf(SA, f, c_pm);
          } else {
            SA = c_pm;
            SB = 0.f;
          }
          prev_ref = Lpm;
          prev_pm = pmk;
          have = true;
          if (k > 0) {
            float l = Ls[e];
            vl = ex2f(tau2 * (-l - Lpm)) * fmaf(1.f + tau * (pmk - l), SA, tau * SB);
          }
          if (k == 0) {
            pm0 = pmk;
            Lpm0 = Lpm;
          }
        }
      }
      accR.step(vr, wbase, k, gr, L);
      accL.step(vl, wbase, k, gl, L);
    }
  }
  accR.flush(gr, L);
  accL.flush(gl, L);
  // a-prefix elements j = t + i, i = 0..a, all with k0 = 0
  for (int i = 0; i <= p.a; ++i) {
    float vl = 0.f;
    if (K > 0) {
      float l = Ls[tid + i];
      if (MODE == M_LSE) vl = SA * ex2f(tau2 * (pm0 - l));
      else vl = ex2f(tau2 * (-l - Lpm0)) * fmaf(1.f + tau * (pm0 - l), SA, tau * SB);
    }
    accL.step(vl, wbase - p.a, i, gl, L);
  }
  accL.flush(gl, L);
  (void)lane;
  (void)base;
}

// ---------------------------------------------------------------------------
// untimed hard Until: O(T) clamp scan
// ---------------------------------------------------------------------------
// f_t(v) = (v >= l_t) ? l_t : ((v <= A_t) ? A_t : v),  A_t = (l_t <= r_t) ? l_t : r_t
// out[L-1] = A_{L-1};  out[t] = f_t(out[t+1]).
// Composition stays in this clamp family: F(v) = v >= hi ? hi : (v <= lo ? lo : v)
// with lo <= hi (values only; ties between +0 and -0 at chunk seams follow the
// composed form).
struct Clamp {
  float lo, hi;
};
// (G o F)(v) = G(F(v)): F applied first (later time), G after (earlier time)
__device__ __forceinline__ float clamp_apply(Clamp f, float v) {
  return (v >= f.hi) ? f.hi : ((v <= f.lo) ? f.lo : v);
}
__device__ __forceinline__ Clamp clamp_compose(Clamp g, Clamp f) {
  return Clamp{clamp_apply(g, f.lo), clamp_apply(g, f.hi)};
}

constexpr int UH_T = 256, UH_E = 8, UH_CH = UH_T * UH_E, UH_S = UH_E + 1;
__device__ __forceinline__ int uhpos(int k) { return (k >> 3) * UH_S + (k & 7); }

template <int MODE>
__global__ void __launch_bounds__(UH_T) k_until_unt_hard_fwd(const __grid_constant__ UParams p) {
  __shared__ float Ls[UH_T * UH_S];
  __shared__ float Rs[UH_T * UH_S];
  __shared__ Clamp cb[UH_T];
  const long long row = blockIdx.x, L = p.L;
  const int tid = threadIdx.x;
  // f_{L-1}(-inf) = A_{L-1}: the recurrence starts uniformly from -inf
  float carry = -INFINITY;
  for (long long c0 = ((L - 1) / UH_CH) * UH_CH; c0 >= 0; c0 -= UH_CH) {
    for (int k = tid; k < UH_CH; k += UH_T) {
      long long t = c0 + k;
      Ls[uhpos(k)] = t < L ? expr_eval<MODE>(p.left, row, t, p.mp) : 0.f;
      Rs[uhpos(k)] = t < L ? expr_eval<MODE>(p.right, row, t, p.mp) : 0.f;
    }
    __syncthreads();
    // this thread's function f_{t0} o f_{t0+1} o ... o f_{t0+E-1} (identity past the end)
    Clamp f{-INFINITY, INFINITY};
    for (int e = UH_E - 1; e >= 0; --e) {
      if (c0 + tid * UH_E + e >= L) continue;
      float l = Ls[tid * UH_S + e], r = Rs[tid * UH_S + e];
      Clamp ft{(l <= r) ? l : r, l};
      f = clamp_compose(ft, f);
    }
    cb[tid] = f;
    __syncthreads();
    for (int off = 1; off < UH_T; off <<= 1) {  // suffix composition C_i = F_i o F_{i+1} o ...
      Clamp x = cb[tid];
      if (tid + off < UH_T) x = clamp_compose(x, cb[tid + off]);
      __syncthreads();
      cb[tid] = x;
      __syncthreads();
    }
    float v = (tid + 1 < UH_T) ? clamp_apply(cb[tid + 1], carry) : carry;
    for (int e = UH_E - 1; e >= 0; --e) {  // exact sequential walk with the reference tie rules
      if (c0 + tid * UH_E + e >= L) continue;
      float l = Ls[tid * UH_S + e], r = Rs[tid * UH_S + e];
      float A = (l <= r) ? l : r;
      float Bv = (l <= v) ? l : v;
      v = (A >= Bv) ? A : Bv;
      Ls[tid * UH_S + e] = v;
    }
    __syncthreads();
    carry = Ls[0];
    for (int k = tid; k < UH_CH; k += UH_T) {
      long long t = c0 + k;
      if (t < L) p.out[row * L + t] = Ls[uhpos(k)];
    }
    __syncthreads();
  }
}

// backward: terminator test per t with the stored out[t+1]; runs of equal
// source end at their terminator, whose own index is the source index, so
// each child cotangent is final when its run ends (no atomics, fused VJPs).
template <int MODE>
__global__ void __launch_bounds__(UH_T) k_until_unt_hard_bwd(const __grid_constant__ UParams p) {
  __shared__ float sums[UH_T];
  __shared__ int flags[UH_T];
  __shared__ float carry_sh;
  const long long row = blockIdx.x, L = p.L;
  const int tid = threadIdx.x;
  const float* outr = p.out_in + row * L;
  const float* cot = p.cot + row * L;
  float carry = 0.f;  // cotangent accumulated since the last terminator (earlier chunks)
  for (long long c0 = 0; c0 < L; c0 += UH_CH) {
    float g[UH_E];
    int term[UH_E];  // 0: pass to the next sample's source, 1: l_t, 2: r_t
    float tail = 0.f;
    int anyterm = 0;
#pragma unroll
    for (int e = 0; e < UH_E; ++e) {
      long long t = c0 + tid * UH_E + e;
      term[e] = 0;
      g[e] = 0.f;
      if (t >= L) continue;
      float l = expr_eval<MODE>(p.left, row, t, p.mp);
      float r = expr_eval<MODE>(p.right, row, t, p.mp);
      bool a_is_l = l <= r;
      float A = a_is_l ? l : r;
      int src;
      if (t == L - 1) {
        src = a_is_l ? 1 : 2;
      } else {
        float v = outr[t + 1];
        bool b_is_l = l <= v;
        float Bv = b_is_l ? l : v;
        src = (A >= Bv) ? (a_is_l ? 1 : 2) : (b_is_l ? 1 : 0);
      }
      term[e] = src;
      g[e] = cot[t];
      if (src) {
        anyterm = 1;
        tail = 0.f;
      } else {
        tail += g[e];
      }
    }
    sums[tid] = tail;
    flags[tid] = anyterm;
    __syncthreads();
    if (tid == 0) {  // exclusive segmented prefix over the 256 thread aggregates
      float run = carry;
      for (int i = 0; i < UH_T; ++i) {
        float s = sums[i];
        int f = flags[i];
        sums[i] = run;
        run = f ? s : run + s;
      }
      carry_sh = run;
    }
    __syncthreads();
    float run = sums[tid];
#pragma unroll
    for (int e = 0; e < UH_E; ++e) {
      long long t = c0 + tid * UH_E + e;
      if (t >= L) break;
      run += g[e];
      float gl = 0.f, gr = 0.f;
      if (term[e] == 1) {
        gl = run;
        run = 0.f;
      } else if (term[e] == 2) {
        gr = run;
        run = 0.f;
      }
      expr_vjp<MODE>(p.left, row, t, gl, p.mp);
      expr_vjp<MODE>(p.right, row, t, gr, p.mp);
    }
    carry = carry_sh;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <typename KernT>
static cudaError_t set_smem_u(KernT k, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static const size_t kUSmemMax = 220 * 1024;

static size_t fwd_smem(const UParams& p) {
  long long span = p.untimed ? p.L : (long long)U_THREADS + p.b;
  if (span > p.L && !p.fill) span = p.L;
  return (size_t)2 * span * 4;
}
static size_t bwd_smem(const UParams& p) {
  long long span = p.untimed ? p.L : (long long)U_THREADS + p.b;
  if (span > p.L && !p.fill) span = p.L;
  long long kmax = p.untimed ? p.L : p.K;
  long long nck = (kmax + U_CB - 1) / U_CB;
  return (size_t)2 * span * 4 + (size_t)nck * 3 * U_THREADS * 4 + (size_t)U_CB * 2 * U_THREADS * 4;
}

template <int MODE>
static cudaError_t until_fwd_mode(UParams& p, cudaStream_t st) {
  if (p.untimed && MODE == M_HARD && !p.fill) {
    k_until_unt_hard_fwd<MODE><<<(unsigned)p.B, UH_T, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  size_t smem = fwd_smem(p);
  if (smem > kUSmemMax) return cudaErrorNotSupported;
  cudaError_t e = set_smem_u(k_until_fwd<MODE>, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + U_THREADS - 1) / U_THREADS), (unsigned)p.B);
  k_until_fwd<MODE><<<grid, U_THREADS, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t until_bwd_mode(UParams& p, cudaStream_t st) {
  if (p.untimed && MODE == M_HARD && !p.fill) {
    k_until_unt_hard_bwd<MODE><<<(unsigned)p.B, UH_T, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  size_t smem = bwd_smem(p);
  if (smem > kUSmemMax) return cudaErrorNotSupported;
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.gl, 0, sizeof(float) * p.B * p.L, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p.gr, 0, sizeof(float) * p.B * p.L, st)) != cudaSuccess) return e;
  if ((e = set_smem_u(k_until_bwd<MODE>, smem)) != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + U_THREADS - 1) / U_THREADS), (unsigned)p.B);
  k_until_bwd<MODE><<<grid, U_THREADS, smem, st>>>(p);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // child VJPs from the accumulated cotangents (left first: first-writer order)
  FGParams q;
  memset(&q, 0, sizeof(q));
  q.B = p.B;
  q.L = p.L;
  q.mp = p.mp;
  q.child = p.left;
  if ((e = launch_pointwise_vjp(MODE, q, p.gl, st)) != cudaSuccess) return e;
  q.child = p.right;
  return launch_pointwise_vjp(MODE, q, p.gr, st);
}

cudaError_t launch_until_fwd(int mode, UParams& p, cudaStream_t st) {
  if (mode == M_HARD) return until_fwd_mode<M_HARD>(p, st);
  if (mode == M_LSE) return until_fwd_mode<M_LSE>(p, st);
  return until_fwd_mode<M_SOFT>(p, st);
}

cudaError_t launch_until_bwd(int mode, UParams& p, cudaStream_t st) {
  if (mode == M_HARD) return until_bwd_mode<M_HARD>(p, st);
  if (mode == M_LSE) return until_bwd_mode<M_LSE>(p, st);
  return until_bwd_mode<M_SOFT>(p, st);
}

}  // namespace stlg
