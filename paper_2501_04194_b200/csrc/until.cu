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
//     min(l_t, out[t+1])) as a block scan of clamp functions, one CTA per
//     1024-sample chunk with look-back carries (lookback.cuh); the backward
//     finds each output's gradient source locally (terminator test with the
//     stored out[t+1]) and sums cotangents over runs — no atomics, the child
//     VJPs are fused.
#include "detacc.cuh"
#include "kernels.cuh"
#include "lookback.cuh"

namespace stlg {

constexpr int U_THREADS = 128;
constexpr int U_CB_S = 16;  // checkpoint interval, shared-memory variant (short timed windows)
constexpr int U_CB_G = 32;  // checkpoint interval, global-slab variant (untimed / long windows)
constexpr int U_PERSIST_PER_SM = 6;  // resident CTAs per SM of the persistent backward

// ---------------------------------------------------------------------------
// shared staging of the two child traces
// ---------------------------------------------------------------------------
// rows of the left / right child in "value space" over [lo, lo + n)
template <int MODE>
__device__ __forceinline__ void stage_children(const UParams& p, long long row, long long lo, int n,
                                               float* Ls, float* Rs) {
  const ChildEval cl(p.left, row), cr(p.right, row);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    long long j = lo + i;
    if (j < p.L) {
      Ls[i] = cl.value<MODE>(j, p.mp);
      Rs[i] = cr.value<MODE>(j, p.mp);
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

// 2^x as a double for x in fp32 range: the fraction through ex2 (fp32, ~2^-22
// relative), the integer part as exponent bits; 0 below 2^-1022
__device__ __forceinline__ double ex2d(float x) {
  if (!(x > -1022.f)) return 0.0;
  const float n = floorf(fminf(x, 1023.f));
  const double scale = __longlong_as_double((long long)((int)n + 1023) << 52);
  return (double)ex2f(x - n) * scale;
}

// ---------------------------------------------------------------------------
// per-output forward (all modes, timed; untimed LSE / softmax)
// ---------------------------------------------------------------------------
// State of the running pm over x = -l ("max space"):
//   hard: value;  lse: (m, s);  soft: (m, s, q)
// fp64 running sums: the LSE / softmax states of Until accumulate up to T terms
// (untimed), and fp32 additions of terms far below the running sum round
// systematically (error ~ T eps); each term's own ex2 error stays independent.
__device__ __forceinline__ void lse_add_d(float& m, double& s, float u, float tau2) {
  const float d = u - m;
  const double e = ex2f(-tau2 * fabsf(d));
  const bool up = d > 0.f;
  s = up ? fma(s, e, 1.0) : s + e;
  m = up ? u : m;
}
__device__ __forceinline__ void soft_add_d(float& m, double& s, double& q, float u, float tau2) {
  const float d = u - m;
  const double e = ex2f(-tau2 * fabsf(d));
  const bool up = d > 0.f;
  const double s_up = fma(s, e, 1.0), q_up = e * fma(-(double)d, s, q);
  const double s_dn = s + e, q_dn = fma((double)d, e, q);
  s = up ? s_up : s_dn;
  q = up ? q_up : q_dn;
  m = up ? u : m;
}

template <int MODE>
struct PmState {
  float m;
  double s, q;
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
      lse_add_d(m, s, x, tau2);
    } else {
      soft_add_d(m, s, q, x, tau2);
    }
  }
  // pm value (l space)
  __device__ __forceinline__ float value(float itau2) const {
    if (MODE == M_HARD) return -m;
    if (MODE == M_LSE) return -fmaf(lg2f((float)s), itau2, m);
    return -(m + (float)(q / s));
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
    MX = fmaf(lg2f((float)pm.s), itau2, pm.m);
    lse = MX;
  } else {
    MX = pm.m + (float)(pm.q / pm.s);
    lse = fmaf(lg2f((float)pm.s), itau2, pm.m);
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

// Child value access for one tile of U_THREADS outputs starting at t0: staged in
// shared memory (tile-local index e, span covers every window of the tile), or
// read directly through the fused expression (untimed / long windows: any T).
// Rows past the signal end hold the pad value (masked_fill windows read them).
template <int MODE, bool STAGED>
struct USrc {
  const float* Ls;
  const float* Rs;
  const UParams* p;
  long long row, t0;
  ChildEval cl, cr;
  __device__ __forceinline__ USrc(const float* ls, const float* rs, const UParams* pp, long long r, long long t)
      : Ls(ls), Rs(rs), p(pp), row(r), t0(t), cl(pp->left, r), cr(pp->right, r) {}
  __device__ __forceinline__ float val(const ChildEval& ce, long long j) const {
    if (j < p->L) return ce.value<MODE>(j, p->mp);
    return p->pad_last ? ce.value<MODE>(p->L - 1, p->mp) : p->pad_value;
  }
  __device__ __forceinline__ float l(int e) const { return STAGED ? Ls[e] : val(cl, t0 + e); }
  __device__ __forceinline__ float r(int e) const { return STAGED ? Rs[e] : val(cr, t0 + e); }
};

template <int MODE, bool STAGED>
__device__ __forceinline__ void until_fwd_tile(const UParams& p, long long row, long long t0, float* sm) {
  const long long L = p.L;
  const long long nvalid = (p.untimed || p.fill) ? L : L - p.b;
  const int span = p.untimed ? (int)(L - t0) : U_THREADS + p.b;
  const int nst = (int)((t0 + span <= L || p.fill) ? span : (L - t0));
  const long long rows = p.untimed ? L : L + p.b;  // column height (masked_fill)
  USrc<MODE, STAGED> src(sm, sm + nst, &p, row, t0);
  if (STAGED) {
    if (t0 < nvalid) stage_children<MODE>(p, row, t0, nst, sm, sm + nst);
    __syncthreads();
  }
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
    pm.init(src.l(i0), i0);
    for (int i = 1; i <= p.a; ++i) pm.push(src.l(i0 + i), i0 + i, tau2);
    // outer max over k, in max space of the terms
    float M = 0.f;
    double S = 0.0, Q = 0.0;
    for (int k = 0; k < K; ++k) {
      int e = i0 + p.a + k;
      if (k > 0) pm.push(src.l(e), e, tau2);
      float w1, w2;
      float pmv, rv = src.r(e);
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
          S = 1.0;
        } else {
          lse_add_d(M, S, term, tau2);
        }
      } else {
        if (k == 0) {
          M = term;
          S = 1.0;
          Q = 0.0;
        } else {
          soft_add_d(M, S, Q, term, tau2);
        }
      }
    }
    if (MODE == M_HARD) v = M;
    else if (MODE == M_LSE) v = fmaf(lg2f((float)S), itau2, M);
    else v = M + (float)(Q / S);
    if (p.fill && p.untimed && t > 0) {  // slices past the end: -sentinel terms (masking.py:271-273)
      float lse = (MODE == M_SOFT) ? fmaf(lg2f((float)S), itau2, M) : v;
      fill_merge<MODE>(v, lse, (float)t, p.sent, false, tau2, itau2);
    }
  }
  if (p.canon) v = __fadd_rn(v, 0.f);
  p.out[row * L + t] = v;
}

template <int MODE>
__global__ void __launch_bounds__(U_THREADS) k_until_fwd(const __grid_constant__ UParams p) {
  extern __shared__ __align__(16) float sm[];
  until_fwd_tile<MODE, true>(p, blockIdx.y, (long long)blockIdx.x * U_THREADS, sm);
}
// direct reads: any T (untimed windows longer than shared memory)
template <int MODE>
__global__ void __launch_bounds__(U_THREADS) k_until_fwd_g(const __grid_constant__ UParams p) {
  until_fwd_tile<MODE, false>(p, blockIdx.y, (long long)blockIdx.x * U_THREADS, nullptr);
}

// ---------------------------------------------------------------------------
// warp-systolic scatter: lane i contributes `val` to element base + k + i;
// owner lane o = (i + k) mod 32 accumulates element base + k + ((o - k) mod 32)
// ---------------------------------------------------------------------------
struct Systolic {
  float acc;
  long long cur;   // element currently accumulated by this lane (-1 none)
  float pacc;      // the previous element's finished total, not yet written
  long long pcur;  // (-1 none)
  __device__ __forceinline__ void reset() {
    acc = 0.f;
    cur = -1;
    pacc = 0.f;
    pcur = -1;
  }
  // called by all 32 lanes with the same k (warp-uniform); dst = row base pointer.  A
  // lane's element changes once per 32 consecutive k (at k = lane + 1 mod 32 descending,
  // k = lane ascending): the finished total waits in (pcur, pacc) and every lane writes
  // at once when k = 0 mod 32 — uniform, instead of one diverged lane per step
  __device__ __forceinline__ void step(float val, long long base, int k, const DetRow& dst, long long L) {
    const int lane = threadIdx.x & 31;
    int src = (lane - k) & 31;
    float got = __shfl_sync(0xffffffffu, val, src);
    long long j = base + k + ((lane - k) & 31);
    if (j != cur) {
      pcur = cur;
      pacc = acc;
      cur = j;
      acc = 0.f;
    }
    acc += got;
    if ((k & 31) == 0) put_pending(dst, L);
  }
  // padded positions (masked_fill windows past the end) feed element L - 1 under
  // 'last' padding (pad_last is set by the caller) and nothing under a constant pad
  int pad_last = 0;
  __device__ __forceinline__ void put1(long long e, float v, const DetRow& dst, long long L) const {
    if (e >= 0 && v != 0.f) {
      if (e < L) dst.add(e, v);
      else if (pad_last) dst.add(L - 1, v);
    }
  }
  __device__ __forceinline__ void put_pending(const DetRow& dst, long long L) {
    put1(pcur, pacc, dst, L);
    pcur = -1;
    pacc = 0.f;
  }
  __device__ __forceinline__ void flush(const DetRow& dst, long long L) {
    put_pending(dst, L);
    put1(cur, acc, dst, L);
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
// Checkpoints CK[nck][3] and the block buffer BUF[CB][2] of every thread: in shared
// memory (stride U_THREADS, slot tid) or in a global slab owned by a persistent
// grid (stride = resident threads, slot = global thread index).
struct UScr {
  float* ck;
  float* buf;
  long long stride;  // checkpoints
  long long slot;
  int bstride;       // block buffer (shared memory in both variants)
  int bslot;
  __device__ __forceinline__ float& CK(int i, int c) const { return ck[((long long)i * 3 + c) * stride + slot]; }
  __device__ __forceinline__ float& BUF(int i, int c) const { return buf[(i * 2 + c) * bstride + bslot]; }
};

template <int MODE, bool STAGED, int CB>
__device__ __forceinline__ void until_bwd_tile(const UParams& p, long long row, long long t0, float* sm,
                                               const UScr& scr) {
  const long long L = p.L;
  const long long nvalid = (p.untimed || p.fill) ? L : L - p.b;
  const int span = p.untimed ? (int)(L - t0) : U_THREADS + p.b;
  const int nst = (int)((t0 + span <= L || p.fill) ? span : (L - t0));
  const long long rows = p.untimed ? L : L + p.b;  // column height (masked_fill)
  const int Kmax = p.untimed ? (int)(L - t0) : p.K;
  USrc<MODE, STAGED> src(sm, sm + nst, &p, row, t0);
  const int tid = threadIdx.x;
  const long long t = t0 + tid;
  const bool active = t < nvalid;
  const long long BL = p.B * L;
  const DetRow gl = det_row(p.dacc, p.dacc + BL, p.dscale, row, L, MODE == M_SOFT);
  const DetRow gr = det_row(p.dacc + 2 * BL, p.dacc + 3 * BL, p.dscale, row, L, MODE == M_SOFT);
  const float* cot = p.cot + row * L;
  if (t0 < L) {
    // overrun outputs route to the pad sources (last padding): left if pl <= pr
    if (t < L && !active && p.pad_last) {
      float g = cot[t];
      if (g != 0.f) {
        float pl = expr_eval<MODE>(p.left, row, L - 1, p.mp);
        float pr = expr_eval<MODE>(p.right, row, L - 1, p.mp);
        (pl <= pr ? gl : gr).add(L - 1, g);
      }
    }
  }
  if (t0 >= nvalid) return;  // whole tile overruns (uniform)
  if (STAGED) {
    stage_children<MODE>(p, row, t0, nst, sm, sm + nst);
    __syncthreads();
  }
  (void)Kmax;
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
    pm.init(src.l(tid), tid);
    for (int i = 1; i <= p.a; ++i) pm.push(src.l(tid + i), tid + i, tau2);
    float best = 0.f;
    int bsrc = 0;  // tile-local index; bit 30 set: right child; -1: a sentinel won
    for (int k = 0; k < K; ++k) {
      int e = tid + p.a + k;
      if (k > 0) pm.push(src.l(e), e, tau2);
      float pmv = -pm.m, r = src.r(e);
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
    ((bsrc & (1 << 30)) ? gr : gl).add(j, g);
    return;
  }

  // ---- pass 1: forward over k, checkpoints of the pm state; outer LSE ------------
  PmState<MODE> pm;
  pm.init(src.l(tid), tid);
  for (int i = 1; i <= p.a; ++i) pm.push(src.l(tid + i), tid + i, tau2);
  float Lout = 0.f;  // LSE over the terms (softmax needs it; LSE: equals out)
  {
    float M = 0.f;
    double S = 0.0;
    for (int k = 0; k < K; ++k) {
      int e = tid + p.a + k;
      if (k > 0) pm.push(src.l(e), e, tau2);
      if (k % CB == 0) {
        scr.CK(k / CB, 0) = pm.m;
        scr.CK(k / CB, 1) = (float)pm.s;
        scr.CK(k / CB, 2) = (float)pm.q;
      }
      if (MODE == M_SOFT) {
        float w1, w2;
        float pmv = pm.value(itau2), rv = src.r(e);
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
          S = 1.0;
        } else {
          lse_add_d(M, S, term, tau2);
        }
      }
    }
    if (MODE == M_SOFT && p.fill && p.untimed && t > 0 && K > 0) {
      float Sf = (float)S;
      lse_merge(M, Sf, -p.sent, (float)t, tau2);
      S = Sf;
    }
    Lout = (MODE == M_SOFT) ? fmaf(lg2f((float)S), itau2, M) : out_t;
  }
  // ---- pass 2: backwards over checkpoint blocks -------------------------------
  Systolic accL, accR;
  accL.reset();
  accR.reset();
  accL.pad_last = accR.pad_last = p.pad_last;
  const long long base = t0 + p.a;  // lane i, step k -> element base + k + i (within the warp's t0)
  const int lane = tid & 31;
  const long long wbase = t0 + (tid & ~31) + p.a;
  // suffix accumulators over k, fp64 in a fixed reference frame R: each term gets
  // its own 2^x (no chained per-step rescaling, whose ex2 errors would compound
  // over long windows); R is re-based only when a term would exceed 2^500.
  //   LSE:  A = sum_{k'>=k} c_k' 2^{tau2 (pm_k' - R)}          (R <= pm_k', l space)
  //         dl_e = A 2^{tau2 (R - l_e)}
  //   soft: A = sum c_k' 2^{tau2 (R - Lpm_k')},  Bc = sum c_k' 2^{..} (pm_k' - C)
  //         dl_e = 2^{tau2 (-l_e - R)} [(1 + tau (pm_k - l_e)) A + tau (Bc - (pm_k - C) A)]
  double A = 0.0, Bc = 0.0;
  float R = 0.f, Cc = 0.f;
  bool have = false;
  float pm0 = 0.f;
  for (int cb = (Kw + CB - 1) / CB - 1; cb >= 0; --cb) {
    const int k_lo = cb * CB;
    const int k_hi = min(k_lo + CB, Kw);
    // recompute the block forward from its checkpoint into BUF
    if (k_lo < K) {
      PmState<MODE> st;
      st.m = scr.CK(cb, 0);
      st.s = scr.CK(cb, 1);
      st.q = scr.CK(cb, 2);
      st.i = 0;
      for (int k = k_lo; k < min(k_hi, K); ++k) {
        int e = tid + p.a + k;
        if (k > k_lo) st.push(src.l(e), e, tau2);
        if (p.fill) {  // the filled column's min and LSE
          float MX, lse;
          bool kept;
          pm_mx<MODE>(st, itau2, MX, lse);
          scr.BUF(k - k_lo, 0) = fill_min<MODE>(MX, lse, (float)(rows - (p.a + k + 1)), p.sent, t > 0, tau2, itau2, kept);
          scr.BUF(k - k_lo, 1) = lse;
        } else {
          scr.BUF(k - k_lo, 0) = st.value(itau2);                                          // pm_k
          scr.BUF(k - k_lo, 1) = (MODE == M_SOFT) ? fmaf(lg2f((float)st.s), itau2, st.m) : 0.f;  // L_pm (x space)
        }
      }
    }
    for (int k = k_hi - 1; k >= k_lo; --k) {
      float vr = 0.f, vl = 0.f;
      if (k < K) {
        int e = tid + p.a + k;
        float pmk = scr.BUF(k - k_lo, 0);
        float r = src.r(e);
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
          const float c_pm = g * wk * w1;  // = g exp(tau (2 term - out - pm))
          if (!have) {
            R = pmk;
            have = true;
          } else if (tau2 * (pmk - R) > 500.f) {
            A *= ex2d(tau2 * (R - pmk));
            R = pmk;
          }
          A += (double)c_pm * ex2d(tau2 * (pmk - R));
          // element e = t + a + k receives dpm via exp(tau (pm_k - l_e)) (k >= 1;
          // k == 0 elements are the a-prefix, handled after the loop)
          if (k > 0) vl = (float)(A * ex2d(tau2 * (R - src.l(e))));
          if (k == 0) pm0 = pmk;
        } else {
          float Wk = ex2f(tau2 * (term - Lout)) * fmaf(tau, term - out_t, 1.f);
          vr = g * Wk * w2 * dr;
          const float c_pm = g * Wk * w1;
          const float Lpm = scr.BUF(k - k_lo, 1);
          if (!have) {
            R = Lpm;
            Cc = pmk;
            have = true;
          } else if (tau2 * (R - Lpm) > 500.f) {
            const double f = ex2d(tau2 * (Lpm - R));
            A *= f;
            Bc *= f;
            R = Lpm;
          }
          const double w = (double)c_pm * ex2d(tau2 * (R - Lpm));
          A += w;
          Bc += w * (double)(pmk - Cc);
          if (k > 0) {
            const float l = src.l(e);
            const double sb = Bc - (double)(pmk - Cc) * A;
            vl = (float)(ex2d(tau2 * (-l - R)) * ((1.0 + (double)tau * (pmk - l)) * A + (double)tau * sb));
          }
          if (k == 0) pm0 = pmk;
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
      float l = src.l(tid + i);
      if (MODE == M_LSE) {
        vl = (float)(A * ex2d(tau2 * (R - l)));
      } else {
        const double sb = Bc - (double)(pm0 - Cc) * A;
        vl = (float)(ex2d(tau2 * (-l - R)) * ((1.0 + (double)tau * (pm0 - l)) * A + (double)tau * sb));
      }
    }
    accL.step(vl, wbase - p.a, i, gl, L);
  }
  accL.flush(gl, L);
  (void)lane;
  (void)base;
}

template <int MODE>
__global__ void __launch_bounds__(U_THREADS) k_until_bwd(const __grid_constant__ UParams p) {
  extern __shared__ __align__(16) float sm[];
  const long long L = p.L;
  const long long t0 = (long long)blockIdx.x * U_THREADS;
  const int span = p.untimed ? (int)(L - t0) : U_THREADS + p.b;
  const int nst = (int)((t0 + span <= L || p.fill) ? span : (L - t0));
  const int Kmax = p.untimed ? (int)(L - t0) : p.K;
  const int nck = (Kmax + U_CB_S - 1) / U_CB_S;
  float* ck = sm + 2 * nst;
  UScr scr{ck, ck + (size_t)nck * 3 * U_THREADS, U_THREADS, threadIdx.x, U_THREADS, (int)threadIdx.x};
  until_bwd_tile<MODE, true, U_CB_S>(p, blockIdx.y, t0, sm, scr);
}

// persistent grid, direct child reads, per-thread checkpoints in the global slab
// `p.scratch` (U_CB_G-step blocks): any T, occupancy independent of the window
template <int MODE>
__global__ void __launch_bounds__(U_THREADS) k_until_bwd_g(const __grid_constant__ UParams p, int ntx,
                                                            long long ntiles) {
  extern __shared__ __align__(16) float sm[];  // block buffer [U_CB_G][2][U_THREADS]
  const long long stride = (long long)gridDim.x * U_THREADS;
  UScr scr{p.scratch, sm, stride, (long long)blockIdx.x * U_THREADS + threadIdx.x, U_THREADS,
           (int)threadIdx.x};
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row = tile / ntx;
    const long long t0 = (tile - row * ntx) * U_THREADS;
    until_bwd_tile<MODE, false, U_CB_G>(p, row, t0, nullptr, scr);
    __syncwarp();
  }
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

// Two shapes (as fg_unt.cu): LB = false, one CTA of 256 threads per row walking its
// 2048-sample chunks with the carry in registers (large batches); LB = true, one CTA of
// 128 threads per 1024-sample chunk (grid: chunks x rows, blockIdx.x = scan index) that
// publishes its aggregate (forward: the composed clamp; backward: the segmented run sum)
// and folds the aggregates of the chunks before it in scan order (lookback.cuh).
constexpr int UH_E = 8, UH_S = UH_E + 1, UH_SEQ = 256, UH_LB = 128;
static_assert(UH_LB * UH_E == LB_MIN_TILE, "look-back slots are sized for 1024-sample tiles");
__device__ __forceinline__ int uhpos(int k) { return (k >> 3) * UH_S + (k & 7); }

template <int MODE, bool LB>
__global__ void __launch_bounds__(LB ? UH_LB : UH_SEQ) k_until_unt_hard_fwd(const __grid_constant__ UParams p) {
  constexpr int UH_T = LB ? UH_LB : UH_SEQ, UH_CH = UH_T * UH_E;
  __shared__ float Ls[UH_T * UH_S];
  __shared__ float Rs[UH_T * UH_S];
  __shared__ Clamp cb[UH_T / 32];
  const int L = (int)p.L;  // < 2^31 (launcher)
  const int nch = (L + UH_CH - 1) / UH_CH;
  const int tk = LB ? lb_ticket(p.lb) : 0;  // look-back shape: (row, chunk) from a ticket
  const long long row = LB ? tk / nch : blockIdx.x;
  const int tid = threadIdx.x;
  const ChildEval cl(p.left, row), cr(p.right, row);
  unsigned* slots = LB ? p.lb + LB_WORDS + (size_t)row * nch * LB_WORDS : nullptr;
  // f_{L-1}(-inf) = A_{L-1}: the recurrence starts uniformly from -inf
  float seq = -INFINITY;  // sequential shape: the value entering the current chunk
  for (int s = LB ? tk - (int)row * nch : 0; s < (LB ? tk - (int)row * nch + 1 : nch); ++s) {
  const int c0 = (nch - 1 - s) * UH_CH;  // scan order: from the row end
  {  // all of the thread's loads in flight before the first store
    float lv[UH_E], rv[UH_E];
    if (cl.kind != 0 && cr.kind != 0) {
#pragma unroll
      for (int e = 0; e < UH_E; ++e) {
        const int t = c0 + tid + e * UH_T;
        const int tc = t < L ? t : L - 1;
        lv[e] = cl.raw(tc);
        rv[e] = cr.raw(tc);
      }
#pragma unroll
      for (int e = 0; e < UH_E; ++e) {
        const bool in = c0 + tid + e * UH_T < L;
        lv[e] = in ? cl.apply(lv[e]) : 0.f;
        rv[e] = in ? cr.apply(rv[e]) : 0.f;
      }
    } else {
#pragma unroll
      for (int e = 0; e < UH_E; ++e) {
        const int t = c0 + tid + e * UH_T;
        lv[e] = t < L ? cl.value<MODE>(t, p.mp) : 0.f;
        rv[e] = t < L ? cr.value<MODE>(t, p.mp) : 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < UH_E; ++e) {
      Ls[uhpos(tid + e * UH_T)] = lv[e];
      Rs[uhpos(tid + e * UH_T)] = rv[e];
    }
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
  // suffix composition over the later threads: warp shuffles, then the later warps
  const int lane = tid & 31, warp = tid >> 5;
  Clamp C = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Clamp n{__shfl_down_sync(0xffffffffu, C.lo, o), __shfl_down_sync(0xffffffffu, C.hi, o)};
    if (lane + o < 32) C = clamp_compose(C, n);
  }
  Clamp ex{__shfl_down_sync(0xffffffffu, C.lo, 1), __shfl_down_sync(0xffffffffu, C.hi, 1)};
  if (lane == 31) ex = Clamp{-INFINITY, INFINITY};
  if (lane == 0) cb[warp] = C;
  __syncthreads();
  float carry = seq;
  if (LB) {
    if (tid == 0 && s + 1 < nch) {  // the chunk's function cb[0] o cb[1] o ... (later last)
      Clamp F = cb[UH_T / 32 - 1];
      for (int w = UH_T / 32 - 2; w >= 0; --w) F = clamp_compose(cb[w], F);
      const unsigned pw[2] = {__float_as_uint(F.lo), __float_as_uint(F.hi)};
      lb_publish<2>(slots + (size_t)s * LB_WORDS, pw);
    }
    // the value entering the chunk: the later chunks' functions applied in scan order
    carry = lb_carry<2>(slots, s, -INFINITY, [](float x, const unsigned* w) {
      return clamp_apply(Clamp{__uint_as_float(w[0]), __uint_as_float(w[1])}, x);
    });
  }
  float vw = carry;  // the carry pushed through the later warps of the chunk
  for (int w = UH_T / 32 - 1; w > warp; --w) vw = clamp_apply(cb[w], vw);
  float v = clamp_apply(ex, vw);
  for (int e = UH_E - 1; e >= 0; --e) {  // exact sequential walk with the reference tie rules
    if (c0 + tid * UH_E + e >= L) continue;
    float l = Ls[tid * UH_S + e], r = Rs[tid * UH_S + e];
    float A = (l <= r) ? l : r;
    float Bv = (l <= v) ? l : v;
    v = (A >= Bv) ? A : Bv;
    Ls[tid * UH_S + e] = v;
  }
  __syncthreads();
  if (!LB) seq = Ls[0];
  for (int k = tid; k < UH_CH; k += UH_T) {
    const int t = c0 + k;
    if (t < L) p.out[row * L + t] = Ls[uhpos(k)];
  }
  __syncthreads();
  }
}

// backward: terminator test per t with the stored out[t+1]; runs of equal
// source end at their terminator, whose own index is the source index, so
// each child cotangent is final when its run ends (no atomics, fused VJPs).
// Chunk carry: the cotangent accumulated since the last terminator in the chunks
// before (scan order from the row start).
template <int MODE, bool LB>
__global__ void __launch_bounds__(LB ? UH_LB : UH_SEQ) k_until_unt_hard_bwd(const __grid_constant__ UParams p) {
  constexpr int UH_T = LB ? UH_LB : UH_SEQ, UH_CH = UH_T * UH_E;
  __shared__ float Ls[UH_T * UH_S], Rs[UH_T * UH_S], Os[UH_T * UH_S], Gs[UH_T * UH_S];
  __shared__ double wsum[UH_T / 32];
  __shared__ int wflag[UH_T / 32];
  const int L = (int)p.L;  // < 2^31 (launcher)
  const int nch = (L + UH_CH - 1) / UH_CH;
  const int tk = LB ? lb_ticket(p.lb) : 0;  // look-back shape: (row, chunk) from a ticket
  const long long row = LB ? tk / nch : blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* outr = p.out_in + row * L;
  const float* cot = p.cot + row * L;
  const ChildEval cl(p.left, row), cr(p.right, row);
  unsigned* slots = LB ? p.lb + LB_WORDS + (size_t)row * nch * LB_WORDS : nullptr;
  double seq = 0.0;  // sequential shape: cotangent accumulated since the last terminator
  for (int s = LB ? tk - (int)row * nch : 0; s < (LB ? tk - (int)row * nch + 1 : nch); ++s) {
  const int c0 = s * UH_CH;
  {  // coalesced staging of l, r, out[t + 1] and the cotangent, all loads in flight first
    float lv[UH_E], rv[UH_E], ov[UH_E], gv[UH_E];
    const bool fast = cl.kind != 0 && cr.kind != 0;
#pragma unroll
    for (int e = 0; e < UH_E; ++e) {
      const int t = c0 + tid + e * UH_T;
      const int tc = t < L ? t : L - 1;
      const int to = t + 1 < L ? t + 1 : L - 1;
      if (fast) {
        lv[e] = cl.raw(tc);
        rv[e] = cr.raw(tc);
      }
      ov[e] = outr[to];
      gv[e] = cot[tc];
    }
#pragma unroll
    for (int e = 0; e < UH_E; ++e) {
      const int t = c0 + tid + e * UH_T;
      const bool in = t < L;
      if (fast) {
        lv[e] = in ? cl.apply(lv[e]) : 0.f;
        rv[e] = in ? cr.apply(rv[e]) : 0.f;
      } else {
        lv[e] = in ? cl.value<MODE>(t, p.mp) : 0.f;
        rv[e] = in ? cr.value<MODE>(t, p.mp) : 0.f;
      }
      ov[e] = (t + 1 < L) ? ov[e] : 0.f;
      gv[e] = in ? gv[e] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < UH_E; ++e) {
      const int q = uhpos(tid + e * UH_T);
      Ls[q] = lv[e];
      Rs[q] = rv[e];
      Os[q] = ov[e];
      Gs[q] = gv[e];
    }
  }
  __syncthreads();
  float g[UH_E];
  int term[UH_E];  // 0: pass to the next sample's source, 1: l_t, 2: r_t
  double tail = 0.0;
  int anyterm = 0;
#pragma unroll
  for (int e = 0; e < UH_E; ++e) {
    const int t = c0 + tid * UH_E + e;
    const int q = tid * UH_S + e;
    term[e] = 0;
    g[e] = 0.f;
    if (t < L) {
      const float l = Ls[q], r = Rs[q];
      const bool a_is_l = l <= r;
      const float A = a_is_l ? l : r;
      int src;
      if (t == L - 1) {
        src = a_is_l ? 1 : 2;
      } else {
        const float v = Os[q];
        const bool b_is_l = l <= v;
        const float Bv = b_is_l ? l : v;
        src = (A >= Bv) ? (a_is_l ? 1 : 2) : (b_is_l ? 1 : 0);
      }
      term[e] = src;
      g[e] = Gs[q];
      if (src) {
        anyterm = 1;
        tail = 0.0;
      } else {
        tail += (double)g[e];
      }
    }
  }
  // exclusive segmented prefix (sum since the last terminator) over the earlier threads:
  // (s, f) then (s', f')  ->  (f' ? s' : s + s', f | f'); warp shuffles, then the warps
  double is = tail;
  int iflag = anyterm;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ps = __shfl_up_sync(0xffffffffu, is, o);
    const int pf = __shfl_up_sync(0xffffffffu, iflag, o);
    if (lane >= o) {
      if (!iflag) is += ps;
      iflag |= pf;
    }
  }
  double xs = __shfl_up_sync(0xffffffffu, is, 1);
  int xf = __shfl_up_sync(0xffffffffu, iflag, 1);
  if (lane == 0) xs = 0.0, xf = 0;
  if (lane == 31) {
    wsum[warp] = is;
    wflag[warp] = iflag;
  }
  __syncthreads();
  double carry = seq;
  if (LB) {
    if (tid == 0 && s + 1 < nch) {  // the chunk's (sum since its last terminator, any terminator)
      double cs = 0.0;
      int cf = 0;
      for (int w = 0; w < UH_T / 32; ++w) {
        cs = wflag[w] ? wsum[w] : cs + wsum[w];
        cf |= wflag[w];
      }
      const unsigned long long b = (unsigned long long)__double_as_longlong(cs);
      const unsigned pw[3] = {(unsigned)b, (unsigned)(b >> 32), (unsigned)cf};
      lb_publish<3>(slots + (size_t)s * LB_WORDS, pw);
    }
    carry = lb_carry<3>(slots, s, 0.0, [](double x, const unsigned* w) {
      const double cs = __longlong_as_double((long long)((unsigned long long)w[0] | ((unsigned long long)w[1] << 32)));
      return w[2] ? cs : x + cs;
    });
  } else {
    for (int w = 0; w < UH_T / 32; ++w) seq = wflag[w] ? wsum[w] : seq + wsum[w];
  }
  double before = carry;  // carry, then the earlier warps, then the earlier lanes
  for (int w = 0; w < warp; ++w) before = wflag[w] ? wsum[w] : before + wsum[w];
  double run = xf ? xs : before + xs;
  // the thread's gradients into its own staging slots (l -> Ls, r -> Rs)
#pragma unroll
  for (int e = 0; e < UH_E; ++e) {
    const int q = tid * UH_S + e;
    run += (double)g[e];
    float gl = 0.f, gr = 0.f;
    if (term[e] == 1) {
      gl = (float)run;
      run = 0.0;
    } else if (term[e] == 2) {
      gr = (float)run;
      run = 0.0;
    }
    Ls[q] = gl;
    Rs[q] = gr;
  }
  __syncthreads();
  // coalesced child VJPs (left first: first-writer order)
  for (int k = tid; k < UH_CH; k += UH_T) {
    const int t = c0 + k;
    if (t >= L) break;
    const int q = uhpos(k);
    cl.grad<MODE>(t, Ls[q], p.mp);
    cr.grad<MODE>(t, Rs[q], p.mp);
  }
  __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// untimed LogSumExp Until in reciprocal form (non-fill)
// ---------------------------------------------------------------------------
// With S_k(t) = sum_{j=t..k} e^{-tau l_j} and E_k = e^{-tau r_k}, the reference's
// incremental pm_k gives e^{-tau pm_k} = S_k, its two-element LSE-min gives
// e^{tau term_k} = 1 / (S_k + E_k) =: 1 / D_k, and the outer LSE-max is
//   out[t] = (1/tau) ln A_t,   A_t = sum_{k >= t} 1 / D_k(t)        (same function)
// with the VJP
//   d out / d r_k = E_k D_k^-2 / A_t,   d out / d l_j = e_j sum_{k >= j} D_k^-2 / A_t.
// Still O(T^2) pairs, but one reciprocal per pair instead of the per-pair ex2 / lg2 of
// the incremental form.  Columns come in chunks of 32 (one warp's share of a
// 128-column stage): the chunk's fp64 prefix Q_k and B_k = Q_k + E_k are shared by
// every output t before the chunk, D_k(t) = base_t + B_k with base_t = S over
// [t, chunk start) (built by additions only: no cancellation), and each thread
// evaluates its pairs in fp32 under a per-chunk power-of-two frame that puts its
// largest terms at ~1 (smaller terms may flush: they are below 2^-100 of the sum).
// A thread's own chunk is done exactly in fp64.  Rows whose values span more than
// UL_RANGE log2 units (or hold non-finite values) run the per-pair kernels'
// tile functions inside the same launch.
constexpr int UL_T = 128;
constexpr int UL_C = 32;
constexpr float UL_RANGE = 400.f;
#ifndef UL_MINB
#define UL_MINB 3  // backward: 168 registers, no spills (the default 128 spills)
#endif

struct UlStage {
  double ex[UL_T], E[UL_T];  // e^{-tau l}, e^{-tau r} under the tile frame F
  float bk[UL_T];            // B_k / 2^fmin
  float rho[UL_T], eta[UL_T];  // E_k / B_k, e_k / B_k (backward)
  double qtot[4], bmin[4];
  int fmin[4];
};

// 1 / x for x in the frames' normal fp64 range: the MUFU seed plus one Newton step
// (~2^-44 relative; a correctly rounded fp64 division or __drcp_rn is a long sequence)
__device__ __forceinline__ double ur_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ int ilogb_d(double x) { return (int)((__double2hiint(x) >> 20) & 0x7ff) - 1023; }
__device__ __forceinline__ double pow2d(int e) { return __hiloint2double((e + 1023) << 20, 0); }
__device__ __forceinline__ float pow2f(int e) {
  if (e < -126) return 0.f;
  return __int_as_float((min(e, 127) + 127) << 23);
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// tile frame F = max over [t0, kend) of -tau2 l and -tau2 r (kend = L untimed, the last
// window end of the tile timed); false: take the per-pair path
__device__ __forceinline__ bool ul_frame(const UParams& p, long long row, long long t0, long long kend, float& F,
                                         float* red) {
  const float tau2 = p.mp.tau2;
  float hi = -INFINITY, lo = INFINITY;
  bool ok = true;
  for (long long k = t0 + threadIdx.x; k < kend; k += UL_T) {
    const float u = -tau2 * expr_eval<M_LSE>(p.left, row, k, p.mp);
    const float v = -tau2 * expr_eval<M_LSE>(p.right, row, k, p.mp);
    ok = ok && isfinite(u) && isfinite(v);
    hi = fmaxf(hi, fmaxf(u, v));
    lo = fminf(lo, fminf(u, v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[w] = hi;
    red[4 + w] = lo;
  }
  ok = __syncthreads_and(ok);
  hi = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  lo = fminf(fminf(red[4], red[5]), fminf(red[6], red[7]));
  F = hi;
  __syncthreads();
  return ok && hi - lo <= UL_RANGE;
}

// one 128-column stage at k0: warp w builds chunk w
template <bool BWD>
__device__ __forceinline__ void ul_stage(const UParams& p, long long row, long long k0, float F, UlStage& S) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long k = k0 + tid;
  const bool valid = k < p.L;
  const float tau2 = p.mp.tau2;
  double ex = 0.0, E = 0.0;
  if (valid) {
    ex = ex2d(fmaf(-tau2, expr_eval<M_LSE>(p.left, row, k, p.mp), -F));
    E = ex2d(fmaf(-tau2, expr_eval<M_LSE>(p.right, row, k, p.mp), -F));
  }
  double qc = ex;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, qc, o);
    if (lane >= o) qc += y;
  }
  const double B = qc + E;
  double bm = valid ? B : INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bm = fmin(bm, __shfl_xor_sync(0xffffffffu, bm, o));
  const int fm = ilogb_d(bm);  // warp-uniform (unused when the whole chunk is past L)
  S.ex[tid] = ex;
  S.E[tid] = E;
  S.bk[tid] = valid ? (float)fmin(B * pow2d(-fm), 3.0e38) : 3.0e38f;
  if (BWD) {
    S.rho[tid] = valid ? (float)(E / B) : 0.f;
    S.eta[tid] = valid ? (float)(ex / B) : 0.f;
  }
  if (lane == 31) {
    S.qtot[w] = qc;
    S.bmin[w] = bm;
    S.fmin[w] = fm;
  }
}

// sum over the chunk of 1 / D_k(t), D = base + B (fp64 result, tile frame)
__device__ __forceinline__ double ul_chunk_fwd(const UlStage& S, int c, int n, double base) {
  const double den = base + S.bmin[c];
  const int g = -ilogb_d(den);                 // den 2^g in [1, 2): every D 2^g >= 1
  const float scale = pow2f(S.fmin[c] + g);    // <= 1
  const float bb = (float)(base * pow2d(g));
  const float* bk = S.bk + c * UL_C;
  float s0 = 0.f, s1 = 0.f;
  if (n == UL_C) {
#pragma unroll
    for (int j = 0; j < UL_C; j += 2) {
      s0 += rcp_approx(fmaf(bk[j], scale, bb));
      s1 += rcp_approx(fmaf(bk[j + 1], scale, bb));
    }
  } else {
    for (int j = 0; j < n; ++j) s0 += rcp_approx(fmaf(bk[j], scale, bb));
  }
  return (double)(s0 + s1) * pow2d(g);
}

// the same sum over the chunk columns [jlo, jhi) only (timed windows cut chunks)
__device__ __forceinline__ double ul_chunk_fwd_rng(const UlStage& S, int c, int jlo, int jhi, double base) {
  const double den = base + S.bmin[c];
  const int g = -ilogb_d(den);
  const float scale = pow2f(S.fmin[c] + g);
  const float bb = (float)(base * pow2d(g));
  const float* bk = S.bk + c * UL_C;
  float s0 = 0.f;
  for (int j = jlo; j < jhi; ++j) s0 += rcp_approx(fmaf(bk[j], scale, bb));
  return (double)s0 * pow2d(g);
}

// overrun output (t + b > L-1, timed): the hard min of the pad values in every mode
// (masking.py:180-192); its gradient source: left if pl <= pr
__device__ __forceinline__ void ul_pads(const UParams& p, long long row, float& pl, float& pr) {
  pl = p.pad_value;
  pr = p.pad_value;
  if (p.pad_last) {
    pl = expr_eval<M_LSE>(p.left, row, p.L - 1, p.mp);
    pr = expr_eval<M_LSE>(p.right, row, p.L - 1, p.mp);
  }
}

// Reciprocal form, untimed (every column k >= t) or timed (columns [t + a, t + b]; the pm
// sum still starts at t, so base accumulates every column from t on).
template <bool TIMED>
__global__ void __launch_bounds__(UL_T) k_until_rcp_lse_fwd(const __grid_constant__ UParams p) {
  __shared__ UlStage S;
  __shared__ float red[8];
  const long long row = blockIdx.y, t0 = (long long)blockIdx.x * UL_T;
  const long long L = p.L;
  const long long kend = TIMED ? min(L, t0 + UL_T - 1 + p.b + 1) : L;  // columns the tile reads
  float F;
  if (!ul_frame(p, row, t0, kend, F, red)) {
    until_fwd_tile<M_LSE, false>(p, row, t0, nullptr);
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long t = t0 + tid;
  const bool live = !TIMED || t + p.b <= L - 1;
  const long long u = TIMED ? t + p.a : t, v = TIMED ? (live ? t + p.b : -1) : L - 1;  // columns
  double A = 0.0, base = 0.0;
  for (long long k0 = t0; k0 < kend; k0 += UL_T) {
    __syncthreads();
    ul_stage<false>(p, row, k0, F, S);
    __syncthreads();
    const bool diag = k0 == t0;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      const long long c0 = k0 + c * UL_C;
      if (c0 >= kend) break;
      const int n = (int)min((long long)UL_C, L - c0);
      if (diag && c == w) {  // the thread's own chunk, exactly
        double s = 0.0;
        for (int j = lane; j < n; ++j) {
          s += S.ex[c * UL_C + j];
          const long long col = c0 + j;
          if (!TIMED || (col >= u && col <= v)) A += ur_rcp(s + S.E[c * UL_C + j]);
        }
        base = s;
      } else if (!diag || c > w) {
        if (!TIMED) {
          A += ul_chunk_fwd(S, c, n, base);
        } else if (c0 <= v && c0 + n > u) {
          const int jlo = (int)max(0LL, u - c0), jhi = (int)min((long long)n, v - c0 + 1);
          A += (jlo == 0 && jhi == n) ? ul_chunk_fwd(S, c, n, base) : ul_chunk_fwd_rng(S, c, jlo, jhi, base);
        }
        base += S.qtot[c];
      }
    }
  }
  if (t < L) {
    float o;
    if (live) {
      o = (float)((log2(A) - (double)F) / (double)p.mp.tau2);
    } else {
      float pl, pr;
      ul_pads(p, row, pl, pr);
      o = (pl <= pr) ? pl : pr;
    }
    p.out[row * L + t] = p.canon ? __fadd_rn(o, 0.f) : o;
  }
}

// Timed LSE Until backward in reciprocal form, one thread per output t (the per-output
// kernels' structure, the reciprocal form's arithmetic): with ex_j = e^{-tau l_j},
// E_s = e^{-tau r_s} staged in fp64 under the tile frame and D_s = sum_{j=t..s} ex_j + E_s,
//   A = sum_{s in [u, v]} 1 / D_s,   d out / d r_s = E_s D_s^-2 / A,
//   d out / d l_j = ex_j sum_{s >= max(j, u)} D_s^-2 / A,
// pass 1 accumulates S and A ascending with a checkpoint of S every UR_CB columns, pass 2
// walks the blocks descending (q = 1/D recomputed from the checkpoint into QB), and the
// contributions scatter warp-systolically into the reproducible int64 accumulators.
// Tiles whose values span more than UL_RANGE log2 units run the per-pair tile function
// (global-slab checkpoints; the grid is persistent for that slab).
constexpr int UR_CB = 16;
__host__ __device__ __forceinline__ int ur_span(int b) { return U_THREADS + b; }

static size_t ur_smem(const UParams& p) {
  const size_t qb = (size_t)UR_CB * U_THREADS * 8;
  const size_t st = (size_t)2 * ur_span(p.b) * 8;
  const size_t ck = (size_t)((p.K + UR_CB - 1) / UR_CB) * U_THREADS * 8;
  const size_t fallback = (size_t)U_CB_G * 2 * U_THREADS * 4;  // the per-pair tiles' block buffer
  return max(qb + st + ck, fallback);
}

__global__ void __launch_bounds__(U_THREADS) k_until_rcp_lse_bwd_timed(const __grid_constant__ UParams p, int ntx,
                                                                      long long ntiles) {
  extern __shared__ __align__(16) float dsm[];
  __shared__ float red[8];
  const long long L = p.L;
  const int K = p.K, tid = threadIdx.x, span = ur_span(p.b);
  double* QB = reinterpret_cast<double*>(dsm);  // [UR_CB][U_THREADS] (the fallback's block buffer
                                                //  overlays the start of the region)
  double* EXs = QB + UR_CB * U_THREADS;           // [span]
  double* ERs = EXs + span;                       // [span]
  double* CK = ERs + span;                        // [ceil(K / UR_CB)][U_THREADS]
  const long long stride = (long long)gridDim.x * U_THREADS;
  UScr scr{p.scratch, dsm, stride, (long long)blockIdx.x * U_THREADS + tid, U_THREADS, tid};
  const long long BL = p.B * L;
  const float tau2 = p.mp.tau2;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row = tile / ntx;
    const long long t0 = (tile - row * ntx) * U_THREADS;
    const long long t = t0 + tid;
    const long long kend = min(L, t0 + span);
    float g = t < L ? p.cot[row * L + t] : 0.f;
    if (!__syncthreads_or(g != 0.f)) continue;
    float F;
    if (!ul_frame(p, row, t0, kend, F, red)) {
      until_bwd_tile<M_LSE, false, U_CB_G>(p, row, t0, nullptr, scr);
      __syncthreads();
      continue;
    }
    const DetRow gl = det_row(p.dacc, p.dacc + BL, p.dscale, row, L, false);
    const DetRow gr = det_row(p.dacc + 2 * BL, p.dacc + 3 * BL, p.dscale, row, L, false);
    if (t < L && t + p.b > L - 1) {  // overrun output: the whole cotangent to the pad source
      if (p.pad_last && g != 0.f) {
        float pl, pr;
        ul_pads(p, row, pl, pr);
        (pl <= pr ? gl : gr).add(L - 1, g);
      }
      g = 0.f;
    }
    for (int c = tid; c < span; c += U_THREADS) {
      const long long j = t0 + c;
      double ex = 0.0, E = 0.0;
      if (j < L) {
        ex = ex2d(fmaf(-tau2, expr_eval<M_LSE>(p.left, row, j, p.mp), -F));
        E = ex2d(fmaf(-tau2, expr_eval<M_LSE>(p.right, row, j, p.mp), -F));
      }
      EXs[c] = ex;
      ERs[c] = E;
    }
    __syncthreads();
    // pass 1: A, checkpoints of S (before each block's first column)
    double A = 0.0;
    if (g != 0.f) {
      double S = 0.0;
      for (int i = 0; i < p.a; ++i) S += EXs[tid + i];
      for (int k = 0; k < K; ++k) {
        const int c = tid + p.a + k;
        if (k % UR_CB == 0) CK[(k / UR_CB) * U_THREADS + tid] = S;
        S += EXs[c];
        A += ur_rcp(S + ERs[c]);
      }
    }
    const double cA = (g != 0.f) ? (double)g / A : 0.0;
    // pass 2: descending blocks
    Systolic accL, accR;
    accL.reset();
    accR.reset();
    accL.pad_last = accR.pad_last = p.pad_last;
    const long long wbase = t0 + (tid & ~31) + p.a;  // lane i, step k -> element wbase + k + i
    double R = 0.0;
    for (int cb = (K + UR_CB - 1) / UR_CB - 1; cb >= 0; --cb) {
      const int k_lo = cb * UR_CB, k_hi = min(k_lo + UR_CB, K);
      if (cA != 0.0) {
        double S = CK[cb * U_THREADS + tid];
        for (int k = k_lo; k < k_hi; ++k) {
          const int c = tid + p.a + k;
          S += EXs[c];
          QB[(k - k_lo) * U_THREADS + tid] = ur_rcp(S + ERs[c]);
        }
      }
      for (int k = k_hi - 1; k >= k_lo; --k) {
        float vr = 0.f, vl = 0.f;
        if (cA != 0.0) {
          const int c = tid + p.a + k;
          const double q = QB[(k - k_lo) * U_THREADS + tid];
          const double q2 = q * q;
          R += q2;
          vr = (float)(cA * ERs[c] * q2);
          if (k > 0) vl = (float)(cA * EXs[c] * R);  // k = 0 (s = u) joins the a-prefix below
        }
        accR.step(vr, wbase, k, gr, L);
        accL.step(vl, wbase, k, gl, L);
      }
    }
    accR.flush(gr, L);
    accL.flush(gl, L);
    // l_j for j in [t, u]: every window column, sum_{s >= u} D_s^-2 = R
    for (int i = 0; i <= p.a; ++i) {
      const float vl = (cA != 0.0) ? (float)(cA * EXs[tid + i] * R) : 0.f;
      accL.step(vl, wbase - p.a, i, gl, L);
    }
    accL.flush(gl, L);
    __syncthreads();  // before the next tile's staging
  }
}

// 32 values per lane -> lane i holds the warp's sum of value i
// column sums of a warp's 32 x 32 block through a padded shared transpose (row
// stride 36 floats: conflict-free 128-bit row stores and column loads); lane i
// returns the sum of value i over the warp
__device__ __forceinline__ float warp_colsum(const float (&v)[UL_C], float* buf) {
  const int lane = threadIdx.x & 31;
  float* rowp = buf + lane * 36;
#pragma unroll
  for (int m = 0; m < UL_C / 4; ++m)
    *reinterpret_cast<float4*>(rowp + 4 * m) = make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
  __syncwarp();
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int l = 0; l < 32; l += 2) {
    s0 += buf[l * 36 + lane];
    s1 += buf[(l + 1) * 36 + lane];
  }
  __syncwarp();
  return s0 + s1;
}

// descending pass over one off-diagonal chunk: column sums of
//   P_k = g E_k D_k^-2 / A  (-> d r_k),   Q_k = g e_k R_k / A,  R_k = sum_{k'>=k} D_k'^-2 (-> d l_k)
// in the thread's frame g (the smallest D of this chunk and the tail at ~1); R
// carried in fp64 across chunks (Rt64, frame gprev)
__device__ __forceinline__ void ul_chunk_bwd(const UlStage& S, int c, int n, double base, double A, float gt,
                                             double& dtail, double& Rt64, int& gprev, float* colP,
                                             float* colQ, float* wbuf) {
  const int lane = threadIdx.x & 31;
  const double den = base + S.bmin[c];
  const double dmin = fmin(den, dtail);
  const int g = -ilogb_d(dmin);
  if (Rt64 != 0.0) Rt64 *= pow2d(-2 * (g - gprev));
  gprev = g;
  const float scale = pow2f(min(S.fmin[c] + g, 126));
  const float bb = (float)(base * pow2d(g));
  const float gl = (gt == 0.f) ? 0.f : (float)((double)gt * (pow2d(g) / A));
  const float rt = (float)Rt64;
  const float* bk = S.bk + c * UL_C;
  const float* rho = S.rho + c * UL_C;
  const float* eta = S.eta + c * UL_C;
  float P[UL_C], Q[UL_C];
  float rr = 0.f;
  auto pair = [&](int j, float b, float r, float e) {
    const float t1 = fminf(b * scale, 0x1p120f);  // B_k in the frame
    const float q = rcp_approx(t1 + bb);          // 1 / D_k
    const float gq = gl * q;
    P[j] = gq * (r * t1 * q);
    rr = fmaf(q, q, rr);
    Q[j] = gl * (e * t1) * (rt + rr);
  };
  if (n == UL_C) {
#pragma unroll
    for (int m = UL_C / 4 - 1; m >= 0; --m) {
      const float4 b4 = reinterpret_cast<const float4*>(bk)[m];
      const float4 r4 = reinterpret_cast<const float4*>(rho)[m];
      const float4 e4 = reinterpret_cast<const float4*>(eta)[m];
      pair(4 * m + 3, b4.w, r4.w, e4.w);
      pair(4 * m + 2, b4.z, r4.z, e4.z);
      pair(4 * m + 1, b4.y, r4.y, e4.y);
      pair(4 * m, b4.x, r4.x, e4.x);
    }
  } else {
#pragma unroll
    for (int j = UL_C - 1; j >= 0; --j) {
      if (j < n) {
        pair(j, bk[j], rho[j], eta[j]);
      } else {
        P[j] = 0.f;
        Q[j] = 0.f;
      }
    }
  }
  Rt64 += (double)rr;
  dtail = dmin;
  // per-warp slots (summed in warp order after the stage): no shared float atomics
  const int w = threadIdx.x >> 5;
  colP[w * UL_T + c * UL_C + lane] = warp_colsum(P, wbuf);
  colQ[w * UL_T + c * UL_C + lane] = warp_colsum(Q, wbuf);
}

// persistent grid; tiles that fail the range check run the per-pair backward with
// its checkpoints in the global slab (same layout as k_until_bwd_g)
__global__ void __launch_bounds__(UL_T, UL_MINB) k_until_unt_lse_bwd(const __grid_constant__ UParams p, int ntx,
                                                             long long ntiles) {
  // block buffer of the per-pair fallback [U_CB_G][2][UL_T] (the fast path's per-warp
  // transpose tiles [4][32][36] when the tile takes the fast path), then CQ[nch]
  extern __shared__ __align__(16) float dsm[];
  __shared__ UlStage S;
  __shared__ float colP[(UL_T / 32) * UL_T], colQ[(UL_T / 32) * UL_T];  // [warp][column]
  __shared__ float red[8];
  const long long stride = (long long)gridDim.x * U_THREADS;
  UScr scr{p.scratch, dsm, stride, (long long)blockIdx.x * U_THREADS + threadIdx.x, U_THREADS,
           (int)threadIdx.x};
  double* CQ = (double*)(dsm + U_CB_G * 2 * U_THREADS);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long L = p.L;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row = tile / ntx;
    const long long t0 = (tile - row * ntx) * UL_T;
    const long long t = t0 + tid;
    const float gt = t < L ? p.cot[row * L + t] : 0.f;
    if (!__syncthreads_or(gt != 0.f)) continue;
    float F;
    if (!ul_frame(p, row, t0, L, F, red)) {
      until_bwd_tile<M_LSE, false, U_CB_G>(p, row, t0, nullptr, scr);
      __syncthreads();
      continue;
    }
    // ---- pass 1 (ascending): A_t, the thread's own-chunk sum, base after the first stage,
    //      and the running chunk totals CQ (chunks of later stages)
    double A = 0.0, base = 0.0, sown = 0.0, head = 0.0, X = 0.0;
    int ci = 0;
    for (long long k0 = t0; k0 < L; k0 += UL_T, ci += 4) {
      __syncthreads();
      ul_stage<false>(p, row, k0, F, S);
      __syncthreads();
      const bool diag = k0 == t0;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const long long c0 = k0 + c * UL_C;
        if (c0 >= L) break;
        const int n = (int)min((long long)UL_C, L - c0);
        if (tid == 0) {
          CQ[ci + c] = X;
          if (!diag) X += S.qtot[c];
        }
        if (diag && c == w) {
          double s = 0.0;
          for (int j = lane; j < n; ++j) {
            s += S.ex[c * UL_C + j];
            A += ur_rcp(s + S.E[c * UL_C + j]);
          }
          sown = s;
          base = s;
        } else if (!diag || c > w) {
          A += ul_chunk_fwd(S, c, n, base);
          base += S.qtot[c];
        }
      }
      if (diag) head = base;
    }
    // ---- pass 2 (descending)
    double dtail = INFINITY, Rt64 = 0.0;
    int gprev = 0;
    const int nstage = (int)((L - t0 + UL_T - 1) / UL_T);
    const long long BL = p.B * L;
    const DetRow gl_row = det_row(p.dacc, p.dacc + BL, p.dscale, row, L, false);
    const DetRow gr_row = det_row(p.dacc + 2 * BL, p.dacc + 3 * BL, p.dscale, row, L, false);
    for (int s = nstage - 1; s >= 0; --s) {
      const long long k0 = t0 + (long long)s * UL_T;
      __syncthreads();
      ul_stage<true>(p, row, k0, F, S);
      for (int q = tid; q < (UL_T / 32) * UL_T; q += UL_T) colP[q] = colQ[q] = 0.f;
      __syncthreads();
      const bool diag = s == 0;
#pragma unroll 1
      for (int c = 3; c >= 0; --c) {
        const long long c0 = k0 + c * UL_C;
        if (c0 >= L) continue;
        if (diag && c < w) break;
        const int n = (int)min((long long)UL_C, L - c0);
        if (diag && c == w) {  // own chunk: exact fp64, tail R in the tile frame
          double Rt = Rt64 * pow2d(2 * gprev);
          const double cA = (gt == 0.f) ? 0.0 : (double)gt / A;
          for (int k = n - 1; k >= 0; --k) {
            float pv = 0.f, qv = 0.f;
            if (k >= lane && cA != 0.0) {
              double sk = 0.0;
              for (int j = lane; j <= k; ++j) sk += S.ex[c * UL_C + j];
              const double D = sk + S.E[c * UL_C + k];
              const double qd = ur_rcp(D);
              const double w2 = qd * qd;
              Rt += w2;
              pv = (float)(cA * S.E[c * UL_C + k] * w2);
              qv = (float)(cA * S.ex[c * UL_C + k] * Rt);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              pv += __shfl_xor_sync(0xffffffffu, pv, o);
              qv += __shfl_xor_sync(0xffffffffu, qv, o);
            }
            if (lane == 0) {  // this warp's slot of the column (summed in warp order below)
              colP[w * UL_T + c * UL_C + k] += pv;
              colQ[w * UL_T + c * UL_C + k] += qv;
            }
          }
          continue;
        }
        double bc;
        if (diag) {
          bc = sown;
          for (int cc = w + 1; cc < c; ++cc) bc += S.qtot[cc];
        } else {
          bc = head + CQ[4 * s + c];
        }
        ul_chunk_bwd(S, c, n, bc, A, gt, dtail, Rt64, gprev, colP, colQ, dsm + w * (32 * 36));
      }
      __syncthreads();
      const long long k = k0 + tid;
      if (k < L) {
        float sp = 0.f, sq = 0.f;
#pragma unroll
        for (int ww = 0; ww < UL_T / 32; ++ww) {
          sp += colP[ww * UL_T + tid];
          sq += colQ[ww * UL_T + tid];
        }
        gr_row.add(k, sp);
        gl_row.add(k, sq);
      }
    }
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
// shared-memory backward: staging + checkpoints every U_CB_S steps + block buffer
static size_t bwd_smem(const UParams& p) {
  long long span = p.untimed ? p.L : (long long)U_THREADS + p.b;
  if (span > p.L && !p.fill) span = p.L;
  long long kmax = p.untimed ? p.L : p.K;
  long long nck = (kmax + U_CB_S - 1) / U_CB_S;
  return (size_t)2 * span * 4 + (size_t)nck * 3 * U_THREADS * 4 + (size_t)U_CB_S * 2 * U_THREADS * 4;
}
// the shared variant keeps >= 3 CTAs per SM; beyond that, the persistent global-slab one
static bool bwd_uses_smem(const UParams& p) { return !p.untimed && bwd_smem(p) <= 72 * 1024; }

static int until_sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// timed LSE Until in reciprocal form: windows long enough that one rcp per pair beats the
// incremental per-pair ex2 / lg2 (forward: the staged chunk kernel; backward: one thread
// per output, k_until_rcp_lse_bwd_timed — the staged chunk form of the backward measured
// 40.1 ms at C5 U[0,100] against 18.3 ms for the per-output one)
static bool ul_timed(const UParams& p) { return !p.untimed && !p.fill && p.K >= 16 && p.L < (1LL << 30); }

size_t until_bwd_scratch_bytes(int mode, int untimed, int fill, long long L, int b, int K) {
  UParams p;
  memset(&p, 0, sizeof(p));
  p.L = L;
  p.b = b;
  p.K = K;
  p.untimed = untimed;
  p.fill = fill;
  if (mode == M_HARD) return 0;  // one source per output: no checkpoints
  // the reciprocal-form timed LSE backward falls back per tile to the per-pair tile
  // function with its checkpoints in the global slab
  if (bwd_uses_smem(p) && !(mode == M_LSE && ul_timed(p))) return 0;
  const long long stride = (long long)until_sm_count() * U_PERSIST_PER_SM * U_THREADS;
  const long long nck = (untimed ? L : K) / U_CB_G + 1;
  return (size_t)(nck * 3) * stride * 4;
}

// ---------------------------------------------------------------------------
// reproducible accumulation (detacc.cuh)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_det_row_scale(const float* __restrict__ cot, long long L, int span,
                                                       int* __restrict__ S) {
  __shared__ float red[8];
  const long long row = blockIdx.x;
  float m = 0.f;
  for (long long t = threadIdx.x; t < L; t += 256) m = fmaxf(m, fabsf(cot[row * L + t]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
    S[row] = (m > 0.f && m < INFINITY) ? (span < 0 ? 28 : 61 - span) - ilogbf(m) : 0;
  }
}

__global__ void k_det_finish(const unsigned long long* __restrict__ hi, const unsigned long long* __restrict__ lo,
                             const int* __restrict__ S, long long B, long long L, float* __restrict__ out) {
  const long long n = B * L;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int s = S[i / L];
    const double h = (double)(long long)hi[i] * ldexp(1.0, -s);
    out[i] = (float)(lo != nullptr ? h + (double)(long long)lo[i] * ldexp(1.0, -s - 40) : h);
  }
}

// softmax: two-word grid (weights outside [0, 1]); hard / LSE: one word, sized for the
// largest number of outputs that reach one element (b + 1 timed, L untimed / masked_fill)
static int det_span(int mode, const UParams& p) {
  if (mode == M_SOFT) return -1;
  const long long w = (p.untimed || p.fill) ? p.L + 1 : (long long)p.b + 2;
  int bits = 0;
  while ((1LL << bits) < w) ++bits;
  return bits + 1;
}

static cudaError_t det_begin(int mode, const UParams& p, cudaStream_t st) {
  const size_t n = (size_t)(p.B * p.L);
  cudaError_t e = cudaMemsetAsync(p.dacc, 0, sizeof(unsigned long long) * n, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.dacc + 2 * n, 0, sizeof(unsigned long long) * n, st);
  if (e == cudaSuccess && mode == M_SOFT) {
    e = cudaMemsetAsync(p.dacc + n, 0, sizeof(unsigned long long) * n, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.dacc + 3 * n, 0, sizeof(unsigned long long) * n, st);
  }
  if (e != cudaSuccess) return e;
  k_det_row_scale<<<(unsigned)p.B, 256, 0, st>>>(p.cot, p.L, det_span(mode, p), p.dscale);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t det_end(int mode, const UParams& p, cudaStream_t st) {
  const long long n = p.B * p.L;
  const unsigned grid = (unsigned)min((n + 255) / 256, 148LL * 16);
  const bool two = mode == M_SOFT;
  k_det_finish<<<grid, 256, 0, st>>>(p.dacc, two ? p.dacc + n : nullptr, p.dscale, p.B, p.L, p.gl);
  count_launch();
  k_det_finish<<<grid, 256, 0, st>>>(p.dacc + 2 * n, two ? p.dacc + 3 * n : nullptr, p.dscale, p.B, p.L, p.gr);
  count_launch();
  return cudaGetLastError();
}

// untimed hard Until: the look-back shape when the rows alone leave the GPU short of CTAs
static bool uh_use_lb(const UParams& p) { return p.lb != nullptr && p.B < 2 * 148 && p.L >= 4 * LB_MIN_TILE; }

template <int MODE>
static cudaError_t until_fwd_mode(UParams& p, cudaStream_t st) {
  if (MODE == M_HARD && until_ht_applicable(p)) return launch_until_ht_fwd(p, st);  // O(T), until_ht.cu
  if (p.untimed && MODE == M_HARD && !p.fill) {
    if (p.L >= (1LL << 31)) return cudaErrorNotSupported;  // 32-bit time indices
    if (uh_use_lb(p)) {
      const long long nch = (p.L + LB_MIN_TILE - 1) / LB_MIN_TILE;  // (+ the ticket slot)
      cudaError_t e = cudaMemsetAsync(p.lb, 0, sizeof(unsigned) * LB_WORDS * (size_t)(p.B * nch + 1), st);
      if (e != cudaSuccess) return e;
      k_until_unt_hard_fwd<MODE, true><<<(unsigned)(nch * p.B), UH_LB, 0, st>>>(p);
    } else {
      k_until_unt_hard_fwd<MODE, false><<<(unsigned)p.B, UH_SEQ, 0, st>>>(p);
    }
    count_launch();
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((p.L + U_THREADS - 1) / U_THREADS), (unsigned)p.B);
  if (MODE == M_LSE && !p.fill && (p.untimed || ul_timed(p))) {
    if (p.untimed) k_until_rcp_lse_fwd<false><<<grid, UL_T, 0, st>>>(p);
    else k_until_rcp_lse_fwd<true><<<grid, UL_T, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  size_t smem = fwd_smem(p);
  if (smem <= 64 * 1024) {
    cudaError_t e = set_smem_u(k_until_fwd<MODE>, smem);
    if (e != cudaSuccess) return e;
    k_until_fwd<MODE><<<grid, U_THREADS, smem, st>>>(p);
  } else {  // long untimed windows: direct reads
    k_until_fwd_g<MODE><<<grid, U_THREADS, 0, st>>>(p);
  }
  count_launch();
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t until_bwd_mode(UParams& p, cudaStream_t st) {
  if (p.untimed && MODE == M_HARD && !p.fill) {
    if (p.L >= (1LL << 31)) return cudaErrorNotSupported;  // 32-bit time indices
    if (uh_use_lb(p)) {
      const long long nch = (p.L + LB_MIN_TILE - 1) / LB_MIN_TILE;  // (+ the ticket slot)
      cudaError_t e = cudaMemsetAsync(p.lb, 0, sizeof(unsigned) * LB_WORDS * (size_t)(p.B * nch + 1), st);
      if (e != cudaSuccess) return e;
      k_until_unt_hard_bwd<MODE, true><<<(unsigned)(nch * p.B), UH_LB, 0, st>>>(p);
    } else {
      k_until_unt_hard_bwd<MODE, false><<<(unsigned)p.B, UH_SEQ, 0, st>>>(p);
    }
    count_launch();
    return cudaGetLastError();
  }
  cudaError_t e;
  if (MODE == M_HARD && until_ht_applicable(p)) {  // O(T), deterministic (until_ht.cu)
    if (p.src_in != nullptr) return launch_until_ht_bwd(p, st);  // stored sources, fused child VJPs
    if ((e = launch_until_ht_bwd(p, st)) != cudaSuccess) return e;
  } else {
  if (p.dacc == nullptr || p.dscale == nullptr) return cudaErrorInvalidValue;
  if ((e = det_begin(MODE, p, st)) != cudaSuccess) return e;
  const int ntx = (int)((p.L + U_THREADS - 1) / U_THREADS);
  const size_t ul_smem = (size_t)U_CB_G * 2 * U_THREADS * 4 + (size_t)(ntx * 4 + 4) * sizeof(double);
  const size_t ur_sm = ur_smem(p);
  if (MODE == M_LSE && ul_timed(p) && p.scratch != nullptr && ur_sm <= 100 * 1024) {
    if ((e = set_smem_u(k_until_rcp_lse_bwd_timed, ur_sm)) != cudaSuccess) return e;
    const long long ntiles = (long long)ntx * p.B;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_until_rcp_lse_bwd_timed, U_THREADS, ur_sm) !=
            cudaSuccess || occ <= 0)
      occ = 1;
    long long grid = (long long)until_sm_count() * min(occ, U_PERSIST_PER_SM);
    if (grid > ntiles) grid = ntiles;
    k_until_rcp_lse_bwd_timed<<<(unsigned)grid, U_THREADS, ur_sm, st>>>(p, ntx, ntiles);
  } else if (MODE == M_LSE && p.untimed && !p.fill && p.scratch != nullptr && ul_smem <= kUSmemMax) {
    if ((e = set_smem_u(k_until_unt_lse_bwd, ul_smem)) != cudaSuccess) return e;
    const long long ntiles = (long long)ntx * p.B;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_until_unt_lse_bwd, UL_T, ul_smem) != cudaSuccess ||
        occ <= 0)
      occ = 1;
    long long grid = (long long)until_sm_count() * min(occ, U_PERSIST_PER_SM);
    if (grid > ntiles) grid = ntiles;
    k_until_unt_lse_bwd<<<(unsigned)grid, UL_T, ul_smem, st>>>(p, ntx, ntiles);
  } else if (bwd_uses_smem(p) || MODE == M_HARD) {
    size_t smem = (MODE == M_HARD) ? fwd_smem(p) : bwd_smem(p);
    if (smem <= kUSmemMax) {
      if ((e = set_smem_u(k_until_bwd<MODE>, smem)) != cudaSuccess) return e;
      dim3 grid((unsigned)ntx, (unsigned)p.B);
      k_until_bwd<MODE><<<grid, U_THREADS, smem, st>>>(p);
    } else if (MODE == M_HARD) {
      // hard (masked_fill, long untimed): one source per output, no checkpoints
      const long long ntiles = (long long)ntx * p.B;
      long long grid = (long long)until_sm_count() * 8;
      if (grid > ntiles) grid = ntiles;
      k_until_bwd_g<MODE><<<(unsigned)grid, U_THREADS, 0, st>>>(p, ntx, ntiles);
    } else {
      return cudaErrorNotSupported;
    }
  } else {
    if (p.scratch == nullptr) return cudaErrorNotSupported;
    const long long ntiles = (long long)ntx * p.B;
    long long grid = (long long)until_sm_count() * U_PERSIST_PER_SM;
    if (grid > ntiles) grid = ntiles;
    const size_t bsm = (size_t)U_CB_G * 2 * U_THREADS * 4;
    k_until_bwd_g<MODE><<<(unsigned)grid, U_THREADS, bsm, st>>>(p, ntx, ntiles);
  }
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = det_end(MODE, p, st)) != cudaSuccess) return e;
  }
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
