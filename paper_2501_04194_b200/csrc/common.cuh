// common.cuh — device-side building blocks shared by every stlg kernel.
//
//  * DExpr: a fused elementwise sub-formula (Pred / NormPred / Not / And / Or /
//    TRUE / reads of materialised temporal traces) evaluated at one (row, t)
//    inside the consumer's load — the "formula-tree executor" of the north
//    star.  Negations are pushed to the leaves at compile time (exact: the
//    reference computes min as -max(-x), masking.py:164-167, tape.py:390-391),
//    so an expression is a DAG of max/min steps over signed affine leaves.
//  * pair reductions (And / Or) with the reference's tie rule (ties go to the
//    left operand, tape.py:347) and their VJPs.
//  * monoid states for the windowed reductions (hard arg-max, log-sum-exp,
//    softmax) and fast exp2/log2 (MUFU) helpers.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace stlg {

constexpr int MAX_LEAF = 16;
constexpr int MAX_STEP = 31;
constexpr int MAX_SRC = 16;

enum LeafKind { LEAF_AFFINE = 0, LEAF_CONST = 1, LEAF_NORM = 2, LEAF_SRC = 3 };
enum StepOp { ST_LEAF = 0, ST_MAX = 1, ST_MIN = 2 };
enum Mode { M_HARD = 0, M_SOFT = 1, M_LSE = 2 };

struct DSrc {
  const float* p;
  long long rs, es;
};
struct DDst {
  float* p;
  long long rs, es;
};

// value = s_out * (s_in * x + c)   (LEAF_AFFINE: Pred on a channel, masking.py:319-323)
// value = s_out * (s_in * d + c)   (LEAF_NORM:   d = ||(x,y) - (cx,cy)||)
// value = s_out * x                (LEAF_SRC:    a materialised trace, no rounding step)
// value = c                        (LEAF_CONST:  +/- top_value, masking.py:316-318)
struct DLeaf {
  int kind, src, src2;
  int st1, st2;  // gradient write of src / src2: 1 = store (first writer), 0 = accumulate
  int pad_;
  float s_in, s_out, c, cx, cy, pad2_;
};
struct DStep {
  unsigned char op, a, b, pad_;
};
struct DExpr {
  int n_step, n_leaf, n_src, pad_;
  DLeaf leaf[MAX_LEAF];
  DStep step[MAX_STEP];
  DSrc src[MAX_SRC];
  DDst dst[MAX_SRC];  // gradient destinations, parallel to src (backward only)
};

struct ModeP {
  float tau;       // temperature
  float tau2;      // tau * log2(e): e^{tau x} = 2^{tau2 x}
  float inv_tau2;  // 1 / tau2: ln(s) / tau = log2(s) / tau2
};

// ---------------------------------------------------------------------------
// MUFU helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------------------
// expression evaluation
// ---------------------------------------------------------------------------
// streaming loads that do not allocate in L1: the pipelined kernels give most of
// the unified L1 to shared memory, and L1-allocating loads then cap the bytes in flight
__device__ __forceinline__ float ld_na(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
// Low word of the double-float LSE trace (M = hi + lo, |lo| <= ulp(hi) / 2), kept as a
// bf16 plane in the first half of the row's aux words: 2 B per sample instead of 4 in the
// forward's write and the backward's read.  Rounding lo to 8 bits moves M by at most
// 2^-9 |lo| <= 2^-10 ulp(hi), far below the fp32 rounding the low word corrects.
__device__ __forceinline__ unsigned short lo_pack(float v) {  // round to nearest even, one F2F
  unsigned short h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(v));
  return h;
}
__device__ __forceinline__ float lo_ld(const unsigned short* p) {
  unsigned short h;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(h) : "l"(p));
  return __uint_as_float((unsigned)h << 16);
}
__device__ __forceinline__ float2 ld_na2(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ float ld_src(const DSrc& s, long long b, long long j) {
  return __ldg(s.p + b * s.rs + j * s.es);
}

__device__ __forceinline__ float leaf_val(const DExpr& e, const DLeaf& L, long long b,
                                          long long j) {
  if (L.kind == LEAF_CONST) return L.c;
  if (L.kind == LEAF_SRC) return L.s_out * ld_src(e.src[L.src], b, j);
  float x;
  if (L.kind == LEAF_AFFINE) {
    x = ld_src(e.src[L.src], b, j);
  } else {
    float dx = ld_src(e.src[L.src], b, j) - L.cx;
    float dy = ld_src(e.src[L.src2], b, j) - L.cy;
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(fmaf(dx, dx, dy * dy)));
    x = y;
  }
  // one rounding, exactly as x + (-c) / (-x) + c in the reference
  float t = __fadd_rn(L.s_in * x, L.c);
  return L.s_out * t;
}

__device__ __forceinline__ void acc_dst(const DDst& d, long long b, long long j, float g, int st) {
  if (d.p != nullptr) {
    float* q = d.p + b * d.rs + j * d.es;
    if (st) *q = g;
    else *q += g;
  }
}

__device__ __forceinline__ void leaf_vjp(const DExpr& e, const DLeaf& L, long long b, long long j,
                                         float g) {
  if (L.kind == LEAF_CONST) return;
  if (L.kind == LEAF_SRC) {
    acc_dst(e.dst[L.src], b, j, g * L.s_out, L.st1);
    return;
  }
  float gx = g * L.s_out * L.s_in;
  if (L.kind == LEAF_AFFINE) {
    acc_dst(e.dst[L.src], b, j, gx, L.st1);
    return;
  }
  float dx = ld_src(e.src[L.src], b, j) - L.cx;
  float dy = ld_src(e.src[L.src2], b, j) - L.cy;
  float d = sqrtf(fmaf(dx, dx, dy * dy));
  float inv = d > 0.f ? 1.f / d : 0.f;
  acc_dst(e.dst[L.src], b, j, gx * dx * inv, L.st1);
  acc_dst(e.dst[L.src2], b, j, gx * dy * inv, L.st2);
}

// Two-element reduction (And / Or), masking.py:326-330 -> tape.smooth_max/min.
// sg = +1 for max (Or), -1 for min (And): min(l, r) = -max(-l, -r).
// p1 / p2 receive d out / d l and d out / d r.
template <int MODE>
__device__ __forceinline__ float pair_red(float l, float r, float sg, const ModeP& mp, float& p1,
                                          float& p2) {
  float u1 = sg * l, u2 = sg * r;
  bool first = u1 >= u2;  // first arg-max: ties to the left operand
  float m = first ? u1 : u2;
  if (MODE == M_HARD) {
    p1 = first ? 1.f : 0.f;
    p2 = first ? 0.f : 1.f;
    return sg * m;
  }
  float e1 = ex2f(mp.tau2 * (u1 - m));
  float e2 = ex2f(mp.tau2 * (u2 - m));
  float s = e1 + e2;
  float inv = __frcp_rn(s);  // s in [1, 2]: the correctly rounded reciprocal, = 1.f / s
  if (MODE == M_LSE) {
    p1 = e1 * inv;
    p2 = e2 * inv;
    return sg * fmaf(lg2f(s), mp.inv_tau2, m);
  }
  float M = (u1 * e1 + u2 * e2) * inv;
  p1 = e1 * inv * fmaf(mp.tau, u1 - M, 1.f);
  p2 = e2 * inv * fmaf(mp.tau, u2 - M, 1.f);
  return sg * M;
}

template <int MODE>
__device__ __forceinline__ float expr_eval(const DExpr& e, long long b, long long j,
                                           const ModeP& mp) {
  if (e.n_step == 1) return leaf_val(e, e.leaf[0], b, j);
  float v[MAX_STEP];
#pragma unroll 1
  for (int k = 0; k < e.n_step; ++k) {
    DStep s = e.step[k];
    if (s.op == ST_LEAF) {
      v[k] = leaf_val(e, e.leaf[s.a], b, j);
    } else {
      float p1, p2;
      v[k] = pair_red<MODE>(v[s.a], v[s.b], s.op == ST_MAX ? 1.f : -1.f, mp, p1, p2);
    }
  }
  return v[e.n_step - 1];
}

// Route cotangent g of the expression value at (b, j) into the gradient
// destinations (reverse walk of the SSA steps).
template <int MODE>
__device__ __forceinline__ void expr_vjp(const DExpr& e, long long b, long long j, float g,
                                         const ModeP& mp) {
  if (e.n_step == 1) {
    leaf_vjp(e, e.leaf[0], b, j, g);
    return;
  }
  float v[MAX_STEP], w1[MAX_STEP], w2[MAX_STEP], adj[MAX_STEP];
#pragma unroll 1
  for (int k = 0; k < e.n_step; ++k) {
    DStep s = e.step[k];
    adj[k] = 0.f;
    if (s.op == ST_LEAF) {
      v[k] = leaf_val(e, e.leaf[s.a], b, j);
    } else {
      v[k] = pair_red<MODE>(v[s.a], v[s.b], s.op == ST_MAX ? 1.f : -1.f, mp, w1[k], w2[k]);
    }
  }
  adj[e.n_step - 1] = g;
#pragma unroll 1
  for (int k = e.n_step - 1; k >= 0; --k) {
    DStep s = e.step[k];
    float a = adj[k];
    if (s.op == ST_LEAF) {
      const DLeaf& L = e.leaf[s.a];
      if (a != 0.f || L.st1 || L.st2) leaf_vjp(e, L, b, j, a);
    } else {
      adj[s.a] += a * w1[k];
      adj[s.b] += a * w2[k];
    }
  }
}

// A child expression evaluated with its leaf fields in registers: single-leaf affine /
// trace children (the common Until operands) skip the generic walk's per-sample reads of
// the expression descriptor; anything else falls back to expr_eval.  Same values, bit for
// bit (leaf_val's formulas).
struct ChildEval {
  const DExpr* e;
  long long row;
  const float* p;
  long long es;
  float* gp;       // gradient destination row (or null)
  long long ges;
  int gst;         // 1: store (first writer), 0: accumulate
  float s_in, c, s_out;
  int kind;  // 0 generic, 1 trace (LEAF_SRC), 2 affine (LEAF_AFFINE)
  __device__ __forceinline__ ChildEval(const DExpr& ex, long long r) : e(&ex), row(r) {
    kind = 0;
    p = nullptr;
    gp = nullptr;
    es = ges = 0;
    gst = 0;
    s_in = c = s_out = 0.f;
    if (ex.n_step == 1) {
      const DLeaf& L = ex.leaf[0];
      if (L.kind == LEAF_SRC || L.kind == LEAF_AFFINE) {
        const DSrc& sr = ex.src[L.src];
        p = sr.p + r * sr.rs;
        es = sr.es;
        const DDst& d = ex.dst[L.src];
        if (d.p) {
          gp = d.p + r * d.rs;
          ges = d.es;
        }
        gst = L.st1;
        s_in = L.s_in;
        c = L.c;
        s_out = L.s_out;
        kind = L.kind == LEAF_SRC ? 1 : 2;
      }
    }
  }
  // the child's VJP at j for cotangent g (leaf_vjp / expr_vjp, same arithmetic)
  template <int MODE>
  __device__ __forceinline__ void grad(long long j, float g, const ModeP& mp) const {
    if (kind == 0) {
      expr_vjp<MODE>(*e, row, j, g, mp);
      return;
    }
    if (gp == nullptr) return;
    const float v = kind == 1 ? g * s_out : g * s_out * s_in;
    float* q = gp + j * ges;
    if (gst) *q = v;
    else *q += v;
  }
  template <int MODE>
  __device__ __forceinline__ float value(long long j, const ModeP& mp) const {
    if (kind == 1) return s_out * __ldg(p + j * es);
    if (kind == 2) return s_out * __fadd_rn(s_in * __ldg(p + j * es), c);
    return expr_eval<MODE>(*e, row, j, mp);
  }
  // fast kinds only (kind != 0): the load and the leaf transform apart, so a caller can
  // issue a batch of loads before the first use
  __device__ __forceinline__ float raw(long long j) const { return __ldg(p + j * es); }
  // 32-bit index forms (rows shorter than 2^31 samples, strides below 2^31): one 32-bit
  // multiply and a widening add per access instead of 64-bit arithmetic
  __device__ __forceinline__ float raw(int j) const { return __ldg(p + j * (int)es); }
  template <int MODE>
  __device__ __forceinline__ void grad(int j, float g, const ModeP& mp) const {
    if (kind == 0) {
      expr_vjp<MODE>(*e, row, j, g, mp);
      return;
    }
    if (gp == nullptr) return;
    const float v = kind == 1 ? g * s_out : g * s_out * s_in;
    float* q = gp + j * (int)ges;
    if (gst) *q = v;
    else *q += v;
  }
  __device__ __forceinline__ float apply(float x) const {
    return kind == 1 ? s_out * x : s_out * __fadd_rn(s_in * x, c);
  }
};

// Register-resident forms for expressions of exactly N steps (N small): the step loop is
// unrolled, so the SSA values live in registers and operands are picked by selects
// instead of dynamically indexed (local-memory) arrays.
template <int N>
__device__ __forceinline__ float pick_n(const float (&v)[N], int idx, int k) {
  float r = v[0];
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (i < k) r = (idx == i) ? v[i] : r;
  return r;
}

template <int MODE, int N>
__device__ __forceinline__ float expr_eval_n(const DExpr& e, long long b, long long j, const ModeP& mp) {
  float v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const DStep s = e.step[k];
    if (s.op == ST_LEAF) {
      v[k] = leaf_val(e, e.leaf[s.a], b, j);
    } else {
      float p1, p2;
      v[k] = pair_red<MODE>(pick_n<N>(v, s.a, k), pick_n<N>(v, s.b, k), s.op == ST_MAX ? 1.f : -1.f, mp, p1, p2);
    }
  }
  return v[N - 1];
}

template <int MODE, int N>
__device__ __forceinline__ void expr_vjp_n(const DExpr& e, long long b, long long j, float g, const ModeP& mp) {
  float v[N], w1[N], w2[N], adj[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const DStep s = e.step[k];
    adj[k] = 0.f;
    w1[k] = w2[k] = 0.f;
    if (s.op == ST_LEAF) {
      v[k] = leaf_val(e, e.leaf[s.a], b, j);
    } else {
      v[k] = pair_red<MODE>(pick_n<N>(v, s.a, k), pick_n<N>(v, s.b, k), s.op == ST_MAX ? 1.f : -1.f, mp,
                            w1[k], w2[k]);
    }
  }
  adj[N - 1] = g;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) {
    const DStep s = e.step[k];
    const float a = adj[k];
    if (s.op == ST_LEAF) {
      const DLeaf& L = e.leaf[s.a];
      if (a != 0.f || L.st1 || L.st2) leaf_vjp(e, L, b, j, a);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {  // scatter by selects (i < k: operands precede the step)
        if (i < k) {
          adj[i] += (s.a == i) ? a * w1[k] : 0.f;
          adj[i] += (s.b == i) ? a * w2[k] : 0.f;
        }
      }
    }
  }
}

// Row-hoisted N-step expressions for the pointwise kernels: every leaf step's source /
// gradient row base and its transform are resolved once per row (expressions whose
// leaves are constants, traces or affine predicates over unit-stride planes — the host
// checks, pw_unit), so a sample costs one load per leaf instead of the descriptor walk and
// 64-bit address arithmetic of leaf_val (the transforms stay in the parameter bank).
template <int N>
struct RowLeaves {
  const float* src[N];  // leaf steps: row base of the source (null: constant / not a leaf)
  float* dst[N];        // leaf steps: row base of the gradient destination (or null)
  __device__ __forceinline__ RowLeaves(const DExpr& e, long long row, bool want_dst) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      src[k] = nullptr;
      dst[k] = nullptr;
      const DStep sp = e.step[k];
      if (sp.op != ST_LEAF) continue;
      const DLeaf& L = e.leaf[sp.a];
      if (L.kind == LEAF_CONST) continue;
      src[k] = e.src[L.src].p + row * e.src[L.src].rs;
      if (want_dst && e.dst[L.src].p) dst[k] = e.dst[L.src].p + row * e.dst[L.src].rs;
    }
  }
  __device__ __forceinline__ float value(const DLeaf& L, int k, int j) const {
    if (L.kind == LEAF_CONST) return L.c;
    const float x = __ldg(src[k] + j);
    return L.kind == LEAF_SRC ? L.s_out * x : L.s_out * __fadd_rn(L.s_in * x, L.c);
  }
  __device__ __forceinline__ void grad(const DLeaf& L, int k, int j, float g) const {
    if (dst[k] == nullptr) return;
    const float v = L.kind == LEAF_SRC ? g * L.s_out : g * L.s_out * L.s_in;
    if (L.st1) dst[k][j] = v;
    else dst[k][j] += v;
  }
};

template <int MODE, int N>
__device__ __forceinline__ float expr_eval_rn(const DExpr& e, const RowLeaves<N>& R, int j, const ModeP& mp) {
  float v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const DStep s = e.step[k];
    if (s.op == ST_LEAF) {
      v[k] = R.value(e.leaf[s.a], k, j);
    } else {
      float p1, p2;
      v[k] = pair_red<MODE>(pick_n<N>(v, s.a, k), pick_n<N>(v, s.b, k), s.op == ST_MAX ? 1.f : -1.f, mp, p1, p2);
    }
  }
  return v[N - 1];
}

template <int MODE, int N>
__device__ __forceinline__ void expr_vjp_rn(const DExpr& e, const RowLeaves<N>& R, int j, float g, const ModeP& mp) {
  float v[N], w1[N], w2[N], adj[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const DStep s = e.step[k];
    adj[k] = 0.f;
    w1[k] = w2[k] = 0.f;
    if (s.op == ST_LEAF) {
      v[k] = R.value(e.leaf[s.a], k, j);
    } else {
      v[k] = pair_red<MODE>(pick_n<N>(v, s.a, k), pick_n<N>(v, s.b, k), s.op == ST_MAX ? 1.f : -1.f, mp,
                            w1[k], w2[k]);
    }
  }
  adj[N - 1] = g;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) {
    const DStep s = e.step[k];
    const float a = adj[k];
    if (s.op == ST_LEAF) {
      const DLeaf& L = e.leaf[s.a];
      if (a != 0.f || L.st1) R.grad(L, k, j, a);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (i < k) {
          adj[i] += (s.a == i) ? a * w1[k] : 0.f;
          adj[i] += (s.b == i) ? a * w2[k] : 0.f;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// monoid states for window reductions (all in "max space": u = sg * v)
// ---------------------------------------------------------------------------

// Hard: value + index; on ties the EARLIER index wins (tape.py:346-348 np.argmax).
struct HardAcc {
  float v;
  int i;
};
// e covers earlier positions than l
__device__ __forceinline__ HardAcc hard_comb(HardAcc e, HardAcc l) { return (l.v > e.v) ? l : e; }

// LSE: s = sum exp(tau (u - m)), m = running hard max (tape.py:366 detached shift).
struct LseAcc {
  float m, s;
};
__device__ __forceinline__ LseAcc lse_comb(LseAcc x, LseAcc y, float tau2) {
  if (y.s == 0.f) return x;
  if (x.s == 0.f) return y;
  if (x.m >= y.m) return {x.m, fmaf(y.s, ex2f(tau2 * (y.m - x.m)), x.s)};
  return {y.m, fmaf(x.s, ex2f(tau2 * (x.m - y.m)), y.s)};
}
__device__ __forceinline__ LseAcc lse_push(LseAcc a, float u, float tau2) {
  if (a.s == 0.f) return {u, 1.f};
  if (u > a.m) return {u, fmaf(a.s, ex2f(tau2 * (a.m - u)), 1.f)};
  return {a.m, a.s + ex2f(tau2 * (u - a.m))};
}

// Softmax: s as LSE, d = sum (u - m) exp(tau (u - m)); value = m + d / s.
struct SoftAcc {
  float m, s, d;
};
__device__ __forceinline__ SoftAcc soft_comb(SoftAcc x, SoftAcc y, float tau2) {
  if (y.s == 0.f) return x;
  if (x.s == 0.f) return y;
  if (x.m < y.m) {
    SoftAcc t = x;
    x = y;
    y = t;
  }
  float dm = y.m - x.m;  // <= 0
  float f = ex2f(tau2 * dm);
  return {x.m, fmaf(f, y.s, x.s), fmaf(f, fmaf(dm, y.s, y.d), x.d)};
}
__device__ __forceinline__ SoftAcc soft_push(SoftAcc a, float u, float tau2) {
  if (a.s == 0.f) return {u, 1.f, 0.f};
  if (u > a.m) {
    float dm = a.m - u;
    float f = ex2f(tau2 * dm);
    return {u, fmaf(a.s, f, 1.f), f * fmaf(dm, a.s, a.d)};
  }
  float du = u - a.m;
  float e = ex2f(tau2 * du);
  return {a.m, a.s + e, fmaf(du, e, a.d)};
}

// Backward window sums over outputs t (gather form):
//   LSE:  g_child[j] = sum_t g_t exp(tau (u_j - M_t))           (tape.py:360-380 VJP)
//   Soft: g_child[j] = sum_t g_t exp(tau (u_j - L_t)) (1 + tau (u_j - M_t))
// State (mu, A[, Bc]): sum_t a_t exp(-tau (mu_t - mu)) [ (M_t - c) ], mu = min mu_t.
struct GLse {
  float mu, A;
};
__device__ __forceinline__ GLse glse_comb(GLse x, GLse y, float tau2) {
  if (y.A == 0.f) return x;
  if (x.A == 0.f) return y;
  if (x.mu <= y.mu) return {x.mu, fmaf(y.A, ex2f(tau2 * (x.mu - y.mu)), x.A)};
  return {y.mu, fmaf(x.A, ex2f(tau2 * (y.mu - x.mu)), y.A)};
}
struct GSoft {
  float mu, A, Bc, c;  // Bc = sum a_t w_t (M_t - c); c re-centres to the dominant term
};
__device__ __forceinline__ GSoft gsoft_comb(GSoft x, GSoft y, float tau2) {
  if (y.A == 0.f && y.Bc == 0.f) return x;
  if (x.A == 0.f && x.Bc == 0.f) return y;
  if (x.mu > y.mu) {
    GSoft t = x;
    x = y;
    y = t;
  }
  float f = ex2f(tau2 * (x.mu - y.mu));
  return {x.mu, fmaf(y.A, f, x.A), fmaf(f, fmaf(y.c - x.c, y.A, y.Bc), x.Bc), x.c};
}


// ---------------------------------------------------------------------------
// branch-free single-MUFU monoid updates (used by the v2 window kernels)
// ---------------------------------------------------------------------------
// LSE state (m, s): s = sum exp(tau (u - m)); push one sample u.
__device__ __forceinline__ void lse_add(float& m, float& s, float u, float tau2) {
  float d = u - m;
  float e = ex2f(-tau2 * fabsf(d));
  bool up = d > 0.f;
  s = up ? fmaf(s, e, 1.f) : s + e;
  m = up ? u : m;
}
// merge (m2, s2) into (m, s)
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2, float tau2) {
  float d = m2 - m;
  float e = ex2f(-tau2 * fabsf(d));
  bool up = d > 0.f;
  s = up ? fmaf(s, e, s2) : fmaf(s2, e, s);
  m = up ? m2 : m;
}
// softmax state (m, s, q): q = sum (u - m) exp(tau (u - m)); value m + q / s
__device__ __forceinline__ void soft_add(float& m, float& s, float& q, float u, float tau2) {
  float d = u - m;
  float e = ex2f(-tau2 * fabsf(d));
  bool up = d > 0.f;
  float s_up = fmaf(s, e, 1.f), q_up = e * fmaf(-d, s, q);
  float s_dn = s + e, q_dn = fmaf(d, e, q);
  s = up ? s_up : s_dn;
  q = up ? q_up : q_dn;
  m = up ? u : m;
}
__device__ __forceinline__ void soft_merge(float& m, float& s, float& q, float m2, float s2, float q2,
                                           float tau2) {
  float d = m2 - m;
  float e = ex2f(-tau2 * fabsf(d));
  bool up = d > 0.f;
  float s_up = fmaf(s, e, s2), q_up = fmaf(e, fmaf(-d, s, q), q2);
  float s_dn = fmaf(s2, e, s), q_dn = fmaf(e, fmaf(d, s2, q2), q);
  s = up ? s_up : s_dn;
  q = up ? q_up : q_dn;
  m = up ? m2 : m;
}
// backward window sums (gather form), state (mu, A): sum_t A_t exp(-tau (mu_t - mu)), mu = min
__device__ __forceinline__ void gl_add(float& mu, float& A, float mu2, float A2, float tau2) {
  float d = mu2 - mu;
  float e = ex2f(-tau2 * fabsf(d));
  bool dn = d < 0.f;
  float A_new = dn ? fmaf(A, e, A2) : fmaf(A2, e, A);
  float mu_new = dn ? mu2 : mu;
  bool skip = A2 == 0.f, empty = A == 0.f;
  A = skip ? A : (empty ? A2 : A_new);
  mu = skip ? mu : (empty ? mu2 : mu_new);
}
// softmax backward state (mu, A, Bc, c): Bc = sum A_t w_t (M_t - c), re-centred on the min-mu term
__device__ __forceinline__ void gs_add(float& mu, float& A, float& Bc, float& c, float mu2, float A2,
                                       float B2, float c2, float tau2) {
  bool skip = (A2 == 0.f && B2 == 0.f), empty = (A == 0.f && Bc == 0.f);
  float d = mu2 - mu;
  float e = ex2f(-tau2 * fabsf(d));
  bool dn = d < 0.f;
  // dn: the new term dominates (reference c2); else keep c
  float A_dn = fmaf(A, e, A2), B_dn = fmaf(e, fmaf(c - c2, A, Bc), B2);
  float A_up = fmaf(A2, e, A), B_up = fmaf(e, fmaf(c2 - c, A2, B2), Bc);
  float nA = dn ? A_dn : A_up, nB = dn ? B_dn : B_up, nmu = dn ? mu2 : mu, nc = dn ? c2 : c;
  A = skip ? A : (empty ? A2 : nA);
  Bc = skip ? Bc : (empty ? B2 : nB);
  mu = skip ? mu : (empty ? mu2 : nmu);
  c = skip ? c : (empty ? c2 : nc);
}

// masked_fill compat (masking.py:195-202): the column holds the window plus
// nu sentinel entries (-sent in max space), `sent_first` if some sit before the
// window.  Merges them into the window result M (and its LSE `lse` for
// softmax); returns false when the sentinel wins in hard mode (no gradient).
template <int MODE>
__device__ __forceinline__ bool fill_merge(float& M, float& lse, float nu, float sent,
                                           bool sent_first, float tau2, float itau2) {
  if (nu <= 0.f) return true;
  const float ms = -sent;
  if (MODE == M_HARD) {
    if (M > ms || (M == ms && !sent_first)) return true;
    M = ms;
    return false;
  }
  if (MODE == M_LSE) {
    float m = M, s = 1.f;
    lse_merge(m, s, ms, nu, tau2);
    M = fmaf(lg2f(s), itau2, m);
    return true;
  }
  float m = lse, s = 1.f, q = M - lse;
  soft_merge(m, s, q, ms, nu, 0.f, tau2);
  M = m + q / s;
  lse = fmaf(lg2f(s), itau2, m);
  return true;
}


// ---------------------------------------------------------------------------
// evaluators.  The single-leaf kinds (the common case: a Pred / NormPred / a
// materialised trace directly under a temporal operator) are compile-time
// specialisations with the row's pointers hoisted into registers; EK_GEN
// interprets any fused expression.  Element indices are row-relative ints.
// ---------------------------------------------------------------------------
// EK_AFF: affine leaf, any element stride; EK_AFF1 / EK_NORM / EK_SRC: unit element
// stride of the source(s) and gradient destination(s) (contiguous [B, T] planes:
// addresses are row base + j, so every strided sweep uses immediate offsets);
// EK_PAIR: interleaved (x, y) pair.  expr_kind() checks the strides.
enum ExprKind { EK_GEN = 0, EK_AFF = 1, EK_NORM = 2, EK_SRC = 3, EK_PAIR = 4, EK_AFF1 = 5 };

__device__ __forceinline__ float sqrt_fast(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct LeafRegs {
  const float* p1;
  const float* p2;
  float* g1;
  float* g2;
  int es1, es2, ges1, ges2;
  int st1, st2;
  float s_in, s_out, c, cx, cy;
  __device__ __forceinline__ LeafRegs(const DExpr& e, long long row) {
    const DLeaf& L = e.leaf[0];
    st1 = L.st1;
    st2 = L.st2;
    s_in = L.s_in;
    s_out = L.s_out;
    c = L.c;
    cx = L.cx;
    cy = L.cy;
    p1 = p2 = nullptr;
    g1 = g2 = nullptr;
    es1 = es2 = ges1 = ges2 = 0;
    if (L.kind != LEAF_CONST) {
      const DSrc& s = e.src[L.src];
      p1 = s.p + row * s.rs;
      es1 = (int)s.es;
      const DDst& d = e.dst[L.src];
      if (d.p) {
        g1 = d.p + row * d.rs;
        ges1 = (int)d.es;
      }
    }
    if (L.kind == LEAF_NORM) {
      const DSrc& s = e.src[L.src2];
      p2 = s.p + row * s.rs;
      es2 = (int)s.es;
      const DDst& d = e.dst[L.src2];
      if (d.p) {
        g2 = d.p + row * d.rs;
        ges2 = (int)d.es;
      }
    }
  }
  // store-mode at compile time (every gradient destination of the leaf is a first writer)
  template <bool ST>
  __device__ __forceinline__ static void put1t(float* p, int j, float g) {
    if (p) {
      if (ST) p[j] = g;
      else p[j] += g;
    }
  }
  __device__ __forceinline__ bool all_store() const { return (g1 == nullptr || st1) && (g2 == nullptr || st2); }
  __device__ __forceinline__ static void put1(float* p, int j, float g, int st) {
    if (p) {
      if (st) p[j] = g;
      else p[j] += g;
    }
  }
  __device__ __forceinline__ static void put(float* p, int es, int j, float g, int st) {
    if (p) {
      float* q = p + (long long)j * es;
      if (st) *q = g;
      else *q += g;
    }
  }
};

template <int MODE, int EK>
struct Ev;

template <int MODE>
struct Ev<MODE, EK_AFF> : LeafRegs {
  struct Raw {
    float x;
  };
  __device__ __forceinline__ Ev(const DExpr& e, long long row, const ModeP&) : LeafRegs(e, row) {}
  __device__ __forceinline__ Raw load(int j) const { return Raw{ld_na(p1 + (long long)j * es1)}; }
  __device__ __forceinline__ float value(int, Raw r) const { return s_out * __fadd_rn(s_in * r.x, c); }
  // the reference's float64 value (fp32 inputs / constants are exact in fp64)
  __device__ __forceinline__ double value64(int, Raw r) const {
    return (double)s_out * fma((double)s_in, (double)r.x, (double)c);
  }
  __device__ __forceinline__ void grad(int j, Raw, float g) const { put(g1, ges1, j, g * (s_out * s_in), st1); }
  template <bool ST>
  __device__ __forceinline__ void grad_t(int j, Raw r, float g) const { grad(j, r, g); }
};

template <int MODE>
struct Ev<MODE, EK_AFF1> : LeafRegs {
  struct Raw {
    float x;
  };
  __device__ __forceinline__ Ev(const DExpr& e, long long row, const ModeP&) : LeafRegs(e, row) {}
  __device__ __forceinline__ Raw load(int j) const { return Raw{ld_na(p1 + j)}; }
  __device__ __forceinline__ float value(int, Raw r) const { return s_out * __fadd_rn(s_in * r.x, c); }
  __device__ __forceinline__ double value64(int, Raw r) const {
    return (double)s_out * fma((double)s_in, (double)r.x, (double)c);
  }
  __device__ __forceinline__ void grad(int j, Raw, float g) const { put1(g1, j, g * (s_out * s_in), st1); }
  template <bool ST>
  __device__ __forceinline__ void grad_t(int j, Raw, float g) const { put1t<ST>(g1, j, g * (s_out * s_in)); }
};

template <int MODE>
struct Ev<MODE, EK_SRC> : LeafRegs {
  struct Raw {
    float x;
  };
  __device__ __forceinline__ Ev(const DExpr& e, long long row, const ModeP&) : LeafRegs(e, row) {}
  __device__ __forceinline__ Raw load(int j) const { return Raw{ld_na(p1 + j)}; }
  __device__ __forceinline__ float value(int, Raw r) const { return s_out * r.x; }
  __device__ __forceinline__ double value64(int, Raw r) const { return (double)s_out * (double)r.x; }
  __device__ __forceinline__ void grad(int j, Raw, float g) const { put1(g1, j, g * s_out, st1); }
  template <bool ST>
  __device__ __forceinline__ void grad_t(int j, Raw, float g) const { put1t<ST>(g1, j, g * s_out); }
};

template <int MODE>
struct Ev<MODE, EK_NORM> : LeafRegs {
  struct Raw {
    float x, y;
  };
  bool pair;  // (x, y) interleaved in one [.., T, 2] tensor: one 8-byte load per sample
  __device__ __forceinline__ Ev(const DExpr& e, long long row, const ModeP&) : LeafRegs(e, row) {
    pair = (p2 == p1 + 1) && es1 == 2 && es2 == 2 && ((reinterpret_cast<uintptr_t>(p1) & 7) == 0);
  }
  __device__ __forceinline__ Raw load(int j) const { return Raw{ld_na(p1 + j), ld_na(p2 + j)}; }
  __device__ __forceinline__ float value(int, Raw r) const {
    float dx = r.x - cx, dy = r.y - cy;
    return s_out * __fadd_rn(s_in * sqrt_fast(fmaf(dx, dx, dy * dy)), c);
  }
  __device__ __forceinline__ double value64(int, Raw r) const {
    const double dx = (double)r.x - (double)cx, dy = (double)r.y - (double)cy;
    return (double)s_out * fma((double)s_in, sqrt(fma(dx, dx, dy * dy)), (double)c);
  }
  __device__ __forceinline__ void grad(int j, Raw r, float g) const {
    float dx = r.x - cx, dy = r.y - cy;
    float d2 = fmaf(dx, dx, dy * dy);
    float sc = d2 > 0.f ? g * (s_out * s_in) * rsqrt_fast(d2) : 0.f;
    put1(g1, j, dx * sc, st1);
    put1(g2, j, dy * sc, st2);
  }
  template <bool ST>
  __device__ __forceinline__ void grad_t(int j, Raw r, float g) const {
    float dx = r.x - cx, dy = r.y - cy;
    float d2 = fmaf(dx, dx, dy * dy);
    float sc = d2 > 0.f ? g * (s_out * s_in) * rsqrt_fast(d2) : 0.f;
    put1t<ST>(g1, j, dx * sc);
    put1t<ST>(g2, j, dy * sc);
  }
};

// NormPred over an interleaved (x, y) pair ([.., T, 2] tensor): one 8-byte load
// per sample and, when both gradients are stored into an interleaved buffer,
// one 8-byte store.
template <int MODE>
struct Ev<MODE, EK_PAIR> : LeafRegs {
  struct Raw {
    float x, y;
  };
  bool gpair;
  __device__ __forceinline__ Ev(const DExpr& e, long long row, const ModeP&) : LeafRegs(e, row) {
    gpair = g1 != nullptr && g2 == g1 + 1 && ges1 == 2 && ges2 == 2 && st1 && st2 &&
            ((reinterpret_cast<uintptr_t>(g1) & 7) == 0);
  }
  __device__ __forceinline__ Raw load(int j) const {
    float2 v = ld_na2(reinterpret_cast<const float2*>(p1) + j);
    return Raw{v.x, v.y};
  }
  __device__ __forceinline__ float value(int, Raw r) const {
    float dx = r.x - cx, dy = r.y - cy;
    return s_out * __fadd_rn(s_in * sqrt_fast(fmaf(dx, dx, dy * dy)), c);
  }
  __device__ __forceinline__ double value64(int, Raw r) const {
    const double dx = (double)r.x - (double)cx, dy = (double)r.y - (double)cy;
    return (double)s_out * fma((double)s_in, sqrt(fma(dx, dx, dy * dy)), (double)c);
  }
  __device__ __forceinline__ void grad(int j, Raw r, float g) const {
    float dx = r.x - cx, dy = r.y - cy;
    float d2 = fmaf(dx, dx, dy * dy);
    float sc = d2 > 0.f ? g * (s_out * s_in) * rsqrt_fast(d2) : 0.f;
    if (gpair) {
      reinterpret_cast<float2*>(g1)[j] = make_float2(dx * sc, dy * sc);
    } else {
      put(g1, ges1, j, dx * sc, st1);
      put(g2, ges2, j, dy * sc, st2);
    }
  }
  template <bool ST>
  __device__ __forceinline__ void grad_t(int j, Raw r, float g) const { grad(j, r, g); }
};

template <int MODE>
struct Ev<MODE, EK_GEN> {
  struct Raw {};
  const DExpr* e;
  long long row;
  ModeP mp;
  __device__ __forceinline__ Ev(const DExpr& ex, long long r, const ModeP& m) : e(&ex), row(r), mp(m) {}
  __device__ __forceinline__ Raw load(int) const { return Raw{}; }
  __device__ __forceinline__ float value(int j, Raw) const { return expr_eval<MODE>(*e, row, j, mp); }
  __device__ __forceinline__ double value64(int j, Raw) const { return (double)expr_eval<MODE>(*e, row, j, mp); }
  __device__ __forceinline__ void grad(int j, Raw, float g) const { expr_vjp<MODE>(*e, row, j, g, mp); }
  template <bool ST>
  __device__ __forceinline__ void grad_t(int j, Raw r, float g) const { grad(j, r, g); }
  __device__ __forceinline__ bool all_store() const { return false; }
};

// host-side choice of the evaluator for an expression
__host__ __device__ inline int expr_kind(const DExpr& e) {
  if (e.n_step != 1) return EK_GEN;
  int k = e.leaf[0].kind;
  // unit element stride of source i and of its gradient destination (if any)
  auto unit = [&](int i) { return e.src[i].es == 1 && (e.dst[i].p == nullptr || e.dst[i].es == 1); };
  if (k == LEAF_AFFINE) return unit(e.leaf[0].src) ? EK_AFF1 : EK_AFF;
  if (k == LEAF_NORM) {
    const DSrc& a = e.src[e.leaf[0].src];
    const DSrc& b = e.src[e.leaf[0].src2];
    bool pair = b.p == a.p + 1 && a.es == 2 && b.es == 2 && a.rs == b.rs && (a.rs % 2 == 0) &&
                ((reinterpret_cast<uintptr_t>(a.p) & 7) == 0);
    if (pair) return EK_PAIR;
    return (unit(e.leaf[0].src) && unit(e.leaf[0].src2)) ? EK_NORM : EK_GEN;
  }
  if (k == LEAF_SRC) return unit(e.leaf[0].src) ? EK_SRC : EK_GEN;
  return EK_GEN;
}

// floor(i / K) for 0 <= i < 2^24 with a float reciprocal (exact after correction)
__device__ __forceinline__ int div_k(int i, int K, float invK) {
  int q = __float2int_rz((float)i * invK);
  int r = i - q * K;
  q += (r >= K) ? 1 : 0;
  q -= (r < 0) ? 1 : 0;
  return q;
}

}  // namespace stlg
