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
  int kind, src, src2, pad_;
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
    x = sqrtf(fmaf(dx, dx, dy * dy));
  }
  // one rounding, exactly as x + (-c) / (-x) + c in the reference
  float t = __fadd_rn(L.s_in * x, L.c);
  return L.s_out * t;
}

__device__ __forceinline__ void acc_dst(const DDst& d, long long b, long long j, float g) {
  if (d.p != nullptr) {
    float* q = d.p + b * d.rs + j * d.es;
    *q += g;
  }
}

__device__ __forceinline__ void leaf_vjp(const DExpr& e, const DLeaf& L, long long b, long long j,
                                         float g) {
  if (L.kind == LEAF_CONST) return;
  if (L.kind == LEAF_SRC) {
    acc_dst(e.dst[L.src], b, j, g * L.s_out);
    return;
  }
  float gx = g * L.s_out * L.s_in;
  if (L.kind == LEAF_AFFINE) {
    acc_dst(e.dst[L.src], b, j, gx);
    return;
  }
  float dx = ld_src(e.src[L.src], b, j) - L.cx;
  float dy = ld_src(e.src[L.src2], b, j) - L.cy;
  float d = sqrtf(fmaf(dx, dx, dy * dy));
  float inv = d > 0.f ? 1.f / d : 0.f;
  acc_dst(e.dst[L.src], b, j, gx * dx * inv);
  acc_dst(e.dst[L.src2], b, j, gx * dy * inv);
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
  float inv = 1.f / s;
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
  if (g == 0.f) return;
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
    if (a == 0.f) continue;
    if (s.op == ST_LEAF) {
      leaf_vjp(e, e.leaf[s.a], b, j, a);
    } else {
      adj[s.a] += a * w1[k];
      adj[s.b] += a * w2[k];
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

}  // namespace stlg
