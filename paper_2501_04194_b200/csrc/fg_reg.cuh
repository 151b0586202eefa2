// fg_reg.cuh — timed Eventually / Always (hard and LSE modes), register-blocked
// exact window scans.  The kernels follow `masking.trace_var`'s timed F / G
// (masking.py:160-205: windows [t+a, t+b] of the child, `overrun` outputs take
// the pad value, `+ 0.0` canonicalisation) and their tape VJPs (tape.py:340-380:
// hard max routes the cotangent to the FIRST argmax; LSE to the softmax weights
// with the detached max shift).
//
// Design (van Herk / Gil-Werman over K = b - a + 1 wide blocks, all threads busy):
//   * a tile stages N = 16 * T samples (T = 32 * NW threads, NW a template
//     parameter so every strided offset is an immediate); thread t owns the
//     contiguous chunk [16t, 16t + 16) in registers, shared memory is only the
//     transpose buffer (1 pad word per 16: conflict-free both ways);
//   * one serial sweep per chunk yields both the prefix-direction aggregate (after
//     the last block start) and the suffix-direction aggregate (up to the first
//     block end); segmented warp-shuffle scans + an NW-lane cross-warp scan turn
//     them into per-thread carries (no per-block sequential chains);
//   * pass 2 writes block-prefix states to shared memory; the suffix pass finishes
//     each window as suffix(i) (+) prefix(i + K - 1) and writes the result into the
//     prefix slot it just consumed (each slot is read by exactly one window).
// The monoids are EXACT (max-shifted LSE, first argmax): no data-dependent range
// check or fallback exists on this path.
//
// Monoid kinds (state (m, s)):
//   RK_HARD   max                     (forward, hard)   1 word
//   RK_HARDI  (max, first argmax)     (backward, hard)  s = index bits
//   RK_LSE    (m, sum 2^{tau2 (u-m)})  (forward, LSE)
//   RK_GLSE   the same merge over elements (-M_t, g_t) (backward, LSE, gather form:
//             child j receives 2^{tau2 u_j} sum_t g_t 2^{-tau2 M_t})
#pragma once
#include <cfloat>

#include "kernels.cuh"

namespace stlg {

// RK_HARDV: value-only first argmax (ties keep the earlier operand, so -0 / +0 follow
// the reference where no `+ 0.0` canonicalisation follows, e.g. untimed windows)
enum { RK_HARD = 0, RK_HARDI = 1, RK_LSE = 2, RK_GLSE = 3, RK_SOFT = 4, RK_GSOFT = 5, RK_HARDV = 6 };
constexpr int RG_EPT = 16;  // samples per thread

template <int NW>
struct RC {
  static constexpr int T = NW * 32;            // threads
  static constexpr int N = T * RG_EPT;         // staged samples
  static constexpr int NP = N + N / 16;        // padded words per array
  static constexpr int SS = T + T / 16;        // padded stride of a strided sweep
  static constexpr int MINB = 1024 / T;        // ~32 resident warps per SM (forward kernels)
  static constexpr int MINB_B = 65536 / (T * 72);  // backward kernels: ~72 registers (no spills)
};

__device__ __forceinline__ int rpad(int i) { return i + (i >> 4); }

struct RSt {
  float m, s, q;  // q: softmax payload (RK_SOFT / RK_GSOFT), otherwise unused
};
// monoid kinds with a third state word
template <int RK>
constexpr bool rk3() {
  return RK == RK_SOFT || RK == RK_GSOFT;
}
struct RSeg {
  float m, s;
  int r;  // a block boundary lies inside the covered range
};

template <int RK>
__device__ __forceinline__ RSt rident() {
  if (RK == RK_HARD || RK == RK_HARDV) return {-INFINITY, 0.f, 0.f};
  if (RK == RK_HARDI) return {-INFINITY, __int_as_float(-1), 0.f};
  return {-FLT_MAX, 0.f, 0.f};
}

// e covers earlier positions than l
template <int RK>
__device__ __forceinline__ RSt rcomb(RSt e, RSt l, float tau2) {
  if (RK == RK_HARD) return {fmaxf(e.m, l.m), 0.f, 0.f};
  if (RK == RK_HARDV) return (l.m > e.m) ? l : e;
  if (RK == RK_HARDI) return (l.m > e.m || __float_as_int(e.s) < 0) ? l : e;
  const float d = l.m - e.m;
  const float x = ex2f(-tau2 * fabsf(d));
  const bool up = d > 0.f;
  if (RK == RK_SOFT) {  // (m, s, q): s = sum 2^{tau2 (u - m)}, q = sum (u - m) 2^{tau2 (u - m)}
    const float s_up = fmaf(e.s, x, l.s), q_up = fmaf(x, fmaf(-d, e.s, e.q), l.q);
    const float s_dn = fmaf(l.s, x, e.s), q_dn = fmaf(x, fmaf(d, l.s, l.q), e.q);
    return {up ? l.m : e.m, up ? s_up : s_dn, up ? q_up : q_dn};
  }
  if (RK == RK_GSOFT) {  // (m, a, b): two payloads under one max shift
    return {up ? l.m : e.m, up ? fmaf(e.s, x, l.s) : fmaf(l.s, x, e.s),
            up ? fmaf(e.q, x, l.q) : fmaf(l.q, x, e.q)};
  }
  return {up ? l.m : e.m, up ? fmaf(e.s, x, l.s) : fmaf(l.s, x, e.s), 0.f};
}

// scan-internal combine: both operands are real states (no identity), so the
// first-argmax kind skips the identity test
template <int RK>
__device__ __forceinline__ RSt rcomb_s(RSt e, RSt l, float tau2) {
  if (RK == RK_HARDI) return (l.m > e.m) ? l : e;
  return rcomb<RK>(e, l, tau2);
}

template <int RK>
__device__ __forceinline__ RSeg rshfl_up(RSeg v, int o) {
  RSeg r;
  r.m = __shfl_up_sync(0xffffffffu, v.m, o);
  r.s = (RK == RK_HARD) ? 0.f : __shfl_up_sync(0xffffffffu, v.s, o);
  r.r = __shfl_up_sync(0xffffffffu, v.r, o);
  return r;
}
template <int RK>
__device__ __forceinline__ RSeg rshfl_down(RSeg v, int o) {
  RSeg r;
  r.m = __shfl_down_sync(0xffffffffu, v.m, o);
  r.s = (RK == RK_HARD) ? 0.f : __shfl_down_sync(0xffffffffu, v.s, o);
  r.r = __shfl_down_sync(0xffffffffu, v.r, o);
  return r;
}
template <int RK>
__device__ __forceinline__ RSeg rshfl_idx(RSeg v, int src) {
  RSeg r;
  r.m = __shfl_sync(0xffffffffu, v.m, src);
  r.s = (RK == RK_HARD) ? 0.f : __shfl_sync(0xffffffffu, v.s, src);
  r.r = __shfl_sync(0xffffffffu, v.r, src);
  return r;
}
// prefix direction: a earlier, b later
template <int RK>
__device__ __forceinline__ RSeg rsegP(RSeg a, RSeg b, float tau2) {
  RSt c = rcomb<RK>({a.m, a.s}, {b.m, b.s}, tau2);
  return b.r ? b : RSeg{c.m, c.s, a.r};
}
// suffix direction: a later, b earlier
template <int RK>
__device__ __forceinline__ RSeg rsegS(RSeg a, RSeg b, float tau2) {
  RSt c = rcomb<RK>({b.m, b.s}, {a.m, a.s}, tau2);
  return b.r ? b : RSeg{c.m, c.s, a.r};
}

// bit k (0..16): chunk position 16 t + k starts a K-block (tile-local alignment)
__device__ __forceinline__ unsigned rmask(int t, int K) {
  const int r0 = (RG_EPT * t) % K;
  unsigned m = 0;
  for (int k = r0 ? K - r0 : 0; k <= RG_EPT; k += K) m |= 1u << k;
  return m;
}

// Carry-ins of the calling thread's chunk: cP = fold of the samples of the
// current block before the chunk, cS = fold of the samples of the current block
// after it (identity / discarded where the block starts / ends inside the chunk).
// Contains the barrier that separates the chunk reads from pass 2's writes.
template <int RK, int NW>
__device__ __forceinline__ void rcarries(const RSt (&x)[RG_EPT], unsigned mask, float tau2,
                                         RSeg* WP, RSeg* WS, RSt& cP, RSt& cS) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  RSt run = x[0], sa = x[0];
  bool open = true;
#pragma unroll
  for (int k = 1; k < RG_EPT; ++k) {
    const bool rs = (mask >> k) & 1u;
    const RSt c = rcomb<RK>(run, x[k], tau2);
    run = rs ? x[k] : c;
    open = open && !rs;
    sa = open ? run : sa;
  }
  RSeg p{run.m, run.s, (mask & 0xffffu) != 0u};
  RSeg s{sa.m, sa.s, (mask & 0x1fffeu) != 0u};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const RSeg y = rshfl_up<RK>(p, o);
    const RSeg z = rshfl_down<RK>(s, o);
    if (lane >= o) p = rsegP<RK>(y, p, tau2);
    if (lane + o < 32) s = rsegS<RK>(z, s, tau2);
  }
  const RSeg pex = rshfl_up<RK>(p, 1);
  const RSeg sex = rshfl_down<RK>(s, 1);
  if (lane == 31) WP[warp] = p;
  if (lane == 0) WS[warp] = s;
  __syncthreads();
  const RSt id = rident<RK>();
  RSeg wp = lane < NW ? WP[lane < NW ? lane : 0] : RSeg{id.m, id.s, 0};
  RSeg ws = lane < NW ? WS[lane < NW ? lane : 0] : RSeg{id.m, id.s, 0};
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    const RSeg y = rshfl_up<RK>(wp, o);
    const RSeg z = rshfl_down<RK>(ws, o);
    if (lane >= o) wp = rsegP<RK>(y, wp, tau2);
    if (lane + o < NW) ws = rsegS<RK>(z, ws, tau2);
  }
  const RSeg cw_p = rshfl_idx<RK>(wp, warp > 0 ? warp - 1 : 0);
  const RSeg cw_s = rshfl_idx<RK>(ws, warp + 1 < NW ? warp + 1 : 0);
  if (lane > 0) {
    RSeg c = pex;
    if (!pex.r && warp > 0) c = rsegP<RK>(cw_p, pex, tau2);
    cP = {c.m, c.s};
  } else {
    cP = warp > 0 ? RSt{cw_p.m, cw_p.s} : id;
  }
  if (lane < 31) {
    RSeg c = sex;
    if (!sex.r && warp + 1 < NW) c = rsegS<RK>(cw_s, sex, tau2);
    cS = {c.m, c.s};
  } else {
    cS = warp + 1 < NW ? RSt{cw_s.m, cw_s.s} : id;
  }
}

// pass 2 (prefix): block-prefix states of the chunk into P0 / P1
template <int RK>
__device__ __forceinline__ void rprefix_store(const RSt (&x)[RG_EPT], unsigned mask, RSt run,
                                              float tau2, float* P0, float* P1) {
  const int base = threadIdx.x * (RG_EPT + 1);
#pragma unroll
  for (int k = 0; k < RG_EPT; ++k) {
    const RSt c = rcomb<RK>(run, x[k], tau2);
    run = ((mask >> k) & 1u) ? x[k] : c;
    P0[base + k] = run.m;
    if (RK != RK_HARD) P1[base + k] = run.s;
  }
}

// pass 2 (suffix) + window finish: fin(k, i, w, slot) for every window start
// i = 16 t + k in [lo, hi) in descending k; w = fold of [i, i + K - 1].  FULL: the
// whole chunk lies in [lo, hi) (no per-window bound check).
template <int RK, bool FULL, typename Fin>
__device__ __forceinline__ void rsuffix_windows(const RSt (&x)[RG_EPT], unsigned mask, RSt run,
                                                float tau2, int K, int lo, int hi, const float* P0,
                                                const float* P1, Fin&& fin) {
  const int i0 = threadIdx.x * RG_EPT;
#pragma unroll
  for (int k = RG_EPT - 1; k >= 0; --k) {
    const RSt c = rcomb<RK>(x[k], run, tau2);
    run = ((mask >> (k + 1)) & 1u) ? x[k] : c;
    const int i = i0 + k;
    if (FULL || (i >= lo && i < hi)) {
      const int sl = rpad(i + K - 1);
      RSt w = run;
      if (!((mask >> k) & 1u)) {
        const RSt pv{P0[sl], RK == RK_HARD ? 0.f : P1[sl]};
        w = rcomb<RK>(run, pv, tau2);
      }
      fin(k, i, w, sl);
    }
  }
}

// ---------------------------------------------------------------------------
// forward (hard: RK_HARD, LSE: RK_LSE)
// ---------------------------------------------------------------------------
template <int RK, int MODE, int EK, int NW>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB + 1) k_reg_fwd(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  extern __shared__ float rsm[];
  __shared__ RSeg WP[NW], WS[NW];
  float* P0 = rsm;
  float* P1 = rsm + C::NP;
  const int K = p.K;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = N - K + 1;
  const int t0 = blockIdx.x * J;
  const int nvalid = L - p.b;
  const int s0 = t0 + p.a;
  const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2, sg = p.sg;
  const float czero = p.canon ? 0.f : -0.f;  // x + (-0) == x for every x: canon is one add
  Ev<MODE, EK> ev(p.child, row, p.mp);
  const float padv = p.pad_last ? ev.value(L - 1, ev.load(L - 1)) : p.pad_value;
  float* outr = p.out + row * L;
  const int tend = (t0 + J < L ? t0 + J : L) - t0;
  const int tid = threadIdx.x;
  if (t0 >= nvalid) {  // every output of the tile overruns
    for (int i = tid; i < tend; i += T) outr[t0 + i] = __fadd_rn(padv, czero);
    if (RK == RK_LSE && p.aux != nullptr)
      for (int i = tid; i < tend; i += T) reinterpret_cast<unsigned short*>(p.aux + row * L)[t0 + i] = 0;
    return;
  }
  // phase 1: coalesced loads, child values -> P0 (transpose buffer)
  {
    float* dst = P0 + tid + (tid >> 4);
    const int jb = s0 + tid;
    if (s0 + N <= L) {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        typename Ev<MODE, EK>::Raw r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = ev.load(jb + (h + k) * T);
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[(h + k) * SS] = sg * ev.value(jb + (h + k) * T, r[k]);
      }
    } else {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        typename Ev<MODE, EK>::Raw r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (jb + (h + k) * T < L) r[k] = ev.load(jb + (h + k) * T);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = jb + (h + k) * T;
          // samples past the row end only feed overrun windows: any finite value
          dst[(h + k) * SS] = j < L ? sg * ev.value(j, r[k]) : 0.f;
        }
      }
    }
  }
  __syncthreads();
  RSt x[RG_EPT];
#pragma unroll
  for (int k = 0; k < RG_EPT; ++k) x[k] = RSt{P0[tid * (RG_EPT + 1) + k], 1.f};
  const unsigned mask = rmask(tid, K);
  RSt cP, cS;
  rcarries<RK, NW>(x, mask, tau2, WP, WS, cP, cS);
  rprefix_store<RK>(x, mask, cP, tau2, P0, P1);
  __syncthreads();
  const int i0 = tid * RG_EPT;
  if (i0 + RG_EPT <= J && t0 + i0 + RG_EPT <= nvalid) {
    rsuffix_windows<RK, true>(x, mask, cS, tau2, K, 0, J, P0, P1, [&](int, int, RSt w, int sl) {
      const float l2 = (RK == RK_HARD) ? 0.f : lg2f(w.s);
      const float v = (RK == RK_HARD) ? w.m : fmaf(l2, itau2, w.m);
      P0[sl] = __fadd_rn(sg * v, czero);
      if (RK == RK_LSE) P1[sl] = sg * fmaf(l2, itau2, w.m - v);  // residual of v
    });
  } else {
    rsuffix_windows<RK, false>(x, mask, cS, tau2, K, 0, J, P0, P1, [&](int, int i, RSt w, int sl) {
      const float l2 = (RK == RK_HARD) ? 0.f : lg2f(w.s);
      const float v = (RK == RK_HARD) ? w.m : fmaf(l2, itau2, w.m);
      const bool live = t0 + i < nvalid;
      P0[sl] = __fadd_rn(live ? sg * v : padv, czero);
      if (RK == RK_LSE) P1[sl] = live ? sg * fmaf(l2, itau2, w.m - v) : 0.f;
    });
  }
  __syncthreads();
  {
    const float* src = P0 + rpad(tid + K - 1);
    float* op = outr + t0 + tid;
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k)
      if (tid + k * T < tend) op[k * T] = src[k * SS];
    if (RK == RK_LSE && p.aux != nullptr) {  // low word of the double-float trace (bf16 plane)
      const float* src1 = P1 + rpad(tid + K - 1);
      unsigned short* ap = reinterpret_cast<unsigned short*>(p.aux + row * L) + t0 + tid;
#pragma unroll
      for (int k = 0; k < RG_EPT; ++k)
        if (tid + k * T < tend) ap[k * T] = lo_pack(src1[k * SS]);
    }
  }
}

// ---------------------------------------------------------------------------
// backward, LSE (gather form over outputs t; RK_GLSE)
// ---------------------------------------------------------------------------
template <int EK, int NW>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB_B) k_reg_bwd_lse(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  extern __shared__ float rsm[];
  __shared__ RSeg WP[NW], WS[NW];
  __shared__ float padsum_sh;
  float* P0 = rsm;
  float* P1 = rsm + C::NP;
  const int K = p.K;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = N - K + 1;  // owned child elements per tile
  const int j0 = blockIdx.x * J;
  const int tb = j0 - p.b;  // local index 0 <-> output t = tb
  const int nvalid = L - p.b;
  const float tau2 = p.mp.tau2, sg = p.sg;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  const unsigned short* lor =  // low word of M (double-float, bf16 plane)
      p.aux_in ? reinterpret_cast<const unsigned short*>(p.aux_in + row * L) : nullptr;
  const int tid = threadIdx.x;
  // phase 1: elements (-M_t, g_t) for t in [tb, tb + N); identity outside [0, nvalid)
  {
    float* d0 = P0 + tid + (tid >> 4);
    float* d1 = P1 + tid + (tid >> 4);
    const int tt = tb + tid;
    if (tb >= 0 && tb + N <= nvalid) {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        float gv[8], mv[8], lv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          gv[k] = ld_na(cot + tt + (h + k) * T);
          mv[k] = ld_na(outr + tt + (h + k) * T);
          lv[k] = lor ? lo_ld(lor + tt + (h + k) * T) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          d0[(h + k) * SS] = -sg * mv[k];
          d1[(h + k) * SS] = lor ? gv[k] * ex2f(-tau2 * sg * lv[k]) : gv[k];
        }
      }
    } else {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        float gv[8], mv[8], lv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int t = tt + (h + k) * T;
          const bool v = t >= 0 && t < nvalid;
          gv[k] = v ? ld_na(cot + t) : 0.f;
          mv[k] = v ? ld_na(outr + t) : 0.f;
          lv[k] = (v && lor) ? lo_ld(lor + t) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int t = tt + (h + k) * T;
          const bool v = t >= 0 && t < nvalid;
          d0[(h + k) * SS] = v ? -sg * mv[k] : -FLT_MAX;
          d1[(h + k) * SS] = lor ? gv[k] * ex2f(-tau2 * sg * lv[k]) : gv[k];
        }
      }
    }
  }
  if (tid < 32) {  // overrun outputs route to c[L-1] ('last' padding)
    float ps = 0.f;
    if (p.pad_last && L - 1 >= j0 && L - 1 < j0 + J) {
      const int t_lo = nvalid > 0 ? nvalid : 0;
      for (int t = t_lo + tid; t < L; t += 32) ps += cot[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    }
    if (tid == 0) padsum_sh = ps;
  }
  __syncthreads();
  RSt x[RG_EPT];
#pragma unroll
  for (int k = 0; k < RG_EPT; ++k) {
    const int q = tid * (RG_EPT + 1) + k;
    x[k] = RSt{P0[q], P1[q]};
  }
  const unsigned mask = rmask(tid, K);
  RSt cP, cS;
  rcarries<RK_GLSE, NW>(x, mask, tau2, WP, WS, cP, cS);
  rprefix_store<RK_GLSE>(x, mask, cP, tau2, P0, P1);
  __syncthreads();
  auto fin = [&](int, int, RSt w, int sl) {
    P0[sl] = w.m;
    P1[sl] = w.s;
  };
  if (tid * RG_EPT + RG_EPT <= J) rsuffix_windows<RK_GLSE, true>(x, mask, cS, tau2, K, 0, J, P0, P1, fin);
  else rsuffix_windows<RK_GLSE, false>(x, mask, cS, tau2, K, 0, J, P0, P1, fin);
  __syncthreads();
  // phase 3: child element j = j0 + i <- window over t in [j - b, j - a] (local start i)
  Ev<M_LSE, EK> ev(p.child, row, p.mp);
  const int jn = (j0 + J < L ? j0 + J : L) - j0;
  const float padsum = padsum_sh;
  const int slb = rpad(tid + K - 1);
  const int jb = j0 + tid;
#pragma unroll
  for (int h = 0; h < RG_EPT; h += 8) {
    typename Ev<M_LSE, EK>::Raw r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (tid + (h + u) * T < jn) r[u] = ev.load(jb + (h + u) * T);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (tid + (h + u) * T < jn) {
        const int j = jb + (h + u) * T;
        const int sl = slb + (h + u) * SS;
        // S == 0 comes with m = -FLT_MAX or u_j + m <= 0: the product is an exact 0
        float g = P1[sl] * ex2f(tau2 * fmaf(sg, ev.value(j, r[u]), P0[sl]));
        if (j == L - 1) g += padsum;
        ev.grad(j, r[u], g);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward, hard (RK_HARDI).  The first argmax a(i) of window i is
// non-decreasing in i, so each child element receives a contiguous run of
// windows: a thread accumulates runs in a register; runs strictly inside its
// chunk belong to it alone (plain store), only the two runs touching the chunk
// ends can be shared with neighbours (shared-memory atomic).
// ---------------------------------------------------------------------------
template <int EK, int NW>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB_B) k_reg_bwd_hard(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  extern __shared__ float rsm[];
  __shared__ RSeg WP[NW], WS[NW];
  __shared__ float padsum_sh;
  float* P0 = rsm;
  float* P1 = rsm + C::NP;
  float* G = rsm + 2 * C::NP;
  const int K = p.K;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int Jo = N - 2 * K + 2;    // owned child elements per tile
  const int j0 = blockIdx.x * Jo;
  const int first = j0 - (K - 1);  // local index 0 <-> child element `first`
  const int nvalid = L - p.b;
  const int nwin = N - K + 1;      // windows staged per tile
  const float sg = p.sg;
  const float* cot = p.cot + row * L;
  const int tid = threadIdx.x;
  Ev<M_HARD, EK> ev(p.child, row, p.mp);
  // phase 1: child values u and window cotangents (window start i <-> t = first + i - a)
  {
    float* d0 = P0 + tid + (tid >> 4);
    float* d1 = P1 + tid + (tid >> 4);
    const int jb = first + tid;
    const int tb = jb - p.a;
    if (first >= 0 && first + N <= L && first - p.a >= 0 && first - p.a + nwin <= nvalid) {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        typename Ev<M_HARD, EK>::Raw r[8];
        float gv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          r[k] = ev.load(jb + (h + k) * T);
          gv[k] = (tid + (h + k) * T < nwin) ? ld_na(cot + tb + (h + k) * T) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          d0[(h + k) * SS] = sg * ev.value(jb + (h + k) * T, r[k]);
          d1[(h + k) * SS] = gv[k];
        }
      }
    } else {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        typename Ev<M_HARD, EK>::Raw r[8];
        float gv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = jb + (h + k) * T, t = tb + (h + k) * T;
          if (j >= 0 && j < L) r[k] = ev.load(j);
          gv[k] = (tid + (h + k) * T < nwin && t >= 0 && t < nvalid) ? ld_na(cot + t) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = jb + (h + k) * T;
          d0[(h + k) * SS] = (j >= 0 && j < L) ? sg * ev.value(j, r[k]) : 0.f;
          d1[(h + k) * SS] = gv[k];
        }
      }
    }
  }
  if (tid < 32) {
    float ps = 0.f;
    if (p.pad_last && L - 1 >= j0 && L - 1 < j0 + Jo) {
      const int t_lo = nvalid > 0 ? nvalid : 0;
      for (int t = t_lo + tid; t < L; t += 32) ps += cot[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    }
    if (tid == 0) padsum_sh = ps;
  }
  __syncthreads();
  RSt x[RG_EPT];
  float g[RG_EPT];
  {
    const int q0 = tid * (RG_EPT + 1);
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) {
      x[k] = RSt{P0[q0 + k], __int_as_float(tid * RG_EPT + k)};
      g[k] = P1[q0 + k];
      G[q0 + k] = 0.f;
    }
  }
  const unsigned mask = rmask(tid, K);
  RSt cP, cS;
  rcarries<RK_HARDI, NW>(x, mask, 0.f, WP, WS, cP, cS);
  rprefix_store<RK_HARDI>(x, mask, cP, 0.f, P0, P1);
  __syncthreads();
  {
    int cur = -1;
    float acc = 0.f;
    bool top = true;  // the current run touches the chunk's upper end
    auto fin = [&](int k, int, RSt w, int) {
      const int am = __float_as_int(w.s);
      if (am != cur) {
        if (cur >= 0) {
          if (top) atomicAdd(&G[rpad(cur)], acc);
          else G[rpad(cur)] = acc;
        }
        top = cur < 0;
        cur = am;
        acc = 0.f;
      }
      acc += g[k];
    };
    if (tid * RG_EPT + RG_EPT <= nwin) rsuffix_windows<RK_HARDI, true>(x, mask, cS, 0.f, K, 0, nwin, P0, P1, fin);
    else rsuffix_windows<RK_HARDI, false>(x, mask, cS, 0.f, K, 0, nwin, P0, P1, fin);
    if (cur >= 0) atomicAdd(&G[rpad(cur)], acc);
  }
  __syncthreads();
  // phase 3: owned local indices [K - 1, K - 1 + Jo)
  const int jn = (j0 + Jo < L ? j0 + Jo : L) - j0;
  const float padsum = padsum_sh;
  const int gb = rpad(tid + K - 1);
  const int jb = j0 + tid;
#pragma unroll
  for (int h = 0; h < RG_EPT; h += 8) {
    typename Ev<M_HARD, EK>::Raw r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (tid + (h + u) * T < jn) r[u] = ev.load(jb + (h + u) * T);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (tid + (h + u) * T < jn) {
        const int j = jb + (h + u) * T;
        float gg = G[gb + (h + u) * SS];
        if (j == L - 1) gg += padsum;
        ev.grad(j, r[u], gg);
      }
    }
  }
}

// tile size: NW in [4, 8] warps (N = 512 NW samples) minimising staged samples per row
// Forward kernels run fastest at NW = 4 (smaller barrier groups, 8 resident CTAs)
// even with more staged overlap (C2: 0.041 vs 0.043 ms at NW = 7); backward widths
// minimise the staged samples per row.
inline int reg_pick_nw(long long L, int K, bool hard_bwd, bool fwd = false) {
  // short rows (L < 2048) may take 3-warp tiles (1536 samples) when those stage less
  const int nw_min = L < 2048 ? 3 : 4;
  if (fwd && 2048LL >= 4LL * K) return (nw_min == 3 && 1536LL >= 4LL * K && L <= 1536 - K + 1) ? 3 : 4;
  int best = -1;
  long long best_cost = 0;
  for (int nw = 8; nw >= nw_min; --nw) {
    const long long N = 512LL * nw;
    if (N < 4LL * K) continue;
    const long long J = hard_bwd ? N - 2 * K + 2 : N - K + 1;
    const long long cost = ((L + J - 1) / J) * N;
    if (best < 0 || cost < best_cost) {
      best = nw;
      best_cost = cost;
    }
  }
  return best;
}

template <typename KernT>
inline cudaError_t reg_launch(KernT k, dim3 grid, int threads, size_t smem, const FGParams& p,
                              cudaStream_t st) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<grid, threads, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

#define REG_DISPATCH_NW(NWV, ...)                 \
  switch (NWV) {                                  \
    case 3: { constexpr int NW = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int NW = 4; __VA_ARGS__; } break; \
    case 5: { constexpr int NW = 5; __VA_ARGS__; } break; \
    case 6: { constexpr int NW = 6; __VA_ARGS__; } break; \
    case 7: { constexpr int NW = 7; __VA_ARGS__; } break; \
    default: { constexpr int NW = 8; __VA_ARGS__; } break; \
  }

#define REG_DISPATCH_EK(EKV, ...)      \
  if ((EKV) == EK_AFF1) {              \
    constexpr int EK = EK_AFF1;        \
    __VA_ARGS__;                       \
  } else if ((EKV) == EK_AFF) {        \
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

}  // namespace stlg
