// fg_cav.cuh — timed Eventually / Always (hard and LSE modes) for K = b - a + 1 >= 17:
// chunk-aligned van Herk / Gil-Werman.
//
// Semantics as fg_reg.cuh (masking.py:160-205, tape.py:340-380).  A tile stages
// N = 16 T samples; thread q owns the chunk [16q, 16q + 16) in registers.  The
// reduction blocks ARE the chunks, so no block boundary ever falls inside a thread's
// registers: with K - 1 = 16 d + c (0 <= c < 16), the window starting at i = 16q + k
// ends in chunk q' = q + d + [k + c >= 16] at offset o = (k + c) mod 16, and
//     window(i) = suffix_q(k) (+) fold(chunks q+1 .. q'-1) (+) prefix_q'(o).
// Each thread scans its chunk both ways in registers (prefixes also go to shared
// memory for the remote reads), publishes its chunk total, and folds the d - 1 / d
// middle totals once.  A window finish is two monoid combines and one shared
// load; the result is written into the prefix slot it consumed (each slot is read
// by exactly one window), then stored coalesced.  Exact monoids (fg_reg.cuh).
#pragma once
#include <type_traits>

#include "fg_reg.cuh"

namespace stlg {

// prefix scan of the chunk -> P0 / P1 (own padded slots), total -> TOT; the suffix
// scan overwrites x in registers.
template <int RK>
__device__ __forceinline__ void cav_scans(RSt (&x)[RG_EPT], float tau2, float* P0, float* P1,
                                          float* T0, float* T1, float* P2 = nullptr, float* T2 = nullptr) {
  const int base = threadIdx.x * (RG_EPT + 1);
  RSt run = x[0];
  P0[base] = run.m;
  if (RK != RK_HARD) P1[base] = run.s;
  if (rk3<RK>()) P2[base] = run.q;
#pragma unroll
  for (int k = 1; k < RG_EPT; ++k) {
    run = rcomb_s<RK>(run, x[k], tau2);
    P0[base + k] = run.m;
    if (RK != RK_HARD) P1[base + k] = run.s;
    if (rk3<RK>()) P2[base + k] = run.q;
  }
  T0[threadIdx.x] = run.m;
  if (RK != RK_HARD) T1[threadIdx.x] = run.s;
  if (rk3<RK>()) T2[threadIdx.x] = run.q;
#pragma unroll
  for (int k = RG_EPT - 2; k >= 0; --k) x[k] = rcomb_s<RK>(x[k], x[k + 1], tau2);
}

// middle folds: A0 = chunks q+1 .. q+d-1, A1 = A0 (+) chunk q+d (identity when empty /
// past the tile; such windows are never finished)
template <int RK, int NW>
__device__ __forceinline__ void cav_middle(int d, float tau2, const float* T0, const float* T1, RSt& A0,
                                           RSt& A1, const float* T2 = nullptr) {
  const int q = threadIdx.x;
  RSt a = rident<RK>();
  const int last = q + d < NW * 32 ? q + d : NW * 32;  // exclusive bound of readable chunks
  for (int j = q + 1; j < q + d && j < last; ++j)
    a = rcomb<RK>(a, RSt{T0[j], RK == RK_HARD ? 0.f : T1[j], rk3<RK>() ? T2[j] : 0.f}, tau2);
  A0 = a;
  if (q + d < NW * 32)
    a = rcomb<RK>(a, RSt{T0[q + d], RK == RK_HARD ? 0.f : T1[q + d], rk3<RK>() ? T2[q + d] : 0.f}, tau2);
  A1 = a;
}

// window finish for i = 16 q + k in [lo, hi) (FULL: the whole chunk), descending k:
// fin(k, i, w, slot)
template <int RK, bool FULL, typename Fin>
__device__ __forceinline__ void cav_windows(const RSt (&S)[RG_EPT], RSt A0, RSt A1, int d, int c,
                                            float tau2, int lo, int hi, const float* P0,
                                            const float* P1, Fin&& fin, const float* P2 = nullptr) {
  const int q = threadIdx.x;
  const int i0 = q * RG_EPT;
  const int sb = (q + d) * (RG_EPT + 1) + c;  // slot of o = k + c in chunk q + d
#pragma unroll
  for (int k = RG_EPT - 1; k >= 0; --k) {
    const int i = i0 + k;
    if (FULL || (i >= lo && i < hi)) {
      const bool up = k + c >= RG_EPT;       // the window ends in chunk q + d + 1
      const int sl = sb + k + (up ? 1 : 0);  // 17 (q + d + up) + (k + c - 16 up)
      RSt w = rcomb<RK>(S[k], up ? A1 : A0, tau2);
      const RSt pv{P0[sl], RK == RK_HARD ? 0.f : P1[sl], rk3<RK>() ? P2[sl] : 0.f};
      w = rcomb<RK>(w, pv, tau2);
      fin(k, i, w, sl);
    }
  }
}


// ---------------------------------------------------------------------------
// LSE frame sums.  When every chunk of a tile spans tau2 (max - min) <= FS_RANGE
// (log2 units), chunk q works in the frame f_q = its max: terms E = payload *
// 2^{tau2 (e - f_q)} lie in [2^-120, 1] (normal fp32), so the chunk's prefix /
// suffix sums are plain adds, the chunk total is the exact-form state (f_q, sum)
// for the middle fold, and a window is  S alpha + beta + P gamma  in the frame
// M = max(f_q, m_A, f_q') with per-thread factors for the two remote chunks.
// Any term lost to underflow is < 2^-126 against a sum >= 2^-120 of the dominant
// part, so the result equals the exact monoid to fp32 rounding.  A tile with a
// wider chunk takes the exact path (same kernel, uniform branch).
// ---------------------------------------------------------------------------
constexpr float FS_RANGE = 120.f;
#ifndef CAV_LB
#define CAV_LB 16  // global loads batched per thread in the staging / VJP sweeps
#endif

struct FsCase {
  float M, al, be, ga;
};

// chunk frame (max over live terms; -FLT_MAX if none) and the width flag
__device__ __forceinline__ bool fs_frame(const RSt (&x)[RG_EPT], bool gl, float tau2, float& f) {
  float mx = -FLT_MAX, mn = FLT_MAX;
#pragma unroll
  for (int k = 0; k < RG_EPT; ++k) {
    const bool live = !gl || x[k].s != 0.f;
    mx = live ? fmaxf(mx, x[k].m) : mx;
    mn = live ? fminf(mn, x[k].m) : mn;
  }
  f = mx;
  return mx > mn && tau2 * (mx - mn) > FS_RANGE;
}

// E_k -> prefix sums in P0 (own slots), chunk state (f, total) -> T0 / T1;
// E is overwritten by the suffix sums
__device__ __forceinline__ void fs_scans(float (&E)[RG_EPT], float f, float* P0, float* T0, float* T1) {
  const int base = threadIdx.x * (RG_EPT + 1);
  float run = 0.f;
#pragma unroll
  for (int k = 0; k < RG_EPT; ++k) {
    run += E[k];
    P0[base + k] = run;
  }
  T0[threadIdx.x] = f;
  T1[threadIdx.x] = run;
#pragma unroll
  for (int k = RG_EPT - 2; k >= 0; --k) E[k] += E[k + 1];
}

__device__ __forceinline__ FsCase fs_case(float f, RSt A, float fp, float tau2) {
  FsCase r;
  r.M = fmaxf(fmaxf(f, A.m), fp);
  r.al = ex2f(tau2 * (f - r.M));
  r.be = A.s * ex2f(tau2 * (A.m - r.M));
  r.ga = ex2f(tau2 * (fp - r.M));
  return r;
}

// window finish in frame sums: fin(k, i, M, s, slot), descending k
template <bool FULL, typename Fin>
__device__ __forceinline__ void fs_windows(const float (&S)[RG_EPT], const FsCase& c0, const FsCase& c1,
                                           int d, int c, int lo, int hi, const float* P0, Fin&& fin) {
  const int q = threadIdx.x;
  const int i0 = q * RG_EPT;
  const int sb = (q + d) * (RG_EPT + 1) + c;
#pragma unroll
  for (int k = RG_EPT - 1; k >= 0; --k) {
    const int i = i0 + k;
    if (FULL || (i >= lo && i < hi)) {
      const bool up = k + c >= RG_EPT;
      const int sl = sb + k + (up ? 1 : 0);
      const float s = fmaf(S[k], up ? c1.al : c0.al, fmaf(P0[sl], up ? c1.ga : c0.ga, up ? c1.be : c0.be));
      fin(k, i, up ? c1.M : c0.M, s, sl);
    }
  }
}

// Forward after staging: x = the tile's chunk values (max space).  Scans, middle
// folds, window finish into the consumed prefix slots, coalesced stores.
template <int RK, int NW>
__device__ __forceinline__ void cav_fwd_core(const FGParams& p, long long row, int t0, int J, float padv,
                                             RSt (&x)[RG_EPT], float* P0, float* P1, float* T0, float* T1,
                                             float* P2 = nullptr, float* T2 = nullptr) {
  using C = RC<NW>;
  constexpr int T = C::T, SS = C::SS;
  const int K = p.K;
  const int d = (K - 1) >> 4, c = (K - 1) & 15;
  const int L = (int)p.L;
  const int nvalid = L - p.b;
  const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2, sg = p.sg;
  const float czero = p.canon ? 0.f : -0.f;
  float* outr = p.out + row * L;
  float* auxr = ((RK == RK_LSE || RK == RK_SOFT || RK == RK_HARDI) && p.aux != nullptr) ? p.aux + row * L : nullptr;
  const int tend = (t0 + J < L ? t0 + J : L) - t0;
  const int tid = threadIdx.x;
  const int i0 = tid * RG_EPT;
  const bool full = i0 + RG_EPT <= J && t0 + i0 + RG_EPT <= nvalid;
  bool fs_done = false;
  if constexpr (RK == RK_LSE) {
    float f;
    const bool wide = fs_frame(x, false, tau2, f);
    if (!__syncthreads_or(wide)) {
      fs_done = true;
      float E[RG_EPT];
#pragma unroll
      for (int k = 0; k < RG_EPT; ++k) E[k] = ex2f(tau2 * (x[k].m - f));
      fs_scans(E, f, P0, T0, T1);
      __syncthreads();
      RSt A0, A1;
      cav_middle<RK_LSE, NW>(d, tau2, T0, T1, A0, A1);
      const float fp0 = tid + d < T ? T0[tid + d] : -FLT_MAX;
      const float fp1 = tid + d + 1 < T ? T0[tid + d + 1] : -FLT_MAX;
      const FsCase c0 = fs_case(f, A0, fp0, tau2), c1 = fs_case(f, A1, fp1, tau2);
      auto fin = [&](int, int i, float M, float s, int sl) {
        const float l2 = lg2f(s);
        const float v = fmaf(l2, itau2, M);
        const bool live = full || t0 + i < nvalid;
        P0[sl] = __fadd_rn(live ? sg * v : padv, czero);
        P1[sl] = live ? sg * fmaf(l2, itau2, M - v) : 0.f;  // residual of v
      };
      if (full) fs_windows<true>(E, c0, c1, d, c, 0, J, P0, fin);
      else fs_windows<false>(E, c0, c1, d, c, 0, J, P0, fin);
    }
  }
  if (!fs_done) {
    cav_scans<RK>(x, tau2, P0, P1, T0, T1, P2, T2);  // own slots only: no barrier needed before
    __syncthreads();
    RSt A0, A1;
    cav_middle<RK, NW>(d, tau2, T0, T1, A0, A1, T2);
    auto fin = [&](int, int i, RSt w, int sl) {
      const float l2 = (RK == RK_HARD || RK == RK_HARDI) ? 0.f : lg2f(w.s);
      const bool live = full || t0 + i < nvalid;
      if (RK == RK_HARDI) {  // value; aux: the first arg-max for the backward, as its offset
                             // in the window (K <= 1024: 16 bits; 0xffff: no live window)
        P0[sl] = __fadd_rn(live ? sg * w.m : padv, czero);
        P1[sl] = __int_as_float(live ? __float_as_int(w.s) - (t0 + p.a + i) : 0xffff);
      } else if (RK == RK_SOFT) {  // value m + q / s; aux: the window LSE (max space) for the backward
        const float v = w.m + w.q / w.s;
        P0[sl] = __fadd_rn(live ? sg * v : padv, czero);
        P1[sl] = live ? fmaf(l2, itau2, w.m) : 0.f;
      } else {
        const float v = (RK == RK_HARD) ? w.m : fmaf(l2, itau2, w.m);
        P0[sl] = __fadd_rn(live ? sg * v : padv, czero);
        if (RK == RK_LSE) P1[sl] = live ? sg * fmaf(l2, itau2, w.m - v) : 0.f;  // residual of v
      }
    };
    if (full) cav_windows<RK, true>(x, A0, A1, d, c, tau2, 0, J, P0, P1, fin, P2);
    else cav_windows<RK, false>(x, A0, A1, d, c, tau2, 0, J, P0, P1, fin, P2);
  }
  __syncthreads();
  {
    const float* src = P0 + rpad(tid + K - 1);
    float* op = outr + t0 + tid;
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k)
      if (tid + k * T < tend) op[k * T] = src[k * SS];
    if (auxr != nullptr) {  // LSE: low word of the double-float trace (bf16 plane); softmax:
                            // window LSE; hard: arg-max offset (uint16 plane in the row's aux words)
      const float* src1 = P1 + rpad(tid + K - 1);
      if (RK == RK_HARDI) {
        unsigned short* ap = reinterpret_cast<unsigned short*>(auxr) + t0 + tid;
#pragma unroll
        for (int k = 0; k < RG_EPT; ++k)
          if (tid + k * T < tend) ap[k * T] = (unsigned short)__float_as_int(src1[k * SS]);
      } else if (RK == RK_LSE) {
        unsigned short* ap = reinterpret_cast<unsigned short*>(auxr) + t0 + tid;
#pragma unroll
        for (int k = 0; k < RG_EPT; ++k)
          if (tid + k * T < tend) ap[k * T] = lo_pack(src1[k * SS]);
      } else {
        float* ap = auxr + t0 + tid;
#pragma unroll
        for (int k = 0; k < RG_EPT; ++k)
          if (tid + k * T < tend) ap[k * T] = src1[k * SS];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// forward (hard: RK_HARD, LSE: RK_LSE)
// ---------------------------------------------------------------------------
template <int RK, int MODE, int EK, int NW>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB + 2) k_cav_fwd(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  extern __shared__ float rsm[];
  __shared__ float T0[T], T1[RK == RK_HARD ? 1 : T], T2[rk3<RK>() ? T : 1];
  float* P0 = rsm;
  float* P1 = rsm + C::NP;      // LSE / softmax / arg-max outputs
  float* P2 = rsm + 2 * C::NP;  // softmax only
  const int K = p.K;
  const int d = (K - 1) >> 4, c = (K - 1) & 15;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = N - K + 1;
  const int t0 = blockIdx.x * J;
  const int nvalid = L - p.b;
  const int s0 = t0 + p.a;
  const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2, sg = p.sg;
  const float czero = p.canon ? 0.f : -0.f;  // x + (-0) == x for every x: canon is one add
  (void)d, (void)c, (void)tau2, (void)itau2;  // unused by some instantiations
  Ev<MODE, EK> ev(p.child, row, p.mp);
  const float padv = p.pad_last ? ev.value(L - 1, ev.load(L - 1)) : p.pad_value;
  float* outr = p.out + row * L;
  float* auxr = ((RK == RK_LSE || RK == RK_SOFT || RK == RK_HARDI) && p.aux != nullptr) ? p.aux + row * L : nullptr;
  const int tend = (t0 + J < L ? t0 + J : L) - t0;
  const int tid = threadIdx.x;
  if (t0 >= nvalid) {  // every output of the tile overruns
    for (int i = tid; i < tend; i += T) {
      outr[t0 + i] = __fadd_rn(padv, czero);
      if (auxr && RK == RK_HARDI) reinterpret_cast<unsigned short*>(auxr)[t0 + i] = 0xffff;
      else if (auxr && RK == RK_LSE) reinterpret_cast<unsigned short*>(auxr)[t0 + i] = 0;
      else if (auxr) auxr[t0 + i] = 0.f;
    }
    return;
  }
  {
    float* dst = P0 + tid + (tid >> 4);
    const int jb = s0 + tid;
    if (s0 + N <= L) {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += CAV_LB) {
        typename Ev<MODE, EK>::Raw r[CAV_LB];
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) r[k] = ev.load(jb + (h + k) * T);
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) dst[(h + k) * SS] = sg * ev.value(jb + (h + k) * T, r[k]);
      }
    } else {  // past the row end: replicate the last sample (feeds overrun windows only)
#pragma unroll
      for (int h = 0; h < RG_EPT; h += CAV_LB) {
        typename Ev<MODE, EK>::Raw r[CAV_LB];
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          const int j = jb + (h + k) * T;
          r[k] = ev.load(j < L ? j : L - 1);
        }
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          const int j = jb + (h + k) * T;
          dst[(h + k) * SS] = sg * ev.value(j < L ? j : L - 1, r[k]);
        }
      }
    }
  }
  __syncthreads();
  RSt x[RG_EPT];
#pragma unroll
  for (int k = 0; k < RG_EPT; ++k)  // RK_HARDI: the global child index rides in s
    x[k] = RSt{P0[tid * (RG_EPT + 1) + k], RK == RK_HARDI ? __int_as_float(s0 + tid * RG_EPT + k) : 1.f};
  cav_fwd_core<RK, NW>(p, row, t0, J, padv, x, P0, P1, T0, T1, P2, T2);
}

// ---------------------------------------------------------------------------
// backward, LSE (gather form over outputs t; RK_GLSE)
// ---------------------------------------------------------------------------
template <int EK, int NW>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB_B + 1) k_cav_bwd_lse(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  extern __shared__ float rsm[];
  __shared__ float T0[T], T1[T];
  __shared__ float padsum_sh;
  float* P0 = rsm;
  float* P1 = rsm + C::NP;
  const int K = p.K;
  const int d = (K - 1) >> 4, c = (K - 1) & 15;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = N - K + 1;  // owned child elements per tile
  const int j0 = blockIdx.x * J;
  const int tb = j0 - p.b;  // local index 0 <-> output t = tb
  const int nvalid = L - p.b;
  const float tau2 = p.mp.tau2, sg = p.sg;
  const float nsg = -sg, nt2sg = -tau2 * sg;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  const unsigned short* lor =  // low word of M (double-float, bf16 plane)
      p.aux_in ? reinterpret_cast<const unsigned short*>(p.aux_in + row * L) : nullptr;
  const int tid = threadIdx.x;
  // phase 1: e_t = -M_t (max space), g_t, lo_t; (-FLT_MAX, 0, 0) outside [0, nvalid)
  {
    const int so = tid + (tid >> 4);
    const int tt = tb + tid;
    if (tb >= 0 && tb + N <= nvalid) {
      const float* cp = cot + tt;
      const float* mp = outr + tt;
      const unsigned short* lp = lor ? lor + tt : nullptr;
#pragma unroll
      for (int h = 0; h < RG_EPT; h += CAV_LB) {
        float gv[CAV_LB], mv[CAV_LB], lv[CAV_LB];
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          gv[k] = ld_na(cp + (h + k) * T);
          mv[k] = ld_na(mp + (h + k) * T);
          lv[k] = lp ? lo_ld(lp + (h + k) * T) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          P0[so + (h + k) * SS] = nsg * mv[k];
          // the low word of M folded into the weight: g 2^{-tau2 sg lo} (|tau2 lo| << 1)
          P1[so + (h + k) * SS] = lp ? gv[k] * ex2f(nt2sg * lv[k]) : gv[k];
        }
      }
    } else {
      const int thi = nvalid > 0 ? nvalid - 1 : 0;
#pragma unroll
      for (int h = 0; h < RG_EPT; h += CAV_LB) {
        float gv[CAV_LB], mv[CAV_LB], lv[CAV_LB];
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          const int t = tt + (h + k) * T;
          const int tc = t < 0 ? 0 : (t > thi ? thi : t);  // clamped loads: no branches
          gv[k] = ld_na(cot + tc);
          mv[k] = ld_na(outr + tc);
          lv[k] = lor ? lo_ld(lor + tc) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          const int t = tt + (h + k) * T;
          const bool v = t >= 0 && t < nvalid;
          P0[so + (h + k) * SS] = v ? nsg * mv[k] : -FLT_MAX;
          P1[so + (h + k) * SS] = v ? (lor ? gv[k] * ex2f(nt2sg * lv[k]) : gv[k]) : 0.f;
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
    const int qq = tid * (RG_EPT + 1) + k;
    x[k] = RSt{P0[qq], P1[qq]};
  }
  const bool full = tid * RG_EPT + RG_EPT <= J;
  float f;
  const bool wide = fs_frame(x, true, tau2, f);
  if (!__syncthreads_or(wide)) {
    // E = g' 2^{tau2 (e - f)}, g' = g 2^{-tau2 sg lo} from the staging
    float E[RG_EPT];
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) E[k] = x[k].s != 0.f ? x[k].s * ex2f(tau2 * (x[k].m - f)) : 0.f;
    fs_scans(E, f, P0, T0, T1);
    __syncthreads();
    RSt A0, A1;
    cav_middle<RK_GLSE, NW>(d, tau2, T0, T1, A0, A1);
    const float fp0 = tid + d < T ? T0[tid + d] : -FLT_MAX;
    const float fp1 = tid + d + 1 < T ? T0[tid + d + 1] : -FLT_MAX;
    const FsCase c0 = fs_case(f, A0, fp0, tau2), c1 = fs_case(f, A1, fp1, tau2);
    auto fin = [&](int, int, float M, float s, int sl) {
      P0[sl] = M;
      P1[sl] = s;
    };
    if (full) fs_windows<true>(E, c0, c1, d, c, 0, J, P0, fin);
    else fs_windows<false>(E, c0, c1, d, c, 0, J, P0, fin);
  } else {
    cav_scans<RK_GLSE>(x, tau2, P0, P1, T0, T1);
    __syncthreads();
    RSt A0, A1;
    cav_middle<RK_GLSE, NW>(d, tau2, T0, T1, A0, A1);
    auto fin = [&](int, int, RSt w, int sl) {
      P0[sl] = w.m;
      P1[sl] = w.s;
    };
    if (full) cav_windows<RK_GLSE, true>(x, A0, A1, d, c, tau2, 0, J, P0, P1, fin);
    else cav_windows<RK_GLSE, false>(x, A0, A1, d, c, tau2, 0, J, P0, P1, fin);
  }
  __syncthreads();
  // phase 3: child element j = j0 + i <- window over t in [j - b, j - a] (local start i)
  Ev<M_LSE, EK> ev(p.child, row, p.mp);
  const int jn = (j0 + J < L ? j0 + J : L) - j0;
  const float padsum = padsum_sh;
  const int slb = rpad(tid + K - 1);
  const int jb = j0 + tid;
  const int jpad = L - 1 - jb;  // (h + u) T == jpad <=> element L - 1
#pragma unroll
  for (int h = 0; h < RG_EPT; h += CAV_LB) {
    typename Ev<M_LSE, EK>::Raw r[CAV_LB];
#pragma unroll
    for (int u = 0; u < CAV_LB; ++u)
      if (tid + (h + u) * T < jn) r[u] = ev.load(jb + (h + u) * T);
#pragma unroll
    for (int u = 0; u < CAV_LB; ++u) {
      if (tid + (h + u) * T < jn) {
        const int j = jb + (h + u) * T;
        const int sl = slb + (h + u) * SS;
        // S == 0 comes with m = -FLT_MAX or u_j + m <= 0: the product is an exact 0
        float g = P1[sl] * ex2f(tau2 * fmaf(sg, ev.value(j, r[u]), P0[sl]));
        g += ((h + u) * T == jpad) ? padsum : 0.f;
        ev.grad(j, r[u], g);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward, softmax (gather form over outputs t; RK_GSOFT).  The reference VJP of
// the softmax-weighted window (tape.py:360-380) gives child j
//   sum_t g_t 2^{tau2 (u_j - L_t)} (1 + tau (u_j - M_t))
//     = 2^{tau2 (u_j + m)} [A + tau ((u_j - c) A - Bc)],
//   A = sum g_t 2^{-tau2 L_t - m},  Bc = sum g_t (M_t - c) 2^{-tau2 L_t - m}
// with L_t the forward's window LSE (aux), M_t the trace (max space) and c a
// per-tile centre (keeps the final difference small).
// ---------------------------------------------------------------------------
template <int EK, int NW>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB_B) k_cav_bwd_soft(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  extern __shared__ float rsm[];
  __shared__ float T0[T], T1[T], T2[T];
  __shared__ float padsum_sh;
  float* P0 = rsm;
  float* P1 = rsm + C::NP;
  float* P2 = rsm + 2 * C::NP;
  const int K = p.K;
  const int d = (K - 1) >> 4, c = (K - 1) & 15;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = N - K + 1;  // owned child elements per tile
  const int j0 = blockIdx.x * J;
  const int tb = j0 - p.b;  // local index 0 <-> output t = tb
  const int nvalid = L - p.b;
  const float tau = p.mp.tau, tau2 = p.mp.tau2, sg = p.sg;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  const float* lser = p.aux_in + row * L;
  const int tid = threadIdx.x;
  const int thi = nvalid > 0 ? nvalid - 1 : 0;
  const float cc = nvalid > 0 ? sg * outr[tb < 0 ? 0 : (tb > thi ? thi : tb)] : 0.f;  // centre
  {
    const int so = tid + (tid >> 4);
    const int tt = tb + tid;
    const bool interior = tb >= 0 && tb + N <= nvalid;
#pragma unroll
    for (int h = 0; h < RG_EPT; h += CAV_LB) {
      float gv[CAV_LB], mv[CAV_LB], lv[CAV_LB];
#pragma unroll
      for (int k = 0; k < CAV_LB; ++k) {
        const int t = tt + (h + k) * T;
        const int tc = interior ? t : (t < 0 ? 0 : (t > thi ? thi : t));
        gv[k] = ld_na(cot + tc);
        mv[k] = ld_na(outr + tc);
        lv[k] = ld_na(lser + tc);
      }
#pragma unroll
      for (int k = 0; k < CAV_LB; ++k) {
        const int t = tt + (h + k) * T;
        const bool v = interior || (t >= 0 && t < nvalid);
        P0[so + (h + k) * SS] = v ? -lv[k] : -FLT_MAX;
        P1[so + (h + k) * SS] = v ? gv[k] : 0.f;
        P2[so + (h + k) * SS] = v ? gv[k] * (sg * mv[k] - cc) : 0.f;
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
    const int qq = tid * (RG_EPT + 1) + k;
    x[k] = RSt{P0[qq], P1[qq], P2[qq]};
  }
  const bool full = tid * RG_EPT + RG_EPT <= J;
  cav_scans<RK_GSOFT>(x, tau2, P0, P1, T0, T1, P2, T2);
  __syncthreads();
  {
    RSt A0, A1;
    cav_middle<RK_GSOFT, NW>(d, tau2, T0, T1, A0, A1, T2);
    auto fin = [&](int, int, RSt w, int sl) {
      P0[sl] = w.m;
      P1[sl] = w.s;
      P2[sl] = w.q;
    };
    if (full) cav_windows<RK_GSOFT, true>(x, A0, A1, d, c, tau2, 0, J, P0, P1, fin, P2);
    else cav_windows<RK_GSOFT, false>(x, A0, A1, d, c, tau2, 0, J, P0, P1, fin, P2);
  }
  __syncthreads();
  Ev<M_SOFT, EK> ev(p.child, row, p.mp);
  const int jn = (j0 + J < L ? j0 + J : L) - j0;
  const float padsum = padsum_sh;
  const int slb = rpad(tid + K - 1);
  const int jb = j0 + tid;
  const int jpad = L - 1 - jb;
#pragma unroll
  for (int h = 0; h < RG_EPT; h += CAV_LB) {
    typename Ev<M_SOFT, EK>::Raw r[CAV_LB];
#pragma unroll
    for (int u = 0; u < CAV_LB; ++u)
      if (tid + (h + u) * T < jn) r[u] = ev.load(jb + (h + u) * T);
#pragma unroll
    for (int u = 0; u < CAV_LB; ++u) {
      if (tid + (h + u) * T < jn) {
        const int j = jb + (h + u) * T;
        const int sl = slb + (h + u) * SS;
        const float uj = sg * ev.value(j, r[u]);
        const float A = P1[sl];
        // A == 0 comes with m = -FLT_MAX (nothing live) or u_j + m <= 0: exact 0
        float g = ex2f(tau2 * (uj + P0[sl])) * fmaf(tau, fmaf(uj - cc, A, -P2[sl]), A);
        g += ((h + u) * T == jpad) ? padsum : 0.f;
        ev.grad(j, r[u], g);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward, hard (RK_HARDI).  The first argmax a(i) of window i is
// non-decreasing in i, so the windows routed to one child element form one
// contiguous run of window starts.  Each thread sums its runs in registers; a
// segmented warp-shuffle scan (plus one cross-warp step) carries the runs that
// continue across chunk boundaries, and every run total is written once, by the
// thread holding its last window, with a plain shared store: deterministic, no
// atomics.  Then the fused child VJP over the owned elements.
// ---------------------------------------------------------------------------
struct RunSeg {
  int key;    // key of the trailing run
  float s;    // its (partial) sum
  int whole;  // the trailing run covers the whole covered range
};
__device__ __forceinline__ RunSeg run_comb(RunSeg lo, RunSeg hi) {  // lo: earlier windows
  return (hi.whole && hi.key == lo.key) ? RunSeg{hi.key, lo.s + hi.s, lo.whole} : hi;
}
__device__ __forceinline__ RunSeg run_shfl_up(RunSeg v, int o) {
  return RunSeg{__shfl_up_sync(0xffffffffu, v.key, o), __shfl_up_sync(0xffffffffu, v.s, o),
                __shfl_up_sync(0xffffffffu, v.whole, o)};
}

template <int EK, int NW, bool IDX>
__global__ void __launch_bounds__(RC<NW>::T, RC<NW>::MINB_B + (IDX ? 1 : 0)) k_cav_bwd_hard(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS;
  constexpr int NOKEY = 0x7fffffff;  // windows past the tile: g = 0, key above every element
  extern __shared__ float rsm[];
  __shared__ float T0[T], T1[T];
  __shared__ RunSeg WR[NW];
  __shared__ int WK[NW];
  __shared__ float padsum_sh;
  float* P0 = rsm;
  float* P1 = rsm + C::NP;
  // IDX: no scans reuse P0 / P1 after the keys and cotangents reach registers, so the
  // run totals take P1's space (two arrays: one more resident CTA per SM)
  float* G = IDX ? rsm + C::NP : rsm + 2 * C::NP;
  const int K = p.K;
  const int d = (K - 1) >> 4, c = (K - 1) & 15;
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
  const int lane = tid & 31, warp = tid >> 5;
  Ev<M_HARD, EK> ev(p.child, row, p.mp);
  // IDX: the forward stored every window's first arg-max (its offset in the window, a
  // uint16 plane in the aux words): the keys come from it directly — no child loads, no
  // scans (10 B per sample: g, offset, d c)
  int key[RG_EPT];
  RSt x[RG_EPT];
  float g[RG_EPT];
  if constexpr (IDX) {
    const int so = tid + (tid >> 4);
    const int tb = first + tid - p.a;
    const unsigned short* ix = reinterpret_cast<const unsigned short*>(p.aux_in + row * L);
    const int thi = nvalid > 0 ? nvalid - 1 : 0;
#pragma unroll
    for (int h = 0; h < RG_EPT; h += CAV_LB) {
      float gv[CAV_LB];
      int iv[CAV_LB];
#pragma unroll
      for (int k = 0; k < CAV_LB; ++k) {
        const int t = tb + (h + k) * T;
        const int tc = t < 0 ? 0 : (t > thi ? thi : t);
        gv[k] = ld_na(cot + tc);
        iv[k] = __ldg(ix + tc);
      }
#pragma unroll
      for (int k = 0; k < CAV_LB; ++k) {
        const int t = tb + (h + k) * T;
        const bool wv = tid + (h + k) * T < nwin && t >= 0 && t < nvalid;
        // key = window-local arg-max (offset + window index); keys stay non-decreasing:
        // 0 below the row start, NOKEY past the live windows
        const int kk = wv ? iv[k] + tid + (h + k) * T : (t < 0 ? 0 : NOKEY);
        P0[so + (h + k) * SS] = __int_as_float(kk);
        P1[so + (h + k) * SS] = wv ? gv[k] : 0.f;
      }
    }
  } else {
  // phase 1: child values u (window start i <-> t = first + i - a)
  {
    const int so = tid + (tid >> 4);
    const int jb = first + tid;
    const int tb = jb - p.a;
    if (first >= 0 && first + N <= L && first - p.a >= 0 && first - p.a + nwin <= nvalid) {
#pragma unroll
      for (int h = 0; h < RG_EPT; h += CAV_LB) {
        typename Ev<M_HARD, EK>::Raw r[CAV_LB];
        float gv[CAV_LB];
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          r[k] = ev.load(jb + (h + k) * T);
          gv[k] = ld_na(cot + tb + (h + k) * T);  // i >= nwin: masked below
        }
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          P0[so + (h + k) * SS] = sg * ev.value(jb + (h + k) * T, r[k]);
          P1[so + (h + k) * SS] = (tid + (h + k) * T < nwin) ? gv[k] : 0.f;
        }
      }
    } else {  // clamped loads: samples outside the row feed no live window
      const int thi = nvalid > 0 ? nvalid - 1 : 0;
#pragma unroll
      for (int h = 0; h < RG_EPT; h += CAV_LB) {
        typename Ev<M_HARD, EK>::Raw r[CAV_LB];
        float gv[CAV_LB];
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          const int j = jb + (h + k) * T, t = tb + (h + k) * T;
          r[k] = ev.load(j < 0 ? 0 : (j >= L ? L - 1 : j));
          gv[k] = ld_na(cot + (t < 0 ? 0 : (t > thi ? thi : t)));
        }
#pragma unroll
        for (int k = 0; k < CAV_LB; ++k) {
          const int j = jb + (h + k) * T, t = tb + (h + k) * T;
          const bool wv = tid + (h + k) * T < nwin && t >= 0 && t < nvalid;
          P0[so + (h + k) * SS] = sg * ev.value(j < 0 ? 0 : (j >= L ? L - 1 : j), r[k]);
          P1[so + (h + k) * SS] = wv ? gv[k] : 0.f;
        }
      }
    }
  }
  }
  if (tid < 32) {  // overrun outputs route to c[L-1] ('last' padding)
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
  const float padsum = padsum_sh;
  const int kpad = (padsum != 0.f) ? L - 1 - first : -1;  // local index receiving the pad sum
  {
    const int q0 = tid * (RG_EPT + 1);
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) {
      if (IDX) key[k] = __float_as_int(P0[q0 + k]);
      else x[k] = RSt{P0[q0 + k], __int_as_float(tid * RG_EPT + k), 0.f};
      g[k] = P1[q0 + k];
    }
  }
  if constexpr (IDX) __syncthreads();  // every P1 read done before G (its space) is written
  {
    const int q0 = tid * (RG_EPT + 1);
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) G[q0 + k] = (tid * RG_EPT + k == kpad) ? padsum : 0.f;
  }
  // run totals land in other threads' G slots: every slot zeroed first (the scans' barrier
  // does this on the recomputing path)
  if constexpr (IDX) __syncthreads();
  if constexpr (!IDX) {
    cav_scans<RK_HARDI>(x, 0.f, P0, P1, T0, T1);
    __syncthreads();
    RSt A0, A1;
    cav_middle<RK_HARDI, NW>(d, 0.f, T0, T1, A0, A1);
    auto fin = [&](int k, int, RSt w, int) { key[k] = __float_as_int(w.s); };
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) key[k] = NOKEY;
    if (tid * RG_EPT + RG_EPT <= nwin) cav_windows<RK_HARDI, true>(x, A0, A1, d, c, 0.f, 0, nwin, P0, P1, fin);
    else cav_windows<RK_HARDI, false>(x, A0, A1, d, c, 0.f, 0, nwin, P0, P1, fin);
  }
  // runs of equal keys (ascending window order), branch-free: an interior run is
  // stored where it ends; the first / last runs go through the carry scan
  const int kf = key[0];
  float sf = 0.f, acc = 0.f;
  {
    int cur = kf;
    bool firstrun = true;
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) {
      const bool chg = key[k] != cur;
      if (chg && !firstrun && cur != NOKEY) G[rpad(cur)] = acc + (cur == kpad ? padsum : 0.f);
      sf = (chg && firstrun) ? acc : sf;
      firstrun = firstrun && !chg;
      acc = chg ? g[k] : acc + g[k];
      cur = key[k];
    }
    if (firstrun) sf = acc;
  }
  const float sl = acc;
  const int kl = key[RG_EPT - 1];
  const bool single = kf == kl;
  // carries: inclusive segmented scan of the trailing runs over lanes, then warps
  RunSeg v{kl, sl, single};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const RunSeg y = run_shfl_up(v, o);
    if (lane >= o) v = run_comb(y, v);
  }
  RunSeg ex = run_shfl_up(v, 1);
  const int kf_next_lane = __shfl_down_sync(0xffffffffu, kf, 1);
  if (lane == 31) WR[warp] = v;
  if (lane == 0) WK[warp] = kf;
  __syncthreads();
  RunSeg wc{NOKEY, 0.f, 0};  // fold of the warps below
#pragma unroll
  for (int w = 0; w < NW - 1; ++w)
    if (w < warp) wc = (w == 0) ? WR[0] : run_comb(wc, WR[w]);
  const RunSeg cin = lane == 0 ? wc : (warp > 0 ? run_comb(wc, ex) : ex);
  const float carry = (cin.key == kf && kf != NOKEY) ? cin.s : 0.f;
  const int kn = lane < 31 ? kf_next_lane : (warp + 1 < NW ? WK[warp + 1] : NOKEY - 1);
  if (!single && kf != NOKEY) G[rpad(kf)] = carry + sf + (kf == kpad ? padsum : 0.f);
  if (kl != NOKEY && kn != kl) G[rpad(kl)] = (single ? carry + sl : sl) + (kl == kpad ? padsum : 0.f);
  __syncthreads();
  // phase 3: owned local indices [K - 1, K - 1 + Jo): fused child VJP
  const int jn = (j0 + Jo < L ? j0 + Jo : L) - j0;
  const int gb = rpad(tid + K - 1);
  const int jb = j0 + tid;
  auto vjp = [&](auto store) {
    constexpr bool ST = decltype(store)::value;
#pragma unroll
    for (int h = 0; h < RG_EPT; h += CAV_LB) {
      typename Ev<M_HARD, EK>::Raw r[CAV_LB];
      // (affine / trace children need no value for their VJP: no reload)
      constexpr bool need_raw = !(EK == EK_AFF || EK == EK_AFF1 || EK == EK_SRC);
#pragma unroll
      for (int u = 0; u < CAV_LB; ++u)
        if (need_raw && tid + (h + u) * T < jn) r[u] = ev.load(jb + (h + u) * T);
#pragma unroll
      for (int u = 0; u < CAV_LB; ++u)
        if (tid + (h + u) * T < jn) ev.template grad_t<ST>(jb + (h + u) * T, r[u], G[gb + (h + u) * SS]);
    }
  };
  if (ev.all_store()) vjp(std::true_type{});
  else vjp(std::false_type{});
}

}  // namespace stlg
