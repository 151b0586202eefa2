// fg_unt.cu — untimed Eventually / Always forward, hard and LSE (masking.py:217-227,
// tape.py:475-535: out[t] = R_{j = t .. L-1} s[j], a reverse scan per row, no padding,
// no `+ 0.0` canonicalisation).
//
// Per tile (one CTA walking a row's 4096-sample tiles, or one CTA per 1024-sample tile
// for small batches — UN_SEQ / UN_LB below): coalesced loads through the typed child
// evaluator, a transpose through shared memory, each thread scans its 16-sample chunk in registers, a
// warp-shuffle scan and one cross-warp step give every thread the fold of the rest of
// its tile; the carry of the tiles before it in scan order comes from registers
// (sequential walk) or from the look-back slots (lookback.cuh: aggregates only, folded in
// a fixed order, so the bits do not depend on scheduling); the outputs leave through
// shared memory with coalesced stores.
#include "fg_reg.cuh"
#include "lookback.cuh"

namespace stlg {

// Two shapes of the same kernels:
//   LB = false, NW = 8: one CTA per row walks its 4096-sample tiles from the scan start with
//                       the carry in registers (large batches: rows fill the GPU);
//   LB = true,  NW = 2: one CTA per 1024-sample tile, carries from the look-back slots
//                       (lookback.cuh) — small batches / long rows (BASELINE C5's batch 64).
constexpr int UN_SEQ = 8, UN_LB = 2;
static_assert(RC<UN_LB>::N == LB_MIN_TILE, "look-back slots are sized for 1024-sample tiles");

// scan bounds of this CTA: every tile of the row (sequential, row = blockIdx.x) or the one
// tile of its look-back ticket (row-major over B x ntiles)
template <bool LB>
__device__ __forceinline__ void unt_span(const FGParams& p, int ntiles, long long& row, int& s0, int& s1) {
  if (LB) {
    const int tk = lb_ticket(p.lb);
    row = tk / ntiles;
    s0 = tk - (int)row * ntiles;
    s1 = s0 + 1;
  } else {
    row = blockIdx.x;
    s0 = 0;
    s1 = ntiles;
  }
}

template <int RK, int MODE, int EK, int NW, bool LB>
__global__ void __launch_bounds__(RC<NW>::T, LB ? 8 : 4) k_unt_fwd(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS, NP = C::NP;
  __shared__ float P[NP];
  __shared__ RSt WS[NW];
  const int L = (int)p.L;
  const int ntiles = (L + N - 1) / N;
  long long row;
  int s0, s1;
  unt_span<LB>(p, ntiles, row, s0, s1);
  const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2, sg = p.sg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ev<MODE, EK> ev(p.child, row, p.mp);
  float* outr = p.out + row * L;
  const RSt id = rident<RK>();
  unsigned* slots = LB ? p.lb + LB_WORDS + (size_t)row * ntiles * LB_WORDS : nullptr;
  RSt seq = id;  // sequential shape: fold of every sample after the current tile
  for (int s = s0; s < s1; ++s) {
    const int c0 = (ntiles - 1 - s) * N;  // scan order: from the row end
    const int nt = (L - c0 < N) ? L - c0 : N;  // live samples in this tile
    {
      float* dst = P + tid + (tid >> 4);
      const int jb = c0 + tid;
      if (nt == N) {
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
          for (int k = 0; k < 8; ++k) {
            const int j = jb + (h + k) * T;
            r[k] = ev.load(j < L ? j : L - 1);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = jb + (h + k) * T;
            dst[(h + k) * SS] = sg * ev.value(j < L ? j : L - 1, r[k]);
          }
        }
      }
    }
    __syncthreads();
    // chunk [16 tid, 16 tid + 16): suffix scan in registers (past the row end: identity)
    RSt S[RG_EPT];
    const int q0 = tid * (RG_EPT + 1), i0 = tid * RG_EPT;
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) S[k] = (i0 + k < nt) ? RSt{P[q0 + k], 1.f, 0.f} : id;
#pragma unroll
    for (int k = RG_EPT - 2; k >= 0; --k) S[k] = rcomb_s<RK>(S[k], S[k + 1], tau2);
    // fold of the later threads of the warp, then of the later warps and tiles
    RSt v = S[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      RSt w{__shfl_down_sync(0xffffffffu, v.m, o), RK == RK_HARDV ? 0.f : __shfl_down_sync(0xffffffffu, v.s, o), 0.f};
      if (lane + o < 32) v = rcomb<RK>(v, w, tau2);
    }
    RSt ex{__shfl_down_sync(0xffffffffu, v.m, 1), RK == RK_HARDV ? 0.f : __shfl_down_sync(0xffffffffu, v.s, 1), 0.f};
    if (lane == 0) WS[warp] = v;
    __syncthreads();
    RSt tile = WS[NW - 1];  // the tile's aggregate
#pragma unroll
    for (int w = NW - 2; w >= 0; --w) tile = rcomb<RK>(WS[w], tile, tau2);
    RSt carry = seq;
    if (LB) {
      if (tid == 0 && s + 1 < ntiles) {  // publish (later tiles in scan order fold it)
        const unsigned pw[2] = {__float_as_uint(tile.m), __float_as_uint(tile.s)};
        lb_publish<2>(slots + (size_t)s * LB_WORDS, pw);
      }
      // agg_{s-1} (+) (... (+) (agg_0 (+) id)): the sequential walk's expression
      carry = lb_carry<2>(slots, s, id, [&](RSt x, const unsigned* w) {
        return rcomb<RK>(RSt{__uint_as_float(w[0]), __uint_as_float(w[1]), 0.f}, x, tau2);
      });
    }
    RSt cw = carry;
#pragma unroll
    for (int w = NW - 1; w > 0; --w)
      if (w > warp) cw = rcomb<RK>(WS[w], cw, tau2);
    const RSt cin = lane < 31 ? rcomb<RK>(ex, cw, tau2) : cw;
    float lo[RK == RK_LSE ? RG_EPT : 1];
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) {
      const RSt o = rcomb<RK>(S[k], cin, tau2);
      const float l2 = (RK == RK_HARDV) ? 0.f : lg2f(o.s);
      const float val = (RK == RK_HARDV) ? o.m : fmaf(l2, itau2, o.m);
      // LSE: residual of the fp32 trace (double-float M = val + lo, as k_cav_fwd), so the
      // backward's weights 2^{tau2 (u - M)} do not inherit tau |M| eps32
      if (RK == RK_LSE) lo[k] = sg * fmaf(l2, itau2, o.m - val);
      P[q0 + k] = sg * val;  // own slots: read by the coalesced store after the barrier
    }
    if (!LB) seq = rcomb<RK>(tile, seq, tau2);
    __syncthreads();
    const float* src = P + tid + (tid >> 4);
    float* op = outr + c0 + tid;
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k)
      if (tid + k * T < nt) op[k * T] = src[k * SS];
    if (RK == RK_LSE && p.aux != nullptr) {  // the low words leave through the same buffer
      __syncthreads();
#pragma unroll
      for (int k = 0; k < RG_EPT; ++k) P[q0 + k] = lo[k];
      __syncthreads();
      unsigned short* ap = reinterpret_cast<unsigned short*>(p.aux + row * L) + c0 + tid;  // bf16 plane
#pragma unroll
      for (int k = 0; k < RG_EPT; ++k)
        if (tid + k * T < nt) ap[k * T] = lo_pack(src[k * SS]);
    }
    __syncthreads();
  }
}

// Untimed LSE backward (gather form, tape.py:475-535): child j receives
//   2^{tau2 u_j} sum_{t <= j} g_t 2^{-tau2 M_t}
// — an inclusive prefix scan over the outputs of the (e_t = -M_t, g_t) elements
// (RK_GLSE), scan order from the row start, then the fused child VJP over the tile.
template <int EK, int NW, bool LB>
__global__ void __launch_bounds__(RC<NW>::T, LB ? 8 : 3) k_unt_bwd_lse(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS, NP = C::NP;
  __shared__ float B0[NP], B1[NP];
  __shared__ RSt WP[NW];
  const int L = (int)p.L;
  const int ntiles = (L + N - 1) / N;
  long long row;
  int s0, s1;
  unt_span<LB>(p, ntiles, row, s0, s1);
  const float tau2 = p.mp.tau2, sg = p.sg, nsg = -p.sg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  const unsigned short* lor =  // trace low word (bf16 plane)
      p.aux_in != nullptr ? reinterpret_cast<const unsigned short*>(p.aux_in + row * L) : nullptr;
  Ev<M_LSE, EK> ev(p.child, row, p.mp);
  const RSt id = rident<RK_GLSE>();
  const int so = tid + (tid >> 4), q0 = tid * (RG_EPT + 1), i0 = tid * RG_EPT;
  unsigned* slots = LB ? p.lb + LB_WORDS + (size_t)row * ntiles * LB_WORDS : nullptr;
  RSt seq = id;  // sequential shape: fold of every output before the current tile
  for (int s = s0; s < s1; ++s) {
    const int c0 = s * N;  // scan order: from the row start
    const int nt = (L - c0 < N) ? L - c0 : N;
#pragma unroll
    for (int h = 0; h < RG_EPT; h += 8) {
      float gv[8], mv[8], lv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = c0 + tid + (h + k) * T;
        const int tc = t < L ? t : L - 1;
        gv[k] = ld_na(cot + tc);
        mv[k] = ld_na(outr + tc);
        lv[k] = lor != nullptr ? lo_ld(lor + tc) : 0.f;
      }
      // M = hi + lo: the low word rides in the weight, g 2^{-tau2 lo} (|tau2 lo| << 1)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (lor != nullptr) gv[k] *= ex2f(-tau2 * sg * lv[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool v = tid + (h + k) * T < nt;
        B0[so + (h + k) * SS] = v ? nsg * mv[k] : -FLT_MAX;
        B1[so + (h + k) * SS] = v ? gv[k] : 0.f;
      }
    }
    __syncthreads();
    RSt Pk[RG_EPT];
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) Pk[k] = (i0 + k < nt) ? RSt{B0[q0 + k], B1[q0 + k], 0.f} : id;
#pragma unroll
    for (int k = 1; k < RG_EPT; ++k) Pk[k] = rcomb<RK_GLSE>(Pk[k - 1], Pk[k], tau2);
    RSt v = Pk[RG_EPT - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      RSt w{__shfl_up_sync(0xffffffffu, v.m, o), __shfl_up_sync(0xffffffffu, v.s, o), 0.f};
      if (lane >= o) v = rcomb<RK_GLSE>(w, v, tau2);
    }
    RSt ex{__shfl_up_sync(0xffffffffu, v.m, 1), __shfl_up_sync(0xffffffffu, v.s, 1), 0.f};
    if (lane == 31) WP[warp] = v;
    __syncthreads();
    RSt tile = WP[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) tile = rcomb<RK_GLSE>(tile, WP[w], tau2);
    RSt carry = seq;
    if (LB) {
      if (tid == 0 && s + 1 < ntiles) {
        const unsigned pw[2] = {__float_as_uint(tile.m), __float_as_uint(tile.s)};
        lb_publish<2>(slots + (size_t)s * LB_WORDS, pw);
      }
      // ((id (+) agg_0) (+) agg_1) ... (+) agg_{s-1}
      carry = lb_carry<2>(slots, s, id, [&](RSt x, const unsigned* w) {
        return rcomb<RK_GLSE>(x, RSt{__uint_as_float(w[0]), __uint_as_float(w[1]), 0.f}, tau2);
      });
    }
    RSt cw = carry;
#pragma unroll
    for (int w = 0; w < NW - 1; ++w)
      if (w < warp) cw = rcomb<RK_GLSE>(cw, WP[w], tau2);
    const RSt cin = lane > 0 ? rcomb<RK_GLSE>(cw, ex, tau2) : cw;
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) {
      const RSt o = rcomb<RK_GLSE>(cin, Pk[k], tau2);
      B0[q0 + k] = o.m;  // own slots
      B1[q0 + k] = o.s;
    }
    if (!LB) seq = rcomb<RK_GLSE>(seq, tile, tau2);
    __syncthreads();
    const int jb = c0 + tid;
#pragma unroll
    for (int h = 0; h < RG_EPT; h += 8) {
      typename Ev<M_LSE, EK>::Raw r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (tid + (h + u) * T < nt) r[u] = ev.load(jb + (h + u) * T);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (tid + (h + u) * T < nt) {
          const int j = jb + (h + u) * T;
          const int sl = so + (h + u) * SS;
          // S == 0 comes with m = -FLT_MAX or u_j + m <= 0: the product is an exact 0
          const float g = B1[sl] * ex2f(tau2 * fmaf(sg, ev.value(j, r[u]), B0[sl]));
          ev.grad(j, r[u], g);
        }
      }
    }
    __syncthreads();
  }
}

// Untimed hard backward (tape.py:481-491): out[t] routes its cotangent to the FIRST
// arg-max a(t) of u over [t, L-1].  a(t) is non-decreasing in t and a(i) = i for every
// target i, so the outputs sending to i form one contiguous run [t_start, i]: with the
// positions walked in descending t, the run starts at its target and ends at t_start.
// Every run total is accumulated in fp64 by a segmented scan (threads, warps and the
// carry of the tiles already done, which lie at larger t) and written ONCE, by the
// thread that owns the run's last position t_start, through the fused child VJP at i —
// deterministic (no atomics, no memset, no pointwise pass) and exact to one fp32
// rounding of the fp64 sum.  Every non-target position gets a zero gradient from its
// owner, so each gradient element is written exactly once.
struct HRun {
  int kf, kl;   // key (arg-max target) at the highest / lowest position of the range
  double tail;  // cotangent sum of the lowest run of the range (key kl)
  int whole;    // one key over the whole range
};
// hi covers larger t than lo
__device__ __forceinline__ HRun hrun_comb(HRun hi, HRun lo) {
  if (hi.kf < 0) return lo;
  if (lo.kf < 0) return hi;
  const bool join = lo.whole && lo.kf == hi.kl;
  return HRun{hi.kf, lo.kl, join ? hi.tail + lo.tail : lo.tail, hi.whole && lo.whole && lo.kf == hi.kl};
}
__device__ __forceinline__ HRun hrun_shfl_down(HRun v, int o) {
  HRun r;
  r.kf = __shfl_down_sync(0xffffffffu, v.kf, o);
  r.kl = __shfl_down_sync(0xffffffffu, v.kl, o);
  r.tail = __shfl_down_sync(0xffffffffu, v.tail, o);
  r.whole = __shfl_down_sync(0xffffffffu, v.whole, o);
  return r;
}

template <int EK, int NW, bool LB>
__global__ void __launch_bounds__(RC<NW>::T, LB ? 8 : 3) k_unt_bwd_hard(const __grid_constant__ FGParams p) {
  using C = RC<NW>;
  constexpr int T = C::T, N = C::N, SS = C::SS, NP = C::NP;
  __shared__ float U[NP];  // child values (max space), then the arg-max keys
  __shared__ float G[NP];  // cotangents
  __shared__ HRun WS[NW];
  __shared__ RSt WM[NW];
  const int L = (int)p.L;
  const int ntiles = (L + N - 1) / N;
  long long row;
  int s0, s1;
  unt_span<LB>(p, ntiles, row, s0, s1);
  const float sg = p.sg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* cot = p.cot + row * L;
  Ev<M_HARD, EK> ev(p.child, row, p.mp);
  const RSt idm = rident<RK_HARDI>();
  const HRun idr{-1, -1, 0.0, 1};
  const int so = tid + (tid >> 4), q0 = tid * (RG_EPT + 1), i0 = tid * RG_EPT;
  // look-back: arg-max aggregates in slot row 0, run aggregates in slot row 1
  unsigned* slots = LB ? p.lb + LB_WORDS + (size_t)row * ntiles * LB_WORDS : nullptr;
  unsigned* rslots = LB ? slots + (size_t)p.B * ntiles * LB_WORDS : nullptr;
  RSt mseq = idm;  // sequential shape: (max, first arg-max) of every position after the tile
  HRun rseq = idr; //                   run state of every position after the tile
  for (int s = s0; s < s1; ++s) {
    const int c0 = (ntiles - 1 - s) * N;  // scan order: from the row end
    const int nt = (L - c0 < N) ? L - c0 : N;
    {
      const int jb = c0 + tid;
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        typename Ev<M_HARD, EK>::Raw r[8];
        float gv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = jb + (h + k) * T;
          const int jc = j < L ? j : L - 1;
          r[k] = ev.load(jc);
          gv[k] = ld_na(cot + jc);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = jb + (h + k) * T;
          U[so + (h + k) * SS] = sg * ev.value(j < L ? j : L - 1, r[k]);
          G[so + (h + k) * SS] = gv[k];
        }
      }
    }
    __syncthreads();
    // suffix first-arg-max over the thread's chunk (ties keep the earlier position)
    RSt S[RG_EPT];
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k)
      S[k] = (i0 + k < nt) ? RSt{U[q0 + k], __int_as_float(c0 + i0 + k), 0.f} : idm;
#pragma unroll
    for (int k = RG_EPT - 2; k >= 0; --k) S[k] = rcomb<RK_HARDI>(S[k], S[k + 1], 0.f);
    RSt v = S[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      RSt w{__shfl_down_sync(0xffffffffu, v.m, o), __shfl_down_sync(0xffffffffu, v.s, o), 0.f};
      if (lane + o < 32) v = rcomb<RK_HARDI>(v, w, 0.f);
    }
    RSt ex{__shfl_down_sync(0xffffffffu, v.m, 1), __shfl_down_sync(0xffffffffu, v.s, 1), 0.f};
    if (lane == 0) WM[warp] = v;
    __syncthreads();
    RSt mtile = WM[NW - 1];
#pragma unroll
    for (int w = NW - 2; w >= 0; --w) mtile = rcomb<RK_HARDI>(WM[w], mtile, 0.f);
    RSt mcarry = mseq;
    if (LB) {
      if (tid == 0 && s + 1 < ntiles) {
        const unsigned pw[2] = {__float_as_uint(mtile.m), __float_as_uint(mtile.s)};
        lb_publish<2>(slots + (size_t)s * LB_WORDS, pw);
      }
      mcarry = lb_carry<2>(slots, s, idm, [&](RSt x, const unsigned* w) {
        return rcomb<RK_HARDI>(RSt{__uint_as_float(w[0]), __uint_as_float(w[1]), 0.f}, x, 0.f);
      });
    }
    RSt cw = mcarry;
#pragma unroll
    for (int w = NW - 1; w > 0; --w)
      if (w > warp) cw = rcomb<RK_HARDI>(WM[w], cw, 0.f);
    const RSt cin = lane < 31 ? rcomb<RK_HARDI>(ex, cw, 0.f) : cw;
    int key[RG_EPT];
    float gk[RG_EPT];
#pragma unroll
    for (int k = 0; k < RG_EPT; ++k) {
      const RSt o = rcomb<RK_HARDI>(S[k], cin, 0.f);
      key[k] = (i0 + k < nt) ? __float_as_int(o.s) : -1;
      gk[k] = G[q0 + k];
      if (p.fill) {  // masked_fill: the t sentinel rows of the column win ties (no gradient)
        float M = o.m, l0 = 0.f;
        const int t = c0 + i0 + k;
        if (!fill_merge<M_HARD>(M, l0, (float)t, p.sent, t > 0, 0.f, 0.f)) gk[k] = 0.f;
      }
    }
    if (!LB) mseq = rcomb<RK_HARDI>(mtile, mseq, 0.f);
    // the thread's run state over its chunk, then the segmented scan over later threads
    HRun mine = idr;
#pragma unroll
    for (int k = RG_EPT - 1; k >= 0; --k)
      if (key[k] >= 0) mine = hrun_comb(mine, HRun{key[k], key[k], (double)gk[k], 1});
    HRun rv = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      HRun w = hrun_shfl_down(rv, o);
      if (lane + o < 32) rv = hrun_comb(w, rv);
    }
    HRun rex = hrun_shfl_down(rv, 1);
    if (lane == 31) rex = idr;
    if (lane == 0) WS[warp] = rv;
    __syncthreads();  // WS visible; U / G reads done (keys go into U below)
    HRun rtile = WS[NW - 1];
#pragma unroll
    for (int w = NW - 2; w >= 0; --w) rtile = hrun_comb(rtile, WS[w]);
    HRun rcarry = rseq;
    if (LB) {
      if (tid == 0 && s + 1 < ntiles) {
        const unsigned long long tb = (unsigned long long)__double_as_longlong(rtile.tail);
        const unsigned pw[5] = {(unsigned)rtile.kf, (unsigned)rtile.kl, (unsigned)tb, (unsigned)(tb >> 32),
                                (unsigned)rtile.whole};
        lb_publish<5>(rslots + (size_t)s * LB_WORDS, pw);
      }
      rcarry = lb_carry<5>(rslots, s, idr, [&](HRun x, const unsigned* w) {
        const unsigned long long tb = (unsigned long long)w[2] | ((unsigned long long)w[3] << 32);
        return hrun_comb(x, HRun{(int)w[0], (int)w[1], __longlong_as_double((long long)tb), (int)w[4]});
      });
    }
    HRun rw = rcarry;  // later tiles, then the later warps of this tile, in descending t
#pragma unroll
    for (int w = NW - 1; w > 0; --w)
      if (w > warp) rw = hrun_comb(rw, WS[w]);
    const HRun prev = hrun_comb(rw, rex);  // everything at larger t than the thread's chunk
    if (!LB) rseq = hrun_comb(rseq, rtile);
    // walk the chunk downwards; a run that ends here (the next lower position has another
    // key) is complete: write its total at its target through the child VJP
    int pk = prev.kl;
    double ps = prev.tail;
#pragma unroll
    for (int k = RG_EPT - 1; k >= 0; --k) {
      if (key[k] < 0) continue;
      if (key[k] != pk) {
        if (pk >= 0) ev.grad(pk, ev.load(pk), (float)ps);
        pk = key[k];
        ps = 0.0;
      }
      ps += (double)gk[k];
      U[q0 + k] = __int_as_float(key[k]);
    }
    if (c0 == 0 && tid == 0 && pk >= 0) ev.grad(pk, ev.load(pk), (float)ps);  // row start
    __syncthreads();
    // zero gradient at every non-target position (coalesced)
    {
      const int jb = c0 + tid;
#pragma unroll
      for (int h = 0; h < RG_EPT; h += 8) {
        typename Ev<M_HARD, EK>::Raw r[8];
        bool z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = jb + (h + u) * T;
          z[u] = tid + (h + u) * T < nt && __float_as_int(U[so + (h + u) * SS]) != j;
          if (z[u]) r[u] = ev.load(j);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (z[u]) ev.grad(jb + (h + u) * T, r[u], 0.f);
      }
    }
    __syncthreads();
  }
}

#define UNT_DISPATCH_EK(EKV, ...)      \
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

// shape choice: the look-back kernels when the rows alone would leave the GPU short of
// CTAs (fewer rows than ~2 per SM) and a row spans several 1024-sample tiles
static bool unt_use_lb(const FGParams& p) {
  return p.lb != nullptr && p.B < 2 * 148 && p.L >= 4 * LB_MIN_TILE;
}
static cudaError_t unt_lb_reset(const FGParams& p, int rows_of_slots, cudaStream_t st) {
  const long long ntiles = (p.L + LB_MIN_TILE - 1) / LB_MIN_TILE;  // (+ the ticket slot)
  return cudaMemsetAsync(p.lb, 0, sizeof(unsigned) * LB_WORDS * (size_t)(p.B * ntiles * rows_of_slots + 1), st);
}

// register-blocked untimed forward (hard / LSE without masked_fill); false: not handled
bool launch_unt_fwd(int mode, FGParams& p, cudaStream_t st, cudaError_t& err) {
  if (p.fill || (mode != M_HARD && mode != M_LSE) || p.L >= (1LL << 30)) return false;
  const int ek = expr_kind(p.child);
  if (unt_use_lb(p)) {
    using C = RC<UN_LB>;
    const dim3 grid((unsigned)(((p.L + C::N - 1) / C::N) * p.B));  // tickets, row-major
    if ((err = unt_lb_reset(p, 1, st)) != cudaSuccess) return true;
    if (mode == M_HARD) {
      UNT_DISPATCH_EK(ek, (k_unt_fwd<RK_HARDV, M_HARD, EK, UN_LB, true><<<grid, C::T, 0, st>>>(p)))
    } else {
      UNT_DISPATCH_EK(ek, (k_unt_fwd<RK_LSE, M_LSE, EK, UN_LB, true><<<grid, C::T, 0, st>>>(p)))
    }
  } else {
    using C = RC<UN_SEQ>;
    if (mode == M_HARD) {
      UNT_DISPATCH_EK(ek, (k_unt_fwd<RK_HARDV, M_HARD, EK, UN_SEQ, false><<<(unsigned)p.B, C::T, 0, st>>>(p)))
    } else {
      UNT_DISPATCH_EK(ek, (k_unt_fwd<RK_LSE, M_LSE, EK, UN_SEQ, false><<<(unsigned)p.B, C::T, 0, st>>>(p)))
    }
  }
  count_launch();
  err = cudaGetLastError();
  return true;
}

// register-blocked untimed backward, LSE and hard (no masked_fill); false: not handled
bool launch_unt_bwd(int mode, FGParams& p, cudaStream_t st, cudaError_t& err) {
  // masked_fill: hard only (a sentinel winning the column just zeroes that output's cotangent)
  if ((p.fill && mode != M_HARD) || (mode != M_LSE && mode != M_HARD) || p.L >= (1LL << 30)) return false;
  const int ek = expr_kind(p.child);
  if (unt_use_lb(p)) {
    using C = RC<UN_LB>;
    const dim3 grid((unsigned)(((p.L + C::N - 1) / C::N) * p.B));  // tickets, row-major
    if ((err = unt_lb_reset(p, mode == M_HARD ? 2 : 1, st)) != cudaSuccess) return true;
    if (mode == M_HARD) {
      UNT_DISPATCH_EK(ek, (k_unt_bwd_hard<EK, UN_LB, true><<<grid, C::T, 0, st>>>(p)))
    } else {
      UNT_DISPATCH_EK(ek, (k_unt_bwd_lse<EK, UN_LB, true><<<grid, C::T, 0, st>>>(p)))
    }
  } else {
    using C = RC<UN_SEQ>;
    if (mode == M_HARD) {
      UNT_DISPATCH_EK(ek, (k_unt_bwd_hard<EK, UN_SEQ, false><<<(unsigned)p.B, C::T, 0, st>>>(p)))
    } else {
      UNT_DISPATCH_EK(ek, (k_unt_bwd_lse<EK, UN_SEQ, false><<<(unsigned)p.B, C::T, 0, st>>>(p)))
    }
  }
  count_launch();
  err = cudaGetLastError();
  return true;
}

}  // namespace stlg
