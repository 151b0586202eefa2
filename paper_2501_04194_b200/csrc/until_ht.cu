// until_ht.cu — hard timed Until in O(T) per row (masking.py:238-293 with Hard()).
//
// Reference, per start t with t + b <= L-1 (K = b - a + 1, u = t + a, v = t + b):
//   pm_k = min(l[t .. u+k])  (a tie keeps the earlier element),
//   term_k = min(pm_k, r[u+k])  (a tie keeps pm),   out[t] = max_k term_k  (first k).
// The per-output K loop of until.cu is replaced by block decompositions:
//   out[t] = min(A_t, V(u)),  A_t = min l[t .. u-1]  (+inf for a = 0),
//   V(u)   = max_{s in [u, v]} min(min l[u .. s], r_s),
// and with blocks of K samples aligned at multiples of K (e = end of u's block)
//   V(u)   = max(X(u), min(Smin(u), Y(v)))   (only X(u) when u starts a block)
//   X(u)   = max_{s in [u, e]} min(min l[u .. s], r_s)       clamp recurrence, backwards
//   Smin(u)= min l[u .. e]                                   backwards
//   Y(v)   = max_{s in [e+1, v]} min(min l[e+1 .. s], r_s)   forwards from the next block
// A_t is a window min over blocks of a samples (suffix / prefix walks).  Each output
// costs O(1); each sample is walked a fixed number of times.
//
// Gradient source (the reference's tie rules, one-hot for the hard mode): with
// theta = out[t], p = first position >= t with l_p <= theta and q = first position >= u
// with r_q >= theta, the source is r_q if q < p, else l_p — and theta is that source's
// value (signed zeros included).  The walks carry the source of every partial maximum
// along with its value (derivation in DESIGN.md §5), so the forward writes the value
// AT the source and the backward routes g_t to it.
//
// Backward: the CTA owning child elements [t0, t0 + NT) recomputes the sources of the
// outputs [t0 - b, t0 + NT) (every output that can route into its range) and sums their
// cotangents in shared int64 fixed point at a per-tile power-of-two scale — integer
// addition is associative, so the sums are reproducible bit for bit — then writes
// every owned element once (no memset, no float atomics).
#include <algorithm>

#include "kernels.cuh"

namespace stlg {

constexpr int HT_T = 256;    // threads per CTA
// staged span NS = a multiple of 1024 positions (32 blocks: the walks fill whole warps),
// the smallest leaving at least 512 outputs (forward) / owned elements (backward) per CTA
// after the window halo (b forward, 2b backward): NT = NS - halo
__host__ __device__ __forceinline__ int ht_ns(int halo) { return (halo + 512 + 1023) / 1024 * 1024; }
constexpr int HT_R = 1 << 30;  // source flag: right child

// Range state of the reference's Until over a range R = [s0, s1] of candidate ends s:
//   m  = min l over R, mi its first arg-min,
//   y  = max_{s in R} min(min l[s0 .. s], r_s), yi the gradient source of y.
// Combining adjacent ranges A (earlier) and B (later):
//   m = min(m_A, m_B) (a tie keeps A), y = max(y_A, min(m_A, y_B)) with the source
//   yi_A if y_A >= min(m_A, y_B), else yi_B if y_B < m_A, else l[mi_A]
// — the reference's tie rules, so the state of a range is unique and the combine is
// associative.
struct HS {
  float m, y;
  int mi, yi;
};
__device__ __forceinline__ HS hs_elem(float l, float r, int s) {
  const bool cr = r < l;  // term tie keeps pm
  return HS{l, cr ? r : l, s, cr ? (s | HT_R) : s};
}
__device__ __forceinline__ HS hs_comb(const HS& A, const HS& B) {
  HS o;
  const bool am = A.m <= B.m;
  o.m = am ? A.m : B.m;
  o.mi = am ? A.mi : B.mi;
  const bool yb = B.y < A.m;
  const float cand = yb ? B.y : A.m;
  const int ci = yb ? B.yi : A.mi;
  const bool ya = A.y >= cand;
  o.y = ya ? A.y : cand;
  o.yi = ya ? A.yi : ci;
  return o;
}
// staged arrays, padded one word per 32-block (ht_pad) so that a lane walking its own
// block and a warp reading consecutive positions are both free of bank conflicts:
//   lr[i]  = (l_i, r_i)
//   suf[i] = state over [i, end of i's 32-block],  pre[i] = state over [start of the block, i]
// (states packed as float4 {m, y, mi, yi}: one 128-bit shared load each)
__device__ __forceinline__ int ht_pad(int i) { return i + (i >> 5); }
__device__ __forceinline__ float4 hs_pack(const HS& s) {
  return make_float4(s.m, s.y, __int_as_float(s.mi), __int_as_float(s.yi));
}
__device__ __forceinline__ HS hs_unpack(const float4 v) {
  return HS{v.x, v.y, __float_as_int(v.z), __float_as_int(v.w)};
}
// mb[bk]: the state of the MB whole blocks bk+1 .. bk+MB (MB = (K-1)/32 - 1 when >= 2),
// mb1[bk] the same over MB + 1 blocks: a window of K samples spans MB or MB + 1 whole
// blocks, so it costs suffix + mb / mb1 + prefix — two combines per output for any K
// instead of O(K/32), and no loop
struct HTArr {
  float2* lr;
  float4 *sf, *pf, *mb, *mb1;
  int MB;
  __device__ __forceinline__ HS suf(int i) const { return hs_unpack(sf[ht_pad(i)]); }
  __device__ __forceinline__ HS pre(int i) const { return hs_unpack(pf[ht_pad(i)]); }
  __device__ __forceinline__ float2 at(int i) const { return lr[ht_pad(i)]; }
};

__host__ __device__ __forceinline__ int ht_padded(int NS) { return ((NS + 31) >> 5) * 33; }
// 32-bit words of the staged arrays: mb, mb1 (nb float4 each), then sf / pf (float4) and lr (float2)
__host__ __device__ __forceinline__ int ht_words(int NS) { return ((NS + 31) >> 5) * 8 + ht_padded(NS) * 10; }

__device__ __forceinline__ HTArr ht_carve(float* base, int NS, int K) {
  const int NP = ht_padded(NS);
  HTArr A;
  A.mb = reinterpret_cast<float4*>(base);
  A.mb1 = A.mb + ((NS + 31) >> 5);
  A.sf = A.mb1 + ((NS + 31) >> 5);
  A.pf = A.sf + NP;
  A.lr = reinterpret_cast<float2*>(A.pf + NP);
  const int mb = (K - 1) / 32 - 1;
  A.MB = mb >= 2 ? mb : 0;
  return A;
}

size_t ht_smem_bytes(int NS) { return (size_t)ht_words(NS) * 4; }

// stage the children over [base, base + NS) (coalesced), then walk every 32-block
// serially: one lane per block for the prefix states and one for the suffix states.
// Backward with NS <= 4 HT_T: the cotangents of the outputs at positions
// i = threadIdx.x + k HT_T < NO ride in the same load batches into gk[k] (0 outside the
// signal) and the per-warp max |g| lands in gred (a NaN / inf makes it inf).
__device__ void ht_prepare(const UParams& p, long long row, int base, int NS, const HTArr& A,
                           const float* cot = nullptr, int NO = 0, float* gk = nullptr, float* gred = nullptr) {
  const int L = (int)p.L;
  const int nb = (NS + 31) >> 5;
  const ChildEval cl(p.left, row), cr(p.right, row);
  constexpr int LB = 4;  // global loads in flight per thread before the transforms
  float gm = 0.f;
  for (int i0 = threadIdx.x; i0 < nb * 32; i0 += LB * HT_T) {
    float xl[LB], xr[LB], xg[LB];
#pragma unroll
    for (int k = 0; k < LB; ++k) {
      const int pos = base + i0 + k * HT_T;
      const int pc = pos >= 0 && pos < L ? pos : 0;
      if (cl.kind != 0 && cr.kind != 0) {
        xl[k] = cl.raw(pc);
        xr[k] = cr.raw(pc);
      }
      if (cot) xg[k] = cot[pc];
    }
    if (cot) {
#pragma unroll
      for (int k = 0; k < LB; ++k) {
        const int i = i0 + k * HT_T, pos = base + i;
        if (i >= NO) break;
        const float g = pos >= 0 && pos < L ? xg[k] : 0.f;
        const float ag = fabsf(g);
        gm = (ag == ag) ? fmaxf(gm, ag) : INFINITY;
        gk[k] = g;
      }
    }
#pragma unroll
    for (int k = 0; k < LB; ++k) {
      const int i = i0 + k * HT_T, pos = base + i;
      if (i >= nb * 32) break;
      const bool live = i < NS && pos >= 0 && pos < L;
      float l = 0.f, r = 0.f;
      if (live) {
        if (cl.kind != 0 && cr.kind != 0) {
          l = cl.apply(xl[k]);
          r = cr.apply(xr[k]);
        } else {
          l = cl.value<M_HARD>(pos, p.mp);
          r = cr.value<M_HARD>(pos, p.mp);
        }
      }
      A.lr[ht_pad(i)] = make_float2(l, r);
    }
  }
  if (cot) {
    for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if ((threadIdx.x & 31) == 0) gred[threadIdx.x >> 5] = gm;
  }
  __syncthreads();
  const int nbw = (nb + 31) & ~31;  // suffix walkers start on a warp boundary (no divergence)
  for (int w = threadIdx.x; w < nbw + nb; w += HT_T) {
    const bool fwd = w < nbw;
    if (fwd && w >= nb) continue;
    const int bk = fwd ? w : w - nbw;
    const float2* src = A.lr + bk * 33;
    const int s0 = base + bk * 32;
    if (fwd) {
      float4* dst = A.pf + bk * 33;
      HS s;
#pragma unroll
      for (int h = 0; h < 32; h += 8) {
        float2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = src[h + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const HS e = hs_elem(v[k].x, v[k].y, s0 + h + k);
          s = (h + k == 0) ? e : hs_comb(s, e);
          dst[h + k] = hs_pack(s);
        }
      }
    } else {
      float4* dst = A.sf + bk * 33;
      HS s;
#pragma unroll
      for (int h = 24; h >= 0; h -= 8) {
        float2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = src[h + k];
#pragma unroll
        for (int k = 7; k >= 0; --k) {
          const HS e = hs_elem(v[k].x, v[k].y, s0 + h + k);
          s = (h + k == 31) ? e : hs_comb(e, s);
          dst[h + k] = hs_pack(s);
        }
      }
    }
  }
  __syncthreads();
  if (A.MB > 0) {  // the MB- and (MB+1)-block aggregates (only read where they exist)
    for (int bk = threadIdx.x; bk + A.MB < nb; bk += HT_T) {
      HS s = A.pre((bk + 1) * 32 + 31);
      for (int j = 2; j <= A.MB; ++j) s = hs_comb(s, A.pre((bk + j) * 32 + 31));
      A.mb[bk] = hs_pack(s);
      if (bk + A.MB + 1 < nb) A.mb1[bk] = hs_pack(hs_comb(s, A.pre((bk + A.MB + 1) * 32 + 31)));
    }
    __syncthreads();
  }
}

// state of the staged range [i0, i1] (inclusive, relative indices)
__device__ __forceinline__ HS ht_range(const HTArr& A, int i0, int i1, int base) {
  const int b0 = i0 >> 5, b1 = i1 >> 5;
  if (b0 == b1) {  // inside one block: element by element (at most 32 steps)
    float2 v = A.at(i0);
    HS s = hs_elem(v.x, v.y, base + i0);
    for (int i = i0 + 1; i <= i1; ++i) {
      v = A.at(i);
      s = hs_comb(s, hs_elem(v.x, v.y, base + i));
    }
    return s;
  }
  HS s = A.suf(i0);
  const int m = b1 - b0 - 1;  // whole blocks between
  if (A.MB > 0 && m == A.MB) return hs_comb(hs_comb(s, hs_unpack(A.mb[b0])), A.pre(i1));
  if (A.MB > 0 && m == A.MB + 1) return hs_comb(hs_comb(s, hs_unpack(A.mb1[b0])), A.pre(i1));
  int bk = b0 + 1;
  if (A.MB > 0 && m >= A.MB) {
    s = hs_comb(s, hs_unpack(A.mb[b0]));
    bk += A.MB;
  }
  for (; bk < b1; ++bk) s = hs_comb(s, A.pre(bk * 32 + 31));
  return hs_comb(s, A.pre(i1));
}

// min of l over [i0, i1] with its first arg-min (the a-prefix A_t of the window)
__device__ __forceinline__ void ht_minrange(const HTArr& A, int i0, int i1, int base, float& mv, int& mi) {
  const int b0 = i0 >> 5, b1 = i1 >> 5;
  if (b0 == b1) {
    mv = A.at(i0).x;
    mi = base + i0;
    for (int i = i0 + 1; i <= i1; ++i) {
      const float l = A.at(i).x;
      if (l < mv) {
        mv = l;
        mi = base + i;
      }
    }
    return;
  }
  const HS s = A.suf(i0);
  mv = s.m;
  mi = s.mi;
  for (int bk = b0 + 1; bk <= b1; ++bk) {
    const HS e = A.pre(bk < b1 ? bk * 32 + 31 : i1);
    if (e.m < mv) {
      mv = e.m;
      mi = e.mi;
    }
  }
}

// source of out[t] (t + b <= L - 1): position | HT_R for the right child
__device__ __forceinline__ int ht_source(const UParams& p, int base, int t, const HTArr& A) {
  const int it = t - base, iu = it + p.a, iv = it + p.b;
  const HS V = ht_range(A, iu, iv, base);
  if (p.a > 0) {
    float Av;
    int Ai;
    ht_minrange(A, it, iu - 1, base, Av, Ai);
    if (Av <= V.y) return Ai;  // out = A_t: the first arg-min of l over [t, u - 1]
  }
  return V.yi;
}

// 64-bit integer add into shared memory from two native 32-bit atomics (a 64-bit shared
// atomicAdd compiles to a CAS spin loop): the low word's carry-out is exact per add, so
// the pair holds the exact sum mod 2^64 for any order of arrival
__device__ __forceinline__ void ht_add64(unsigned long long* a, unsigned long long v) {
  unsigned* w = reinterpret_cast<unsigned*>(a);  // little endian: w[0] low, w[1] high
  const unsigned lo = (unsigned)v, hi = (unsigned)(v >> 32);
  const unsigned old = atomicAdd(w, lo);
  const unsigned carry = (old + lo < old) ? 1u : 0u;
  if (hi + carry != 0u) atomicAdd(w + 1, hi + carry);
}

__global__ void __launch_bounds__(HT_T, 5) k_until_ht_fwd(const __grid_constant__ UParams p) {
  extern __shared__ __align__(16) float htsm[];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  // balanced tiles (launch_until_ht_fwd): NT outputs, NS <= ht_ns(b) staged positions
  const int NT = p.ht_nt, NS = p.ht_ns;
  const int t0 = blockIdx.x * NT;
  const HTArr A = ht_carve(htsm, ht_ns(p.b), p.K);
  ht_prepare(p, row, t0, NS, A);
  float* outr = p.out + row * L;
  unsigned short* srcr = p.src != nullptr ? p.src + row * L : nullptr;
  const int tend = min(t0 + NT, L);
  for (int t = t0 + (int)threadIdx.x; t < tend; t += HT_T) {
    float o;
    if (t + p.b <= L - 1) {
      const int d = ht_source(p, t0, t, A);
      const float2 v = A.at((d & (HT_R - 1)) - t0);
      o = (d & HT_R) ? v.y : v.x;
      if (srcr) srcr[t] = (unsigned short)(((d & (HT_R - 1)) - t) | ((d & HT_R) ? 0x8000 : 0));
    } else {  // overrun: hard min of the pad values, a tie keeps the left (reference.py:189)
      if (srcr) srcr[t] = 0xffff;
      float pl = p.pad_value, pr = p.pad_value;
      if (p.pad_last) {
        pl = expr_eval<M_HARD>(p.left, row, L - 1, p.mp);
        pr = expr_eval<M_HARD>(p.right, row, L - 1, p.mp);
      }
      o = (pl <= pr) ? pl : pr;
    }
    outr[t] = p.canon ? __fadd_rn(o, 0.f) : o;
  }
}

__global__ void __launch_bounds__(HT_T, 4) k_until_ht_bwd(const __grid_constant__ UParams p) {
  extern __shared__ __align__(16) float htsm[];
  __shared__ float gred[HT_T / 32];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int NS = ht_ns(2 * p.b), NT = NS - 2 * p.b;
  const int t0 = blockIdx.x * NT;
  const int base = t0 - p.b;
  const HTArr A = ht_carve(htsm, NS, p.K);
  unsigned long long* accL = reinterpret_cast<unsigned long long*>(htsm + ht_words(NS));
  unsigned long long* accR = accL + NT;
  for (int i = threadIdx.x; i < NT; i += HT_T) accL[i] = accR[i] = 0ull;
  const float* cot = p.cot + row * L;
  const int tlo = max(base, 0), thi = min(t0 + NT, L);  // outputs that can reach the range
  // per-tile fixed-point scale: sum |g| over the tile's outputs < 2^62 / scale
  // (a NaN / inf cotangent makes gm inf: the ordered fallback below)
  const bool regs = NS <= 4 * HT_T;  // cotangents staged with the children, in registers
  float gk[4] = {0.f, 0.f, 0.f, 0.f};
  if (regs) {
    ht_prepare(p, row, base, NS, A, cot, NT + p.b, gk, gred);  // (its barriers publish gred / acc)
  } else {
    float gm = 0.f;
    for (int t = tlo + (int)threadIdx.x; t < thi; t += HT_T) {
      const float ag = fabsf(cot[t]);
      gm = (ag == ag) ? fmaxf(gm, ag) : INFINITY;
    }
    for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if ((threadIdx.x & 31) == 0) gred[threadIdx.x >> 5] = gm;
    ht_prepare(p, row, base, NS, A);
  }
  float gm = gred[0];
  for (int w = 1; w < HT_T / 32; ++w) gm = fmaxf(gm, gred[w]);
  int ge = 0;
  frexp((double)gm * (double)(thi - tlo + 1), &ge);  // sum |g| < 2^ge
  const double scale = ldexp(1.0, 62 - ge), inv = ldexp(1.0, ge - 62);
  int padsrc = -1;  // overrun outputs: source of min(pad_l, pad_r) ('last' padding only)
  if (p.pad_last) {
    const float pl = expr_eval<M_HARD>(p.left, row, L - 1, p.mp);
    const float pr = expr_eval<M_HARD>(p.right, row, L - 1, p.mp);
    padsrc = (pl <= pr) ? (L - 1) : ((L - 1) | HT_R);
  }
  if (gm > 0.f && gm < INFINITY) {
    auto route = [&](int t, float g) {
      if (g == 0.f) return;
      const int d = (t + p.b <= L - 1) ? ht_source(p, base, t, A) : padsrc;
      if (d < 0) return;
      const int j = (d & (HT_R - 1)) - t0;
      if (j < 0 || j >= NT) return;
      const long long q = llrint((double)g * scale);
      ht_add64((d & HT_R) ? &accR[j] : &accL[j], (unsigned long long)q);
    };
    if (regs) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = base + (int)threadIdx.x + k * HT_T;
        if (t >= tlo && t < thi) route(t, gk[k]);
      }
    } else {
      for (int t = tlo + (int)threadIdx.x; t < thi; t += HT_T) route(t, cot[t]);
    }
  }
  __syncthreads();
  float* gl = p.gl + row * L;
  float* gr = p.gr + row * L;
  const bool nonfinite = !(gm < INFINITY);  // inf / NaN cotangents: plain (ordered) sums
  for (int j = t0 + (int)threadIdx.x; j < min(t0 + NT, L); j += HT_T) {
    if (!nonfinite) {
      gl[j] = (float)((double)(long long)accL[j - t0] * inv);
      gr[j] = (float)((double)(long long)accR[j - t0] * inv);
    } else {  // sequential over the candidate outputs in t order (rare: non-finite g)
      float sl = 0.f, sr = 0.f;
      for (int t = max(j - p.b, 0); t <= j; ++t) {
        const float g = cot[t];
        if (g == 0.f) continue;
        const int d = (t + p.b <= L - 1) ? ht_source(p, base, t, A) : padsrc;
        if ((d & (HT_R - 1)) != j || d < 0) continue;
        if (d & HT_R) sr += g;
        else sl += g;
      }
      gl[j] = sl;
      gr[j] = sr;
    }
  }
}

// Backward from the forward's stored sources (p.src_in): the CTA owning child elements
// [t0, t0 + HS_NT) reads the cotangents and sources of the outputs [t0 - b, t0 + HS_NT) —
// 6 B per output, no child staging, no block walks — and sums them in shared int64 fixed
// point at a per-tile power-of-two scale (reproducible, as k_until_ht_bwd), then runs the
// children's VJPs on the owned elements (left first: first-writer order) — no gl / gr pass.
constexpr int HS_NT = 2048;
constexpr int HS_R = (HS_NT + HT_T) / HT_T;  // outputs per thread held in registers (b <= HT_T)
__global__ void __launch_bounds__(HT_T) k_until_ht_bwd_src(const __grid_constant__ UParams p) {
  __shared__ unsigned long long acc[2 * HS_NT];  // [left | right]
  __shared__ float gred[HT_T / 32];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int t0 = blockIdx.x * HS_NT;
  const int tlo = max(t0 - p.b, 0), thi = min(t0 + HS_NT, L);
  const float* cot = p.cot + row * L;
  const unsigned short* src = p.src_in + row * L;
  // the first HS_R HT_T outputs: one batch of loads into registers; the rest (b > HT_T) in a loop
  float gv[HS_R];
  unsigned short sv[HS_R];
#pragma unroll
  for (int k = 0; k < HS_R; ++k) {
    const int t = tlo + (int)threadIdx.x + k * HT_T;
    gv[k] = t < thi ? cot[t] : 0.f;
    sv[k] = t < thi ? src[t] : (unsigned short)0xffffu;
  }
  for (int i = threadIdx.x; i < 2 * HS_NT; i += HT_T) acc[i] = 0ull;
  float gm = 0.f;
#pragma unroll
  for (int k = 0; k < HS_R; ++k) {
    const float ag = fabsf(gv[k]);
    gm = (ag == ag) ? fmaxf(gm, ag) : INFINITY;
  }
  for (int t = tlo + (int)threadIdx.x + HS_R * HT_T; t < thi; t += HT_T) {
    const float ag = fabsf(cot[t]);
    gm = (ag == ag) ? fmaxf(gm, ag) : INFINITY;
  }
  for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
  if ((threadIdx.x & 31) == 0) gred[threadIdx.x >> 5] = gm;
  __syncthreads();
  gm = gred[0];
  for (int w = 1; w < HT_T / 32; ++w) gm = fmaxf(gm, gred[w]);
  int ge = 0;
  frexp((double)gm * (double)(thi - tlo + 1), &ge);  // sum |g| < 2^ge
  const double scale = ldexp(1.0, 62 - ge), inv = ldexp(1.0, ge - 62);
  int padsrc = -1;  // overrun outputs: source of min(pad_l, pad_r) ('last' padding only)
  if (p.pad_last && thi - 1 + p.b > L - 1) {
    const float pl = expr_eval<M_HARD>(p.left, row, L - 1, p.mp);
    const float pr = expr_eval<M_HARD>(p.right, row, L - 1, p.mp);
    padsrc = (pl <= pr) ? (L - 1) : ((L - 1) | HT_R);
  }
  auto source_of = [&](int t, unsigned s) {
    return s == 0xffffu ? padsrc : (int)(t + (s & 0x7fffu)) | ((s & 0x8000u) ? HT_R : 0);
  };
  auto source = [&](int t) { return source_of(t, src[t]); };
  auto route = [&](int t, float g, int d) {
    if (g == 0.f || d < 0) return;
    const int j = (d & (HT_R - 1)) - t0;
    if (j < 0 || j >= HS_NT) return;
    ht_add64(&acc[((d & HT_R) ? HS_NT : 0) + j], (unsigned long long)llrint((double)g * scale));
  };
  const bool nonfinite = !(gm < INFINITY);  // inf / NaN cotangents: plain (ordered) sums
  if (gm > 0.f && !nonfinite) {
#pragma unroll
    for (int k = 0; k < HS_R; ++k) {
      const int t = tlo + (int)threadIdx.x + k * HT_T;
      if (t < thi) route(t, gv[k], source_of(t, sv[k]));
    }
    for (int t = tlo + (int)threadIdx.x + HS_R * HT_T; t < thi; t += HT_T) route(t, cot[t], source(t));
  }
  __syncthreads();
  const ChildEval cl(p.left, row), cr(p.right, row);
  for (int j = t0 + (int)threadIdx.x; j < thi; j += HT_T) {
    if (!nonfinite) {
      cl.grad<M_HARD>(j, (float)((double)(long long)acc[j - t0] * inv), p.mp);
      cr.grad<M_HARD>(j, (float)((double)(long long)acc[HS_NT + j - t0] * inv), p.mp);
    } else {  // sequential over the candidate outputs in t order (rare: non-finite g)
      float sl = 0.f, sr = 0.f;
      for (int t = max(j - p.b, 0); t <= j; ++t) {
        const float g = cot[t];
        if (g == 0.f) continue;
        const int d = source(t);
        if (d < 0 || (d & (HT_R - 1)) != j) continue;
        if (d & HT_R) sr += g;
        else sl += g;
      }
      cl.grad<M_HARD>(j, sl, p.mp);
      cr.grad<M_HARD>(j, sr, p.mp);
    }
  }
}

// true when the O(T) kernels apply (hard, timed, no masked_fill, staging fits)
bool until_ht_applicable(const UParams& p) {
  if (p.untimed || p.fill || p.K < 1 || p.L >= (1LL << 29)) return false;
  const int NS = ht_ns(2 * p.b);
  return ht_smem_bytes(NS) + (size_t)(NS - 2 * p.b) * 16 <= 200 * 1024;
}

cudaError_t launch_until_ht_fwd(UParams& p, cudaStream_t st) {
  // balanced tiles: the row's ceil(L / NTmax) tiles share its outputs evenly and each stages
  // only its outputs + the b-halo (T = 1000 was one full tile plus a 76-output one)
  const int NS = ht_ns(p.b), NTM = NS - p.b;
  const long long ntl = (p.L + NTM - 1) / NTM;
  p.ht_nt = (int)((p.L + ntl - 1) / ntl);
  p.ht_ns = std::min(NS, (p.ht_nt + p.b + 31) & ~31);
  const size_t smem = ht_smem_bytes(NS);
  cudaError_t e = cudaFuncSetAttribute(k_until_ht_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)ntl, (unsigned)p.B);
  k_until_ht_fwd<<<grid, HT_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// with p.src_in: runs the child VJPs itself; else writes every element of p.gl / p.gr
// (the caller runs the child VJPs)
cudaError_t launch_until_ht_bwd(UParams& p, cudaStream_t st) {
  if (p.src_in != nullptr) {  // the forward stored every output's source
    dim3 grid((unsigned)((p.L + HS_NT - 1) / HS_NT), (unsigned)p.B);
    k_until_ht_bwd_src<<<grid, HT_T, 0, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  const int NS = ht_ns(2 * p.b), NT = NS - 2 * p.b;
  const size_t smem = ht_smem_bytes(NS) + (size_t)NT * 16;
  cudaError_t e = cudaFuncSetAttribute(k_until_ht_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + NT - 1) / NT), (unsigned)p.B);
  k_until_ht_bwd<<<grid, HT_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
