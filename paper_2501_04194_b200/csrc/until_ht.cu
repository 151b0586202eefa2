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
#include "kernels.cuh"

namespace stlg {

constexpr int HT_T = 128;    // threads per CTA
constexpr int HT_NT = 1024;  // outputs (forward) / owned elements (backward) per CTA
constexpr int HT_R = 1 << 30;  // source flag: right child

// Range state of the reference's Until over a range R = [s0, s1] of candidate ends s:
//   m  = min l over R, mi its first arg-min,
//   y  = max_{s in R} min(min l[s0 .. s], r_s), yi the gradient source of y.
// Combining adjacent ranges A (earlier) and B (later):
//   m = min(m_A, m_B) (a tie keeps A), y = max(y_A, min(m_A, y_B)) with the source
//   yi_A if y_A >= min(m_A, y_B), else yi_B if y_B < m_A, else l[mi_A]
// — the reference's tie rules, so the state of a range is unique and the combine is
// associative (warp scans may use any bracketing).
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
__device__ __forceinline__ HS hs_shfl_up(const HS& v, int o) {
  return HS{__shfl_up_sync(0xffffffffu, v.m, o), __shfl_up_sync(0xffffffffu, v.y, o),
            __shfl_up_sync(0xffffffffu, v.mi, o), __shfl_up_sync(0xffffffffu, v.yi, o)};
}
__device__ __forceinline__ HS hs_shfl_down(const HS& v, int o) {
  return HS{__shfl_down_sync(0xffffffffu, v.m, o), __shfl_down_sync(0xffffffffu, v.y, o),
            __shfl_down_sync(0xffffffffu, v.mi, o), __shfl_down_sync(0xffffffffu, v.yi, o)};
}

// staged arrays: children, and per position the suffix state over [i, end of its
// 32-block] and the prefix state over [start of its block, i] (struct-of-arrays)
struct HTArr {
  float *l, *r;
  float *sm, *sy, *pm, *py;
  int *smi, *syi, *pmi, *pyi;
  __device__ __forceinline__ HS suf(int i) const { return HS{sm[i], sy[i], smi[i], syi[i]}; }
  __device__ __forceinline__ HS pre(int i) const { return HS{pm[i], py[i], pmi[i], pyi[i]}; }
};

__device__ __forceinline__ HTArr ht_carve(float* base, int NS) {
  HTArr A;
  float* f = base;
  A.l = f;
  A.r = f + NS;
  A.sm = f + 2 * NS;
  A.sy = f + 3 * NS;
  A.pm = f + 4 * NS;
  A.py = f + 5 * NS;
  int* q = reinterpret_cast<int*>(f + 6 * NS);
  A.smi = q;
  A.syi = q + NS;
  A.pmi = q + 2 * NS;
  A.pyi = q + 3 * NS;
  return A;
}

size_t ht_smem_bytes(int NS) { return (size_t)NS * 4 * 10; }

// stage the children over [base, base + NS) and scan every 32-block (one warp per block,
// prefix and suffix states by shuffles)
__device__ void ht_prepare(const UParams& p, long long row, int base, int NS, const HTArr& A) {
  const int L = (int)p.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (NS + 31) >> 5;
  const ChildEval cl(p.left, row), cr(p.right, row);
  for (int bk = warp; bk < nb; bk += HT_T / 32) {
    const int i = bk * 32 + lane, pos = base + i;
    const bool live = i < NS && pos >= 0 && pos < L;
    float l = 0.f, r = 0.f;
    if (cl.kind != 0 && cr.kind != 0) {  // loads issued before the transforms
      const int pc = live ? pos : 0;
      const float xl = cl.raw(pc), xr = cr.raw(pc);
      if (live) {
        l = cl.apply(xl);
        r = cr.apply(xr);
      }
    } else if (live) {
      l = cl.value<M_HARD>(pos, p.mp);
      r = cr.value<M_HARD>(pos, p.mp);
    }
    const HS e = hs_elem(l, r, pos);
    HS pre = e, suf = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const HS a = hs_shfl_up(pre, o);
      const HS b = hs_shfl_down(suf, o);
      if (lane >= o) pre = hs_comb(a, pre);
      if (lane + o < 32) suf = hs_comb(suf, b);
    }
    if (i < NS) {
      A.l[i] = l;
      A.r[i] = r;
      A.pm[i] = pre.m;
      A.py[i] = pre.y;
      A.pmi[i] = pre.mi;
      A.pyi[i] = pre.yi;
      A.sm[i] = suf.m;
      A.sy[i] = suf.y;
      A.smi[i] = suf.mi;
      A.syi[i] = suf.yi;
    }
  }
  __syncthreads();
}

// state of the staged range [i0, i1] (inclusive, relative indices)
__device__ __forceinline__ HS ht_range(const HTArr& A, int i0, int i1, int base) {
  const int b0 = i0 >> 5, b1 = i1 >> 5;
  if (b0 == b1) {  // inside one block: element by element (at most 32 steps)
    HS s = hs_elem(A.l[i0], A.r[i0], base + i0);
    for (int i = i0 + 1; i <= i1; ++i) s = hs_comb(s, hs_elem(A.l[i], A.r[i], base + i));
    return s;
  }
  HS s = A.suf(i0);
  for (int bk = b0 + 1; bk < b1; ++bk) s = hs_comb(s, A.pre(bk * 32 + 31));
  return hs_comb(s, A.pre(i1));
}

// min of l over [i0, i1] with its first arg-min (the a-prefix A_t of the window)
__device__ __forceinline__ void ht_minrange(const HTArr& A, int i0, int i1, int base, float& mv, int& mi) {
  const int b0 = i0 >> 5, b1 = i1 >> 5;
  if (b0 == b1) {
    mv = A.l[i0];
    mi = base + i0;
    for (int i = i0 + 1; i <= i1; ++i)
      if (A.l[i] < mv) {
        mv = A.l[i];
        mi = base + i;
      }
    return;
  }
  mv = A.sm[i0];
  mi = A.smi[i0];
  for (int bk = b0 + 1; bk <= b1; ++bk) {
    const int e = bk < b1 ? bk * 32 + 31 : i1;
    if (A.pm[e] < mv) {
      mv = A.pm[e];
      mi = A.pmi[e];
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

__global__ void __launch_bounds__(HT_T) k_until_ht_fwd(const __grid_constant__ UParams p) {
  extern __shared__ float htsm[];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int t0 = blockIdx.x * HT_NT;
  const int NS = HT_NT + p.b;
  const HTArr A = ht_carve(htsm, NS);
  ht_prepare(p, row, t0, NS, A);
  float* outr = p.out + row * L;
  const int tend = min(t0 + HT_NT, L);
  for (int t = t0 + (int)threadIdx.x; t < tend; t += HT_T) {
    float o;
    if (t + p.b <= L - 1) {
      const int d = ht_source(p, t0, t, A);
      o = (d & HT_R) ? A.r[(d & (HT_R - 1)) - t0] : A.l[d - t0];
    } else {  // overrun: hard min of the pad values, a tie keeps the left (reference.py:189)
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

__global__ void __launch_bounds__(HT_T) k_until_ht_bwd(const __grid_constant__ UParams p) {
  extern __shared__ float htsm[];
  __shared__ unsigned long long accL[HT_NT], accR[HT_NT];
  __shared__ float gred[HT_T / 32];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int t0 = blockIdx.x * HT_NT;
  const int base = t0 - p.b;
  const int NS = HT_NT + 2 * p.b;
  const HTArr A = ht_carve(htsm, NS);
  for (int i = threadIdx.x; i < HT_NT; i += HT_T) accL[i] = accR[i] = 0ull;
  const float* cot = p.cot + row * L;
  const int tlo = max(base, 0), thi = min(t0 + HT_NT, L);  // outputs that can reach the range
  // per-tile fixed-point scale: sum |g| over the tile's outputs < 2^62 / scale
  float gm = 0.f;  // (a NaN / inf cotangent makes gm inf: the ordered fallback below)
  for (int t = tlo + (int)threadIdx.x; t < thi; t += HT_T) {
    const float ag = fabsf(cot[t]);
    gm = (ag == ag) ? fmaxf(gm, ag) : INFINITY;
  }
  for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
  if ((threadIdx.x & 31) == 0) gred[threadIdx.x >> 5] = gm;
  ht_prepare(p, row, base, NS, A);  // (contains the barriers that publish gred / acc)
  gm = gred[0];
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
    for (int t = tlo + (int)threadIdx.x; t < thi; t += HT_T) {
      const float g = cot[t];
      if (g == 0.f) continue;
      const int d = (t + p.b <= L - 1) ? ht_source(p, base, t, A) : padsrc;
      if (d < 0) continue;
      const int j = (d & (HT_R - 1)) - t0;
      if (j < 0 || j >= HT_NT) continue;
      const long long q = llrint((double)g * scale);
      atomicAdd((d & HT_R) ? &accR[j] : &accL[j], (unsigned long long)q);
    }
  }
  __syncthreads();
  float* gl = p.gl + row * L;
  float* gr = p.gr + row * L;
  const bool nonfinite = !(gm < INFINITY);  // inf / NaN cotangents: plain (ordered) sums
  for (int j = t0 + (int)threadIdx.x; j < min(t0 + HT_NT, L); j += HT_T) {
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

// true when the O(T) kernels apply (hard, timed, no masked_fill, staging fits)
bool until_ht_applicable(const UParams& p) {
  if (p.untimed || p.fill || p.K < 1 || p.L >= (1LL << 29)) return false;
  return ht_smem_bytes(HT_NT + 2 * p.b) <= 200 * 1024;
}

cudaError_t launch_until_ht_fwd(UParams& p, cudaStream_t st) {
  const size_t smem = ht_smem_bytes(HT_NT + p.b);
  cudaError_t e = cudaFuncSetAttribute(k_until_ht_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + HT_NT - 1) / HT_NT), (unsigned)p.B);
  k_until_ht_fwd<<<grid, HT_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// writes every element of p.gl / p.gr (the caller runs the child VJPs)
cudaError_t launch_until_ht_bwd(UParams& p, cudaStream_t st) {
  const size_t smem = ht_smem_bytes(HT_NT + 2 * p.b);
  cudaError_t e = cudaFuncSetAttribute(k_until_ht_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + HT_NT - 1) / HT_NT), (unsigned)p.B);
  k_until_ht_bwd<<<grid, HT_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
