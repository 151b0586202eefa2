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

struct HTArr {
  float *l, *r, *X, *Sm, *Y, *SA, *PA;
  int *dX, *SI, *dY, *SAI, *PAI;
};

__device__ __forceinline__ HTArr ht_carve(float* base, int NS, bool has_a) {
  HTArr A;
  A.l = base;
  A.r = A.l + NS;
  A.X = A.r + NS;
  A.Sm = A.X + NS;
  A.Y = A.Sm + NS;
  int* ib = reinterpret_cast<int*>(A.Y + NS);
  A.dX = ib;
  A.SI = A.dX + NS;
  A.dY = A.SI + NS;
  float* fb = reinterpret_cast<float*>(A.dY + NS);
  A.SA = has_a ? fb : nullptr;
  A.PA = has_a ? fb + NS : nullptr;
  int* jb = reinterpret_cast<int*>(fb + 2 * NS);
  A.SAI = has_a ? jb : nullptr;
  A.PAI = has_a ? jb + NS : nullptr;
  return A;
}

size_t ht_smem_bytes(int NS, bool has_a) { return (size_t)NS * 4 * (has_a ? 12 : 8); }

// stage the children over [base, base + NS) and run every block walk
__device__ void ht_prepare(const UParams& p, long long row, int base, int NS, const HTArr& A) {
  const int L = (int)p.L, K = p.K, a = p.a;
  const int hi = min(base + NS, L);  // staged positions [lo, hi)
  const int lo = max(base, 0);
  for (int i = threadIdx.x; i < NS; i += blockDim.x) {
    const int pos = base + i;
    if (pos >= lo && pos < hi) {
      A.l[i] = expr_eval<M_HARD>(p.left, row, pos, p.mp);
      A.r[i] = expr_eval<M_HARD>(p.right, row, pos, p.mp);
    }
  }
  __syncthreads();
  if (lo >= hi) return;
  // K blocks: backward X / Smin, forward Y
  const int kb0 = lo / K, kb1 = (hi - 1) / K;
  for (int kb = kb0 + (int)threadIdx.x; kb <= kb1; kb += blockDim.x) {
    const int bs = max(kb * K, lo), be = min(kb * K + K - 1, hi - 1);
    {  // backward walk
      int i = be - base;
      float Ll = A.l[i], Rr = A.r[i];
      bool cR = Rr < Ll;
      float X = cR ? Rr : Ll, Sm = Ll;
      int dX = cR ? (be | HT_R) : be, SI = be;
      A.X[i] = X;
      A.dX[i] = dX;
      A.Sm[i] = Sm;
      A.SI[i] = SI;
      for (int pos = be - 1; pos >= bs; --pos) {
        i = pos - base;
        Ll = A.l[i];
        Rr = A.r[i];
        cR = Rr < Ll;
        const float c = cR ? Rr : Ll;
        const float m2 = (Ll <= X) ? Ll : X;
        if (c >= m2) {  // s = u is the first maximiser
          X = c;
          dX = cR ? (pos | HT_R) : pos;
        } else if (!(X < Ll)) {  // clamped at l_u: theta = l_u, source l_u
          X = Ll;
          dX = pos;
        }  // else X(u) = X(u + 1) with its source
        if (Ll <= Sm) {  // first arg-min: a tie moves to the earlier position
          Sm = Ll;
          SI = pos;
        }
        A.X[i] = X;
        A.dX[i] = dX;
        A.Sm[i] = Sm;
        A.SI[i] = SI;
      }
    }
    {  // forward walk
      int i = bs - base;
      float Ll = A.l[i], Rr = A.r[i];
      float M = Ll;
      int MI = bs;
      bool cR = Rr < M;
      float Y = cR ? Rr : M;
      int dY = cR ? (bs | HT_R) : MI;
      A.Y[i] = Y;
      A.dY[i] = dY;
      for (int pos = bs + 1; pos <= be; ++pos) {
        i = pos - base;
        Ll = A.l[i];
        Rr = A.r[i];
        if (Ll < M) {  // running min keeps the earlier element on ties
          M = Ll;
          MI = pos;
        }
        cR = Rr < M;  // term tie keeps pm
        const float cand = cR ? Rr : M;
        if (!(Y >= cand)) {  // earlier maximiser wins ties
          Y = cand;
          dY = cR ? (pos | HT_R) : MI;
        }
        A.Y[i] = Y;
        A.dY[i] = dY;
      }
    }
  }
  if (a > 0) {  // a blocks: window min of l over [t, t + a - 1]
    const int ab0 = lo / a, ab1 = (hi - 1) / a;
    for (int ab = ab0 + (int)threadIdx.x; ab <= ab1; ab += blockDim.x) {
      const int bs = max(ab * a, lo), be = min(ab * a + a - 1, hi - 1);
      float S = INFINITY;
      int SIx = be;
      for (int pos = be; pos >= bs; --pos) {
        const float Ll = A.l[pos - base];
        if (Ll <= S) {
          S = Ll;
          SIx = pos;
        }
        A.SA[pos - base] = S;
        A.SAI[pos - base] = SIx;
      }
      float Pm = INFINITY;
      int PI = bs;
      for (int pos = bs; pos <= be; ++pos) {
        const float Ll = A.l[pos - base];
        if (Ll < Pm) {
          Pm = Ll;
          PI = pos;
        }
        A.PA[pos - base] = Pm;
        A.PAI[pos - base] = PI;
      }
    }
  }
  __syncthreads();
}

// source of out[t] (t + b <= L - 1): position | HT_R for the right child
__device__ __forceinline__ int ht_source(const UParams& p, int base, int t, const HTArr& A) {
  const int K = p.K, a = p.a;
  const int u = t + a, v = t + p.b;
  const int iu = u - base;
  float V = A.X[iu];
  int d = A.dX[iu];
  if (u % K != 0) {  // the window spills into the next block
    const float Smv = A.Sm[iu], Yv = A.Y[v - base];
    const bool sm = Smv <= Yv;
    const float z = sm ? Smv : Yv;
    if (!(V >= z)) {
      V = z;
      d = sm ? A.SI[iu] : A.dY[v - base];
    }
  }
  if (a > 0) {
    const int it = t - base;
    float Av = A.SA[it];
    int Ai = A.SAI[it];
    if (t % a != 0) {
      const float Pv = A.PA[it + a - 1];
      if (Pv < Av) {
        Av = Pv;
        Ai = A.PAI[it + a - 1];
      }
    }
    if (Av <= V) d = Ai;  // out = A_t: the first arg-min of l over [t, u - 1]
  }
  return d;
}

__global__ void __launch_bounds__(HT_T) k_until_ht_fwd(const __grid_constant__ UParams p) {
  extern __shared__ float htsm[];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int t0 = blockIdx.x * HT_NT;
  const int NS = HT_NT + p.b;
  const HTArr A = ht_carve(htsm, NS, p.a > 0);
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
  const HTArr A = ht_carve(htsm, NS, p.a > 0);
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
  return ht_smem_bytes(HT_NT + 2 * p.b, p.a > 0) <= 200 * 1024;
}

cudaError_t launch_until_ht_fwd(UParams& p, cudaStream_t st) {
  const size_t smem = ht_smem_bytes(HT_NT + p.b, p.a > 0);
  cudaError_t e = cudaFuncSetAttribute(k_until_ht_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + HT_NT - 1) / HT_NT), (unsigned)p.B);
  k_until_ht_fwd<<<grid, HT_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// writes every element of p.gl / p.gr (the caller runs the child VJPs)
cudaError_t launch_until_ht_bwd(UParams& p, cudaStream_t st) {
  const size_t smem = ht_smem_bytes(HT_NT + 2 * p.b, p.a > 0);
  cudaError_t e = cudaFuncSetAttribute(k_until_ht_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((p.L + HT_NT - 1) / HT_NT), (unsigned)p.B);
  k_until_ht_bwd<<<grid, HT_T, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
