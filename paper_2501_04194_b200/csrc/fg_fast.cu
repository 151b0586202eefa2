// fg_fast.cu — timed Eventually / Always, LSE mode: exp-factorised window sums
// with block-wide segmented parallel scans.
//
// For a tile whose samples span a dynamic range the fp32 exponent can carry
// (tau2 * (max - min) <= 100), every window's log-sum-exp shares one shift c
// (the tile max):  out_t = c + log2(sum_{window} E_i) / tau2,  E_i = 2^{tau2 (u_i - c)},
// all E_i normal floats, so the vHGW pieces are plain sums of positive terms.
// The block prefix / suffix sums are computed by ALL threads with segmented
// (reset at each K-block boundary) warp-shuffle scans — no per-block sequential
// chains, no scanner / mover split, 2 shared words per sample.
//
// Backward (gather form): element j receives sum_t g_t 2^{tau2 (u_j - M_t)} over
// t in [j - b, j - a]; with c = min M_t over the tile's live outputs this is
// 2^{tau2 (u_j - c)} * windowsum(h),  h_t = g_t 2^{tau2 (c - M_t)}  (same scans,
// mixed-sign sums), followed by the fused child VJP.
//
// A tile outside the range condition raises a device flag; the exact
// (max-shifted monoid) kernel then re-runs the whole operator, guarded by that
// flag, so correctness never depends on the data and no host sync is needed.
#include "kernels.cuh"

namespace stlg {

constexpr int FF_T = 256;               // threads
constexpr int FF_EPT = 16;              // samples per thread in the scans
constexpr int FF_N = FF_T * FF_EPT;     // samples staged per tile
__device__ __forceinline__ int ffpad(int i) { return i + (i >> 4); }  // 1 word pad per 16
constexpr int FF_NP = FF_N + FF_N / 16;

// ---------------------------------------------------------------------------
// block-wide segmented inclusive scans over FF_N samples in shared memory.
//   prefix: P[i] = sum of v over [start of i's K-block, i]
//   suffix: S[i] = sum of v over [i, end of i's K-block]
// v is read from `src` (padded layout), results written to `dst` (may alias src).
// Thread t owns positions [EPT t, EPT t + EPT) (reversed ownership for the
// suffix scan so lane order is processing order); r0 = (EPT * owner) % K.
// ---------------------------------------------------------------------------
struct SegCarry {
  float s;
  int r;  // a reset happened inside
};
__device__ __forceinline__ SegCarry seg_op(SegCarry a, SegCarry b) {  // a before b
  return SegCarry{b.r ? b.s : a.s + b.s, a.r | b.r};
}

template <bool SUFFIX>
__device__ __forceinline__ void seg_scan(const float* src, float* dst, int K, int r_first,
                                         float* red_s, int* red_r) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int owner = SUFFIX ? (FF_T - 1 - tid) : tid;
  const int base = owner * FF_EPT;
  float v[FF_EPT];
#pragma unroll
  for (int k = 0; k < FF_EPT; ++k) v[k] = src[ffpad(base + k)];
  // reset mask: bit k set where position base + k starts (prefix) / ends (suffix) a block
  unsigned mask = 0;
  {
    int r = r_first;  // offset of `base` in its block
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      if (SUFFIX ? (r == K - 1) : (r == 0)) mask |= 1u << k;
      r = (r + 1 == K) ? 0 : r + 1;
    }
  }
  float run = 0.f;
  if (!SUFFIX) {
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      run = ((mask >> k) & 1u) ? v[k] : run + v[k];
      v[k] = run;
    }
  } else {
#pragma unroll
    for (int k = FF_EPT - 1; k >= 0; --k) {
      run = ((mask >> k) & 1u) ? v[k] : run + v[k];
      v[k] = run;
    }
  }
  SegCarry inc{run, mask != 0u};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float s = __shfl_up_sync(0xffffffffu, inc.s, o);
    int rr = __shfl_up_sync(0xffffffffu, inc.r, o);
    if (lane >= o) inc = seg_op(SegCarry{s, rr}, inc);
  }
  float ex_s = __shfl_up_sync(0xffffffffu, inc.s, 1);
  int ex_r = __shfl_up_sync(0xffffffffu, inc.r, 1);
  SegCarry lane_ex = lane ? SegCarry{ex_s, ex_r} : SegCarry{0.f, 0};
  if (lane == 31) {
    red_s[warp] = inc.s;
    red_r[warp] = inc.r;
  }
  __syncthreads();
  SegCarry wc{0.f, 0};
  for (int w = 0; w < warp; ++w) wc = seg_op(wc, SegCarry{red_s[w], red_r[w]});
  const float carry = seg_op(wc, lane_ex).s;
  // the carry reaches the owned samples before the first reset (in processing order)
  if (!SUFFIX) {
    bool open = true;
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      open = open && !((mask >> k) & 1u);
      dst[ffpad(base + k)] = open ? v[k] + carry : v[k];
    }
  } else {
    bool open = true;
#pragma unroll
    for (int k = FF_EPT - 1; k >= 0; --k) {
      open = open && !((mask >> k) & 1u);
      dst[ffpad(base + k)] = open ? v[k] + carry : v[k];
    }
  }
  __syncthreads();
}

// block min / max
__device__ __forceinline__ void block_or(int& v, int* red) {
  v = __any_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int o = 0;
  for (int w = 0; w < FF_T / 32; ++w) o |= red[w];
  v = o;
}

// exponent budget (log2 units) of the fast path: per sample |u - c_block| and
// between neighbouring block shifts; all terms stay within 2^{+-70} (normal fp32,
// sums of up to 2^20 terms cannot overflow)
constexpr float FF_SAMPLE_RANGE = 60.f;  // E in [2^-60, 2^60]
constexpr float FF_SHIFT_STEP = 50.f;    // neighbour terms stay >= 2^-110 and sums < 2^127

// incremental (q, r) = divmod(i, K) for i = tid + k * FF_T, k = 0, 1, ...
struct DivMod {
  int q, r, dq, dr, K;
  __device__ __forceinline__ DivMod(int i, int K_) : K(K_) {
    q = i / K_;
    r = i - q * K_;
    dq = FF_T / K_;
    dr = FF_T - dq * K_;
  }
  __device__ __forceinline__ void next() {
    q += dq;
    r += dr;
    if (r >= K) {
      r -= K;
      q += 1;
    }
  }
};

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <int EK>
__global__ void __launch_bounds__(FF_T, 4) k_lse_fast_fwd(const __grid_constant__ FGParams p, int* slow) {
  __shared__ float A[FF_NP];   // u -> E -> within-block suffix sums
  __shared__ float Pp[FF_NP];  // within-block prefix sums
  __shared__ float C[FF_N / 2 + 2];  // block shifts c_q = u at the block start
  __shared__ float red_f[FF_T / 32];
  __shared__ int red_i[FF_T / 32];
  const int K = p.K;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = FF_N - K + 1;  // outputs per tile
  const int t0 = blockIdx.x * J;
  const int nvalid = L - p.b;
  const int s0 = t0 + p.a;
  const float tau2 = p.mp.tau2, itau2 = p.mp.inv_tau2, sg = p.sg;
  Ev<M_LSE, EK> ev(p.child, row, p.mp);
  const float padv = p.pad_last ? ev.value(L - 1, ev.load(L - 1)) : p.pad_value;
  float* outr = p.out + row * L;
  const int tend = (t0 + J < L ? t0 + J : L) - t0;
  if (t0 >= nvalid) {  // whole tile overruns: pad values (uniform)
    if (threadIdx.x == 0) p.tile_slow[row * gridDim.x + blockIdx.x] = 0;
    for (int i = threadIdx.x; i < tend; i += FF_T) {
      float v = padv;
      if (p.canon) v = __fadd_rn(v, 0.f);
      outr[t0 + i] = v;
    }
    return;
  }
  const int nlast = L - 1 - s0;  // last local index holding a real sample
  // load u (coalesced, FF_EPT independent loads in flight per thread)
  {
    const bool interior = s0 + FF_N <= L;
    DivMod dm(threadIdx.x, K);
#pragma unroll
    for (int h = 0; h < FF_EPT; h += 8) {  // two batches of 8 loads in flight (register budget)
      typename Ev<M_LSE, EK>::Raw r[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        int idx = s0 + threadIdx.x + (h + k) * FF_T;
        if (interior || idx < L) r[k] = ev.load(idx);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        int i = threadIdx.x + (h + k) * FF_T;
        float u = (interior || s0 + i < L) ? sg * ev.value(s0 + i, r[k]) : 0.f;
        A[ffpad(i)] = u;
        if (dm.r == 0) C[dm.q] = u;
        dm.next();
      }
    }
  }
  __syncthreads();
  // E_i = 2^{tau2 (u_i - c_q)} (0 past the end); range checks
  {
    float e[FF_EPT];
    int bad = 0;
    DivMod dm(threadIdx.x, K);
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      int i = threadIdx.x + k * FF_T;
      float d = tau2 * (A[ffpad(i)] - C[dm.q]);
      bad |= fabsf(d) > FF_SAMPLE_RANGE && i <= nlast;
      e[k] = (i <= nlast) ? ex2f(d) : 0.f;
      if (dm.r == 0 && dm.q > 0 && i <= nlast)
        bad |= fabsf(tau2 * (C[dm.q] - C[dm.q - 1])) > FF_SHIFT_STEP;
      dm.next();
    }
    block_or(bad, red_i);
    if (threadIdx.x == 0) p.tile_slow[row * gridDim.x + blockIdx.x] = bad;
    if (bad) {  // out of the fast range: the exact kernel recomputes this tile
      if (threadIdx.x == 0) atomicOr(slow, 1);
      return;
    }
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) A[ffpad(threadIdx.x + k * FF_T)] = e[k];
  }
  __syncthreads();
  seg_scan<false>(A, Pp, K, (threadIdx.x * FF_EPT) % K, red_f, red_i);
  seg_scan<true>(A, A, K, ((FF_T - 1 - threadIdx.x) * FF_EPT) % K, red_f, red_i);
  // window [s, s + K - 1] = suffix(s) (+ prefix(s + K - 1) of the next block)
  DivMod dm(threadIdx.x, K);
  for (int i = threadIdx.x; i < tend; i += FF_T, dm.next()) {
    const int t = t0 + i;
    float v;
    if (t < nvalid) {
      const float cq = C[dm.q];
      float sum = A[ffpad(i)];
      if (dm.r != 0) sum = fmaf(Pp[ffpad(i + K - 1)], ex2f(tau2 * (C[dm.q + 1] - cq)), sum);
      v = sg * fmaf(lg2f(sum), itau2, cq);
    } else {
      v = padv;
    }
    if (p.canon) v = __fadd_rn(v, 0.f);
    outr[t] = v;
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
template <int EK>
__global__ void __launch_bounds__(FF_T, 4) k_lse_fast_bwd(const __grid_constant__ FGParams p, int* slow) {
  __shared__ float A[FF_NP];
  __shared__ float Pp[FF_NP];
  __shared__ float C[FF_N / 2 + 2];
  __shared__ float red_f[FF_T / 32];
  __shared__ int red_i[FF_T / 32];
  __shared__ float padsum_sh;
  const int K = p.K;
  const int L = (int)p.L;
  const long long row = blockIdx.y;
  const int J = FF_N - K + 1;  // owned child elements per tile
  const int j0 = blockIdx.x * J;
  const int tb = j0 - p.b;      // local h index 0 <-> output t = tb
  const int nvalid = L - p.b;
  const float tau2 = p.mp.tau2, sg = p.sg;
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  float gv[FF_EPT];
  // stage M_t (clamped to the nearest live output so block shifts are always real
  // values) and g_t for t in [tb, tb + FF_N)
  {
    float mv[FF_EPT];
    const int tlo = 0, thi = (nvalid > 0 ? nvalid : 1) - 1;
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      int t = tb + threadIdx.x + k * FF_T;
      bool v = t >= 0 && t < nvalid;
      int tc = t < tlo ? tlo : (t > thi ? thi : t);
      gv[k] = v ? ld_na(cot + t) : 0.f;
      mv[k] = nvalid > 0 ? ld_na(outr + tc) : 0.f;
    }
    DivMod dm(threadIdx.x, K);
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      float M = sg * mv[k];
      Pp[ffpad(threadIdx.x + k * FF_T)] = M;
      if (dm.r == 0) C[dm.q] = M;
      dm.next();
    }
  }
  if (threadIdx.x < 32) {  // overrun outputs route to c[L-1] ('last' padding)
    float ps = 0.f;
    if (p.pad_last && L - 1 >= j0 && L - 1 < j0 + J) {
      int t_lo = nvalid > 0 ? nvalid : 0;
      for (int t = t_lo + (int)threadIdx.x; t < L; t += 32) ps += cot[t];
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    }
    if (threadIdx.x == 0) padsum_sh = ps;
  }
  __syncthreads();
  {
    int bad = 0;
    DivMod dm(threadIdx.x, K);
#pragma unroll
    for (int k = 0; k < FF_EPT; ++k) {
      int i = threadIdx.x + k * FF_T;
      float d = tau2 * (C[dm.q] - Pp[ffpad(i)]);
      bad |= fabsf(d) > FF_SAMPLE_RANGE;
      A[ffpad(i)] = gv[k] != 0.f ? gv[k] * ex2f(d) : 0.f;
      if (dm.r == 0 && dm.q > 0) bad |= fabsf(tau2 * (C[dm.q] - C[dm.q - 1])) > FF_SHIFT_STEP;
      dm.next();
    }
    block_or(bad, red_i);
    if (threadIdx.x == 0) p.tile_slow[row * gridDim.x + blockIdx.x] = bad;
    if (bad) {
      if (threadIdx.x == 0) atomicOr(slow, 1);
      return;
    }
  }
  seg_scan<false>(A, Pp, K, (threadIdx.x * FF_EPT) % K, red_f, red_i);
  seg_scan<true>(A, A, K, ((FF_T - 1 - threadIdx.x) * FF_EPT) % K, red_f, red_i);
  Ev<M_LSE, EK> ev(p.child, row, p.mp);
  const int jn = (j0 + J < L ? j0 + J : L) - j0;
  const float padsum = padsum_sh;
  DivMod dm(threadIdx.x, K);
  for (int i0 = threadIdx.x; i0 < jn; i0 += 4 * FF_T) {
    typename Ev<M_LSE, EK>::Raw r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int i = i0 + u * FF_T;
      if (i < jn) r[u] = ev.load(j0 + i);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int i = i0 + u * FF_T;
      if (i < jn) {
        // element j = j0 + i <- outputs t in [j - b, j - a]: local window start i (block q)
        const float cq = C[dm.q];
        float S = A[ffpad(i)];
        if (dm.r != 0) S = fmaf(Pp[ffpad(i + K - 1)], ex2f(tau2 * (cq - C[dm.q + 1])), S);
        float g = 0.f;
        if (S != 0.f) g = S * ex2f(tau2 * (sg * ev.value(j0 + i, r[u]) - cq));
        if (j0 + i == L - 1) g += padsum;
        ev.grad(j0 + i, r[u], g);
      }
      dm.next();
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
bool fast_lse_applicable(const FGParams& p) {
  return !p.padmode && !p.fill && p.K >= 2 && p.K <= FF_N / 4 && p.L < (1 << 30);
}

int fast_lse_tile(int K) { return FF_N - K + 1; }

cudaError_t launch_lse_fast_fwd(int ek, FGParams& p, int* slow, cudaStream_t st) {
  const int J = FF_N - p.K + 1;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  switch (ek) {
    case EK_AFF1:
    case EK_AFF: k_lse_fast_fwd<EK_AFF><<<grid, FF_T, 0, st>>>(p, slow); break;
    case EK_NORM: k_lse_fast_fwd<EK_NORM><<<grid, FF_T, 0, st>>>(p, slow); break;
    case EK_SRC: k_lse_fast_fwd<EK_SRC><<<grid, FF_T, 0, st>>>(p, slow); break;
    case EK_PAIR: k_lse_fast_fwd<EK_PAIR><<<grid, FF_T, 0, st>>>(p, slow); break;
    default: k_lse_fast_fwd<EK_GEN><<<grid, FF_T, 0, st>>>(p, slow); break;
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_lse_fast_bwd(int ek, FGParams& p, int* slow, cudaStream_t st) {
  const int J = FF_N - p.K + 1;
  dim3 grid((unsigned)((p.L + J - 1) / J), (unsigned)p.B);
  switch (ek) {
    case EK_AFF1:
    case EK_AFF: k_lse_fast_bwd<EK_AFF><<<grid, FF_T, 0, st>>>(p, slow); break;
    case EK_NORM: k_lse_fast_bwd<EK_NORM><<<grid, FF_T, 0, st>>>(p, slow); break;
    case EK_SRC: k_lse_fast_bwd<EK_SRC><<<grid, FF_T, 0, st>>>(p, slow); break;
    case EK_PAIR: k_lse_fast_bwd<EK_PAIR><<<grid, FF_T, 0, st>>>(p, slow); break;
    default: k_lse_fast_bwd<EK_GEN><<<grid, FF_T, 0, st>>>(p, slow); break;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
