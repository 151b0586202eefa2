// smooth.cu — smooth-interval Eventually / Always, LSE and softmax modes
// (masking.py:207-215, 300-305; smoothing.py:85-109; tape.py:360-387).
//
//   w_i = relu(sigmoid(c (i - a L)) - sigmoid(c (i - b L)) - eps),  i = 0..L-1
//   padded = child ++ [pad] * (L - 1)
//   LSE:     out[t] = sg * log(sum_{w_i > 0} w_i exp(tau u_{t+i})) / tau
//   softmax: out[t] = sg * sum w_i u e / sum w_i e,  e = exp(tau u_{t+i})
// with u = sg * padded (max space).  The reference shifts by the hard max of
// the kept entries; here the shift is the running max of the log-weighted
// scores v_i = tau u_{t+i} + ln w_i (the same value in exact arithmetic, and
// it keeps tail weights down to 1e-300 representable: ln w is stored, never w).
// The kept range {i : w_i > 0} is contiguous (a difference of two sigmoids is
// unimodal) and is computed on the host in fp64 together with log2(w_i).
// Hard mode does not come here: it is the vHGW window kernel over the kept
// range with padded-window semantics (fg.cu, padmode).
//
// Backward (gather form, weights recomputed, nothing stored per pair):
//   g_child[j] = sum_{t = j - i} g_t * d out_t / d u_j        (thread per j)
//   d out / d w_i summed over rows and t (thread per i, fp64 atomics), then
//   d_a, d_b, d_c = sum_i dW_i * d w_i / d(a, b, c)            (fp64)
#include "kernels.cuh"

namespace stlg {

constexpr int S_T = 256;    // outputs (or child elements) per CTA
constexpr int S_CH = 1024;  // window offsets staged per chunk

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
// fold a group of n log2-scores v[] with group max gm (>= m) into (m, s):
// s <- s 2^(m - gm) + sum 2^(v_i - gm).  NaN scores propagate through the sum
// (fmaxf drops them from gm), -inf scores add 0, an all -inf state stays (-inf, 0).
__device__ __forceinline__ void lse_group(float& m, float& s, const float* v, int n, float gm) {
  if (gm == -INFINITY) {  // empty state, no finite score: only a NaN can change s
    float a = 0.f;
    for (int i = 0; i < n; ++i) a += ex2f(v[i]);
    s += a;
    return;
  }
  s *= ex2f(m - gm);  // m = -inf (empty state) -> 0
  m = gm;
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int i = 0; i < n; i += 2) {
    a0 += ex2f(v[i] - gm);
    a1 += ex2f(v[i + 1] - gm);
  }
  s += a0 + a1;
}
template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_fwd(const __grid_constant__ SParams p) {
  __shared__ __align__(16) float U[S_T + S_CH + 8];
  __shared__ __align__(16) float LW[S_CH + 4];  // (>= 4 S_T: the fast path's group sums)
  __shared__ float Red[3][S_T / 32];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int t0 = blockIdx.x * S_T;
  const int K = p.i_hi - p.i_lo + 1;
  const float sg = p.sg, tau2 = p.mp.tau2;
  const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
  const int t = t0 + threadIdx.x;
  float m = -INFINITY, s = 0.f, uc = 0.f;
  double S64 = 0.0, D64 = 0.0;  // softmax running sums
  bool first = true;
  for (int k0 = 0; k0 < K; k0 += S_CH) {
    const int kc = min(S_CH, K - k0);
    const int base = t0 + p.i_lo + k0;
    for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
      int idx = base + q;
      U[q] = sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
    }
    for (int q = threadIdx.x; q < kc; q += S_T) LW[q] = p.lw2[p.i_lo + k0 + q];
    __syncthreads();
    if (MODE == M_LSE && K <= S_CH) {
      // factorised window sum: w_i e^{tau u_{t+i}} = (2^{lw_i - lwmax}) (2^{tau2 (u_{t+i} - umax)})
      // x 2^{lwmax + tau2 umax}, so a tile whose staged u span is <= 96 / tau2 needs one
      // ex2 per staged element and one FMA per pair.  Every window holds the largest
      // weight, so its best term is >= 2^-96; a factor or product only flushes below
      // 2^-126, i.e. < 2^-30 of that term, below fp32 resolution of the sum.  Wider tiles
      // (or non-finite values) take the exact grouped path below.
      float umax = -INFINITY, umin = INFINITY, lwmax = -INFINITY;
      bool nan_u = false;  // fmaxf / fminf drop NaN: flag it explicitly (exact path below)
      for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
        umax = fmaxf(umax, U[q]);
        umin = fminf(umin, U[q]);
        nan_u |= U[q] != U[q];
      }
      for (int q = threadIdx.x; q < kc; q += S_T) lwmax = fmaxf(lwmax, LW[q]);
      for (int o = 16; o > 0; o >>= 1) {
        umax = fmaxf(umax, __shfl_xor_sync(0xffffffffu, umax, o));
        umin = fminf(umin, __shfl_xor_sync(0xffffffffu, umin, o));
        lwmax = fmaxf(lwmax, __shfl_xor_sync(0xffffffffu, lwmax, o));
      }
      if ((threadIdx.x & 31) == 0) {
        Red[0][threadIdx.x >> 5] = umax;
        Red[1][threadIdx.x >> 5] = umin;
        Red[2][threadIdx.x >> 5] = lwmax;
      }
      nan_u = __syncthreads_or(nan_u);
      umax = Red[0][0];
      umin = Red[1][0];
      lwmax = Red[2][0];
      for (int w = 1; w < S_T / 32; ++w) {
        umax = fmaxf(umax, Red[0][w]);
        umin = fminf(umin, Red[1][w]);
        lwmax = fmaxf(lwmax, Red[2][w]);
      }
      const float span = tau2 * (umax - umin);  // inf -> NaN span -> exact path
      if (!nan_u && span <= 96.f && lwmax > -INFINITY) {
        __syncthreads();  // every thread has read Red
        // factors in place; zero tails so the 4-wide loads below read finite zeros
        for (int q = threadIdx.x; q < S_T + kc + 7; q += S_T)
          U[q] = q < S_T + kc - 1 ? ex2f(tau2 * (U[q] - umax)) : 0.f;
        for (int q = threadIdx.x; q < kc + 4; q += S_T) LW[q] = q < kc ? ex2f(LW[q] - lwmax) : 0.f;
        __syncthreads();
        // register-blocked correlation: thread (g, o) sums 4 outputs 4o .. 4o+3 over a
        // quarter g of the offsets; per 4 offsets 3 conflict-free LDS.128 feed 16 FMAs
        {
          const int o = threadIdx.x & (S_T / 4 - 1), g = threadIdx.x / (S_T / 4);
          const int kc4 = (kc + 3) & ~3;
          const int chunk = ((kc4 >> 2) + 3) & ~3;
          const int kb = g * chunk, ke = min(kc4, kb + chunk);
          const float4* U4 = reinterpret_cast<const float4*>(U);
          const float4* W4 = reinterpret_cast<const float4*>(LW);
          float r0 = 0.f, r1 = 0.f, r2 = 0.f, r3 = 0.f;
          // (b of one step is a of the next: one LDS.128 of U per 16 FMAs)
          float4 a = kb < ke ? U4[o + (kb >> 2)] : make_float4(0.f, 0.f, 0.f, 0.f);
          for (int k = kb; k < ke; k += 4) {
            const float4 w = W4[k >> 2];
            const float4 b = U4[o + (k >> 2) + 1];
            r0 = fmaf(w.x, a.x, fmaf(w.y, a.y, fmaf(w.z, a.z, fmaf(w.w, a.w, r0))));
            r1 = fmaf(w.x, a.y, fmaf(w.y, a.z, fmaf(w.z, a.w, fmaf(w.w, b.x, r1))));
            r2 = fmaf(w.x, a.z, fmaf(w.y, a.w, fmaf(w.z, b.x, fmaf(w.w, b.y, r2))));
            r3 = fmaf(w.x, a.w, fmaf(w.y, b.x, fmaf(w.z, b.y, fmaf(w.w, b.z, r3))));
            a = b;
          }
          __syncthreads();  // LW is reused as the cross-group reduction buffer
          LW[g * S_T + 4 * o] = r0;
          LW[g * S_T + 4 * o + 1] = r1;
          LW[g * S_T + 4 * o + 2] = r2;
          LW[g * S_T + 4 * o + 3] = r3;
          __syncthreads();
        }
        if (t < L) {
          m = fmaf(tau2, umax, lwmax);
          s = (LW[threadIdx.x] + LW[S_T + threadIdx.x]) + (LW[2 * S_T + threadIdx.x] + LW[3 * S_T + threadIdx.x]);
        }
        first = false;
        __syncthreads();
        continue;  // K <= S_CH: this was the only chunk
      }
    }
    if (MODE == M_LSE && t < L) {
      // groups of SG offsets: scores to registers, one max, one rescale of s,
      // then one ex2 + add per pair (~6 issue slots per pair instead of ~10 for
      // the per-pair online update: the loop is MUFU-bound, not issue-bound)
      constexpr int SG = 32;
      int k = 0;
      for (; k + SG <= kc; k += SG) {
        float v[SG];
        float gm = m;
#pragma unroll
        for (int i = 0; i < SG; ++i) {
          v[i] = fmaf(tau2, U[threadIdx.x + k + i], LW[k + i]);
          gm = fmaxf(gm, v[i]);
        }
        lse_group(m, s, v, SG, gm);
      }
      if (k < kc) {
        float v[SG];
        float gm = m;
#pragma unroll
        for (int i = 0; i < SG; ++i) {
          v[i] = (k + i < kc) ? fmaf(tau2, U[threadIdx.x + k + i], LW[k + i]) : -INFINITY;
          gm = fmaxf(gm, v[i]);
        }
        lse_group(m, s, v, SG, gm);
      }
      first = false;
    } else if (MODE != M_LSE && t < L) {
      // softmax: the same groups; the payload sum D = sum e (u - uc) uses a fixed
      // centre uc (no re-centering when the max moves), group partials in fp32 and
      // the running (S, D) in fp64: only SG terms ever meet in one fp32 sum
      constexpr int SG = 32;
      if (first) {
        uc = U[threadIdx.x];
        first = false;
      }
      for (int k = 0; k < kc; k += SG) {
        float v[SG];
        float gm = m;
#pragma unroll
        for (int i = 0; i < SG; ++i) {
          v[i] = (k + i < kc) ? fmaf(tau2, U[threadIdx.x + k + i], LW[k + i]) : -INFINITY;
          gm = fmaxf(gm, v[i]);
        }
        if (gm == -INFINITY) {  // empty state, no finite score: only a NaN can change S
          float a = 0.f;
          for (int i = 0; i < SG; ++i) a += ex2f(v[i]);
          S64 += a;
          continue;
        }
        const double sc = (double)ex2f(m - gm);
        m = gm;
        float gs0 = 0.f, gs1 = 0.f, gd0 = 0.f, gd1 = 0.f;
#pragma unroll
        for (int i = 0; i < SG; i += 2) {
          const float e0 = ex2f(v[i] - gm), e1 = ex2f(v[i + 1] - gm);
          const float d0 = (k + i < kc) ? U[threadIdx.x + k + i] - uc : 0.f;
          const float d1 = (k + i + 1 < kc) ? U[threadIdx.x + k + i + 1] - uc : 0.f;
          gs0 += e0;
          gs1 += e1;
          gd0 = fmaf(e0, d0, gd0);
          gd1 = fmaf(e1, d1, gd1);
        }
        S64 = fma(S64, sc, (double)(gs0 + gs1));
        D64 = fma(D64, sc, (double)(gd0 + gd1));
      }
    }
    __syncthreads();
  }
  if (t < L) {
    if (MODE == M_LSE) {
      p.out[row * L + t] = sg * ((m + lg2f(s)) * p.mp.inv_tau2);  // log(sum w e^{tau u}) / tau
    } else {
      // double-float window mean M and LSE L (max space) for the fp64 d/dw pass:
      // aux = [L_hi | M_lo | L_lo] (three [B, L] planes)
      const double M64 = (double)uc + D64 / S64;
      const double L64 = ((double)m + log2(S64)) / (double)tau2;
      const float Mh = (float)M64, Lh = (float)L64;
      const long long BL = p.B * (long long)L;
      p.out[row * L + t] = sg * Mh;
      p.aux[row * L + t] = Lh;
      p.aux[BL + row * L + t] = (float)(M64 - (double)Mh);
      p.aux[2 * BL + row * L + t] = (float)(L64 - (double)Lh);
    }
  }
}

// ---------------------------------------------------------------------------
// backward 1: child cotangent, thread per child element j (incl. virtual pad
// positions j >= L, which sum into c[L-1] for 'last' padding)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_bwd_child(const __grid_constant__ SParams p) {
  __shared__ __align__(16) float Gt[S_T + S_CH + 8];
  __shared__ float Mt[S_T + S_CH];
  __shared__ float Lt[(MODE == M_SOFT) ? S_T + S_CH : 1];
  __shared__ __align__(16) float LW[S_CH + 4];
  __shared__ float Rc[6][S_T / 32];
  const long long row = blockIdx.y;
  const int L = (int)p.L;
  const int j0 = blockIdx.x * S_T;
  const int K = p.i_hi - p.i_lo + 1;
  const float sg = p.sg, tau2 = p.mp.tau2, tau = p.mp.tau;
  const int j = j0 + threadIdx.x;
  const int jmax = L - 1;  // real positions only (virtual pad positions: k_smooth_bwd_pad)
  float uj = 0.f;
  if (j <= jmax) uj = sg * expr_eval<MODE>(p.child, row, j, p.mp);
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  float acc = 0.f;
  // offsets i in [i_lo + k0, i_lo + k0 + kc): t = j - i in [j0 - i_lo - k0 - kc + 1, j0 + S_T - 1 - i_lo - k0]
  for (int k0 = 0; k0 < K; k0 += S_CH) {
    const int kc = min(S_CH, K - k0);
    const int tlo = j0 - p.i_lo - k0 - (kc - 1);
    int allnz = 1;
    for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
      int tt = tlo + q;
      bool v = tt >= 0 && tt < L;
      float g = v ? cot[tt] : 0.f;
      allnz &= (g != 0.f) | !v;
      Gt[q] = g;
      // LSE: a staged M of +inf turns an out-of-range t into a 0 weight (branch-free path)
      Mt[q] = (v && g != 0.f) ? sg * outr[tt] : (MODE == M_LSE ? INFINITY : 0.f);
      if (MODE == M_SOFT) Lt[q] = (v && g != 0.f) ? p.aux_in[row * L + tt] : 0.f;
    }
    for (int q = threadIdx.x; q < kc; q += S_T) LW[q] = p.lw2[p.i_lo + k0 + q];
    // dense cotangent over the staged range (e.g. the trace-mode ones seed):
    // no per-pair zero test, 4 issue slots + 2 loads per pair
    const int dense = __syncthreads_and(allnz);
    if (MODE == M_LSE && K <= S_CH) {
      // factorised, as the forward and the d/dw pass:
      //   g_t 2^{tau2 (u_j - M_t) + lw_i} = A_t W_i 2^{tau2 (u_j - mmin) + lwmax + ge},
      //   A_t = ldexp(g_t, -ge) 2^{tau2 (mmin - M_t)},  W_i = 2^{lw_i - lwmax}  (both <= 1),
      // so a tile whose u and M values span <= 100 / tau2 needs one ex2 per staged element
      // and one FMA per pair (the per-pair ex2 below made this kernel MUFU-bound).  A
      // product that flushes to zero is < 2^-26 |g|max: below the tolerance.  The child sum
      // is a convolution in the offset, i.e. a correlation against the reversed weights.
      const int nq = S_T + kc - 1;
      float umx = -INFINITY, umn = INFINITY, mmx = -INFINITY, mmn = INFINITY, gmx = 0.f, lwm = -INFINITY;
      bool bad = false;
      if (j <= jmax) {
        umx = umn = uj;
        bad = !(fabsf(uj) < INFINITY);
      }
      for (int q = threadIdx.x; q < nq; q += S_T) {
        const float g = Gt[q];
        if (g != 0.f) {
          mmx = fmaxf(mmx, Mt[q]);
          mmn = fminf(mmn, Mt[q]);
          gmx = fmaxf(gmx, fabsf(g));
          bad |= !(fabsf(Mt[q]) < INFINITY) || !(fabsf(g) < INFINITY);
        }
      }
      for (int q = threadIdx.x; q < kc; q += S_T) lwm = fmaxf(lwm, LW[q]);
      for (int o = 16; o > 0; o >>= 1) {
        umx = fmaxf(umx, __shfl_xor_sync(0xffffffffu, umx, o));
        umn = fminf(umn, __shfl_xor_sync(0xffffffffu, umn, o));
        mmx = fmaxf(mmx, __shfl_xor_sync(0xffffffffu, mmx, o));
        mmn = fminf(mmn, __shfl_xor_sync(0xffffffffu, mmn, o));
        gmx = fmaxf(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
        lwm = fmaxf(lwm, __shfl_xor_sync(0xffffffffu, lwm, o));
      }
      if ((threadIdx.x & 31) == 0) {
        Rc[0][threadIdx.x >> 5] = umx;
        Rc[1][threadIdx.x >> 5] = umn;
        Rc[2][threadIdx.x >> 5] = mmx;
        Rc[3][threadIdx.x >> 5] = mmn;
        Rc[4][threadIdx.x >> 5] = gmx;
        Rc[5][threadIdx.x >> 5] = lwm;
      }
      bad = __syncthreads_or(bad);
      umx = Rc[0][0], umn = Rc[1][0], mmx = Rc[2][0], mmn = Rc[3][0], gmx = Rc[4][0], lwm = Rc[5][0];
      for (int w = 1; w < S_T / 32; ++w) {
        umx = fmaxf(umx, Rc[0][w]);
        umn = fminf(umn, Rc[1][w]);
        mmx = fmaxf(mmx, Rc[2][w]);
        mmn = fminf(mmn, Rc[3][w]);
        gmx = fmaxf(gmx, Rc[4][w]);
        lwm = fmaxf(lwm, Rc[5][w]);
      }
      if (gmx == 0.f) {  // no cotangent reaches this tile's children: acc stays 0
        __syncthreads();
        continue;  // K <= S_CH: the only chunk
      }
      const float span = tau2 * (fmaxf(umx, mmx) - fminf(umn, mmn));
      if (!bad && span <= 100.f && gmx < INFINITY && lwm > -INFINITY) {
        int ge;
        frexpf(gmx, &ge);
        __syncthreads();  // Rc read everywhere; Gt / LW are rewritten in place below
        for (int q = threadIdx.x; q < S_T + kc + 7; q += S_T) {
          float a = 0.f;
          if (q < nq) {
            const float g = Gt[q];
            a = g != 0.f ? ldexpf(g, -ge) * ex2f(tau2 * (mmn - Mt[q])) : 0.f;
          }
          Gt[q] = a;
        }
        float wr[4];  // reversed weights (each thread rewrites the slots it read)
        const int kc4 = (kc + 3) & ~3;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int q = threadIdx.x + r * S_T;
          wr[r] = q < kc ? ex2f(LW[kc - 1 - q] - lwm) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int q = threadIdx.x + r * S_T;
          if (q < kc4) LW[q] = wr[r];
        }
        __syncthreads();
        {
          const int o = threadIdx.x & (S_T / 4 - 1), g = threadIdx.x / (S_T / 4);
          const int chunk = ((kc4 >> 2) + 3) & ~3;
          const int kb = g * chunk, ke = min(kc4, kb + chunk);
          const float4* A4 = reinterpret_cast<const float4*>(Gt);
          const float4* W4 = reinterpret_cast<const float4*>(LW);
          float r0 = 0.f, r1 = 0.f, r2 = 0.f, r3 = 0.f;
          // carried: b of one step is a of the next
          float4 a = kb < ke ? A4[o + (kb >> 2)] : make_float4(0.f, 0.f, 0.f, 0.f);
          for (int k = kb; k < ke; k += 4) {
            const float4 w = W4[k >> 2];
            const float4 b = A4[o + (k >> 2) + 1];
            r0 = fmaf(w.x, a.x, fmaf(w.y, a.y, fmaf(w.z, a.z, fmaf(w.w, a.w, r0))));
            r1 = fmaf(w.x, a.y, fmaf(w.y, a.z, fmaf(w.z, a.w, fmaf(w.w, b.x, r1))));
            r2 = fmaf(w.x, a.z, fmaf(w.y, a.w, fmaf(w.z, b.x, fmaf(w.w, b.y, r2))));
            r3 = fmaf(w.x, a.w, fmaf(w.y, b.x, fmaf(w.z, b.y, fmaf(w.w, b.z, r3))));
            a = b;
          }
          __syncthreads();  // LW becomes the cross-group reduction buffer
          LW[g * S_T + 4 * o] = r0;
          LW[g * S_T + 4 * o + 1] = r1;
          LW[g * S_T + 4 * o + 2] = r2;
          LW[g * S_T + 4 * o + 3] = r3;
          __syncthreads();
        }
        if (j <= jmax) {
          const float sum = (LW[threadIdx.x] + LW[S_T + threadIdx.x]) + (LW[2 * S_T + threadIdx.x] + LW[3 * S_T + threadIdx.x]);
          acc = ldexpf(sum * ex2f(fmaf(tau2, uj - mmn, lwm)), ge);
        }
        __syncthreads();
        continue;  // K <= S_CH: the only chunk
      }
    }
    if (MODE == M_LSE && dense && fabsf(uj) < INFINITY) {  // (an infinite u_j takes the exact path)
      if (j <= jmax) {
        float a0 = 0.f, a1 = 0.f;
        const float* gq = Gt + threadIdx.x + kc - 1;
        const float* mq = Mt + threadIdx.x + kc - 1;
        int k = 0;
#pragma unroll 8
        for (; k + 1 < kc; k += 2) {
          a0 = fmaf(gq[-k], ex2f(fmaf(tau2, uj - mq[-k], LW[k])), a0);
          a1 = fmaf(gq[-k - 1], ex2f(fmaf(tau2, uj - mq[-k - 1], LW[k + 1])), a1);
        }
        if (k < kc) a0 = fmaf(gq[-k], ex2f(fmaf(tau2, uj - mq[-k], LW[k])), a0);
        acc += a0 + a1;
      }
    } else if (j <= jmax) {
      // t = j - i_lo - k0 - k  ->  index into the staged range: (kc - 1 - k) + threadIdx.x
      for (int k = 0; k < kc; ++k) {
        int q = threadIdx.x + kc - 1 - k;
        float g = Gt[q];
        if (g == 0.f) continue;
        if (MODE == M_LSE) {
          acc = fmaf(g, ex2f(fmaf(tau2, uj - Mt[q], LW[k])), acc);
        } else {
          float w = ex2f(fmaf(tau2, uj - Lt[q], LW[k]));
          acc = fmaf(g * w, fmaf(tau, uj - Mt[q], 1.f), acc);
        }
      }
    }
    __syncthreads();
  }
  float* gb = p.gbuf + row * L;
  if (j < L) {
    if (j == L - 1) atomicAdd(gb + j, acc);
    else gb[j] = acc;
  }
}

// ---------------------------------------------------------------------------
// backward 1b ('last' padding): every virtual pad position j >= L holds the same
// value u_pad and sums into c[L-1], so their total is, per output t,
//   g_t * F_t * sum_{i >= max(L - t, i_lo)} w_i        (one term per t, lw2[L + m])
// with F_t = 2^{tau2 (u_pad - M_t)} (LSE) or 2^{tau2 (u_pad - L_t)} (1 + tau (u_pad - M_t))
// (softmax), both combined with the log2 suffix sum inside one ex2.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_bwd_pad(const __grid_constant__ SParams p) {
  __shared__ float red[S_T / 32];
  const long long row = blockIdx.x;
  const int L = (int)p.L;
  const float sg = p.sg, tau2 = p.mp.tau2, tau = p.mp.tau;
  const float up = sg * expr_eval<MODE>(p.child, row, L - 1, p.mp);
  const float* cot = p.cot + row * L;
  const float* outr = p.out_in + row * L;
  const float* lws = p.lw2 + L;
  float acc = 0.f;
  for (int t = max(0, L - p.i_hi) + (int)threadIdx.x; t < L; t += S_T) {
    const float g = cot[t];
    if (g == 0.f) continue;
    const float ls = lws[max(L - t, p.i_lo)];
    if (MODE == M_LSE) {
      acc = fmaf(g, ex2f(fmaf(tau2, up - sg * outr[t], ls)), acc);
    } else {
      const float w = ex2f(fmaf(tau2, up - p.aux_in[row * L + t], ls));
      acc = fmaf(g * w, fmaf(tau, up - sg * outr[t], 1.f), acc);
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.f;
    for (int w = 0; w < S_T / 32; ++w) sum += red[w];
    if (sum != 0.f) atomicAdd(p.gbuf + row * L + (L - 1), sum);
  }
}

// ---------------------------------------------------------------------------
// backward 2: w_i * d out / d w_i summed over t and rows (thread per offset i)
//   LSE:  w_i exp(tau (u_{t+i} - M_t)) / tau     softmax: w_i exp(tau (u - L_t)) (u - M_t)
// (the weight rides inside the ex2 as log2 w_i: the bare derivative reaches 1e300 on
// 1e-300 tail weights and overflows fp32; k_smooth_abc divides by the same 2^{lw2_i})
// (zero where w_i == 0: the reference masks those entries before exp, tape.py:372)
// ---------------------------------------------------------------------------
// 2^x in fp64 for the d/dw factors: exact power of two times ex2 of the fraction (~2^-22
// relative, the precision of the fp32 partial sums it scales) instead of the fp64 exp2
// routine
__device__ __forceinline__ double sm_ex2d(double x) {
  if (!(x > -1022.0)) return 0.0;
  const double n = floor(fmin(x, 1023.0));
  return (double)ex2f((float)(x - n)) * __hiloint2double(((int)n + 1023) << 20, 0);
}

template <int MODE>
__global__ void __launch_bounds__(S_T) k_smooth_bwd_w(const __grid_constant__ SParams p) {
  __shared__ __align__(16) float U[S_T + S_CH];
  __shared__ __align__(16) float Gt[S_T];
  __shared__ __align__(16) float Mt[S_T];
  __shared__ float Lt[S_T];
  __shared__ double M64t[MODE == M_SOFT ? S_T : 1], L64t[MODE == M_SOFT ? S_T : 1];
  __shared__ float Rw[5][S_T / 32];
  __shared__ double red[S_CH];
  const int L = (int)p.L;
  const int K = p.i_hi - p.i_lo + 1;
  const float sg = p.sg, tau2 = p.mp.tau2, itau = 1.f / p.mp.tau;
  const long long rp = (p.B + gridDim.x - 1) / gridDim.x;  // rows per CTA (smooth_dw_parts)
  const long long r0 = (long long)blockIdx.x * rp;
  const long long r1 = min(r0 + rp, p.B);
  for (int k0 = 0; k0 < K; k0 += S_CH) {
    const int kc = min(S_CH, K - k0);
    // each thread owns offsets i = i_lo + k0 + k, k = threadIdx.x + S_T * c
    double acc[S_CH / S_T];  // per-row tile partials (<= 256 terms) meet in fp64
    float lwi[S_CH / S_T];   // log2 w_i of the thread's offsets, folded into every ex2
#pragma unroll
    for (int c = 0; c < S_CH / S_T; ++c) {
      acc[c] = 0.0;
      const int k = threadIdx.x + S_T * c;
      lwi[c] = k < kc ? p.lw2[p.i_lo + k0 + k] : -INFINITY;
    }
    double accf[4] = {0.0, 0.0, 0.0, 0.0};  // LSE factorised path: offsets 4 tid + r
    float lwf[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = 4 * (int)threadIdx.x + r;
      lwf[r] = k < kc ? p.lw2[p.i_lo + k0 + k] : -INFINITY;
    }
    // the CTA walks every output tile of its rows: one partial row per CTA
    for (int t0 = 0; t0 < L; t0 += S_T)
    for (long long row = r0; row < r1; ++row) {
      const int nt = min(S_T, L - t0);
      const float padv = p.pad_last ? expr_eval<MODE>(p.child, row, L - 1, p.mp) : p.pad_value;
      const int base = t0 + p.i_lo + k0;
      for (int q = threadIdx.x; q < S_T + kc - 1; q += S_T) {
        int idx = base + q;
        U[q] = sg * (idx < L ? expr_eval<MODE>(p.child, row, idx, p.mp) : padv);
      }
      int nz = 1;
      if (threadIdx.x < S_T) {
        int tt = t0 + threadIdx.x;
        bool v = tt < L;
        float g = v ? p.cot[row * L + tt] : 0.f;
        Gt[threadIdx.x] = g;
        Mt[threadIdx.x] = v ? sg * p.out_in[row * L + tt] : 0.f;
        Lt[threadIdx.x] = (MODE == M_SOFT && v) ? p.aux_in[row * L + tt] : 0.f;
        if (MODE == M_SOFT) {  // double-float M and L written by the forward
          const long long BL = p.B * (long long)L;
          M64t[threadIdx.x] = v ? (double)Mt[threadIdx.x] + (double)p.aux_in[BL + row * L + tt] : 0.0;
          L64t[threadIdx.x] = v ? (double)Lt[threadIdx.x] + (double)p.aux_in[2 * BL + row * L + tt] : 0.0;
        }
        nz = (g != 0.f) | !v;
      }
      // dense cotangent row tile: no per-pair zero test, (G, M) read 4 at a time
      const int dense = __syncthreads_and(nz);
      bool done = false;
      if (MODE == M_LSE) {
        // factorised: g_t 2^{tau2 (u_{t+i} - M_t)} = A_t E_{t+i} 2^{tau2 (umax - Mmax)} with
        // A_t = g_t 2^{tau2 (Mmax - M_t)} in [1, 2^100] |g| and E_j = 2^{tau2 (u_j - umax)} in
        // [2^-100, 1]: no factor or product leaves the fp32 range, so one ex2 per staged
        // element and one FMA per pair replace the per-pair ex2
        // |g| enters through a power-of-two scale 2^-ge (exact), so A_t stays within
        // [2^-1, 2^100] for every cotangent magnitude and ge is added back in fp64
        float umx = -INFINITY, umn = INFINITY, mmx = -INFINITY, mmn = INFINITY, gmx = 0.f;
        bool bad = false;  // NaN child samples: the exact path (fmaxf / fminf drop NaN)
        for (int q = threadIdx.x; q < nt + kc - 1; q += S_T) {
          umx = fmaxf(umx, U[q]);
          umn = fminf(umn, U[q]);
          bad |= U[q] != U[q];
        }
        if (threadIdx.x < nt && Gt[threadIdx.x] != 0.f) {
          mmx = mmn = Mt[threadIdx.x];
          gmx = fabsf(Gt[threadIdx.x]);
        }
        for (int o = 16; o > 0; o >>= 1) {
          umx = fmaxf(umx, __shfl_xor_sync(0xffffffffu, umx, o));
          umn = fminf(umn, __shfl_xor_sync(0xffffffffu, umn, o));
          mmx = fmaxf(mmx, __shfl_xor_sync(0xffffffffu, mmx, o));
          mmn = fminf(mmn, __shfl_xor_sync(0xffffffffu, mmn, o));
          gmx = fmaxf(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
        }
        if ((threadIdx.x & 31) == 0) {
          Rw[0][threadIdx.x >> 5] = umx;
          Rw[1][threadIdx.x >> 5] = umn;
          Rw[2][threadIdx.x >> 5] = mmx;
          Rw[3][threadIdx.x >> 5] = mmn;
          Rw[4][threadIdx.x >> 5] = gmx;
        }
        bad = __syncthreads_or(bad);
        umx = Rw[0][0], umn = Rw[1][0], mmx = Rw[2][0], mmn = Rw[3][0], gmx = Rw[4][0];
        for (int w = 1; w < S_T / 32; ++w) {
          umx = fmaxf(umx, Rw[0][w]);
          umn = fminf(umn, Rw[1][w]);
          mmx = fmaxf(mmx, Rw[2][w]);
          mmn = fminf(mmn, Rw[3][w]);
          gmx = fmaxf(gmx, Rw[4][w]);
        }
        // (a NaN / inf span fails the comparisons: exact path)
        if (!bad && tau2 * (umx - umn) <= 100.f && tau2 * (mmx - mmn) <= 100.f && mmx > -INFINITY &&
            gmx > 0.f && gmx < INFINITY) {
          __syncthreads();  // every thread has read Rw; U / Gt are rewritten below
          // E in place; zeros past the staged range (read by the 4-wide loads, times A = 0)
          for (int q = threadIdx.x; q < S_T + S_CH; q += S_T)
            U[q] = q < nt + kc - 1 ? ex2f(tau2 * (U[q] - umx)) : 0.f;
          int ge;
          frexpf(gmx, &ge);  // gmx in [2^(ge-1), 2^ge)
          if (threadIdx.x < S_T) {
            const float g = Gt[threadIdx.x];
            Gt[threadIdx.x] = (threadIdx.x < nt && g != 0.f)
                                  ? ldexpf(g, -ge) * ex2f(tau2 * (mmx - Mt[threadIdx.x])) : 0.f;
          }
          __syncthreads();
          const double cexp = (double)tau2 * ((double)umx - (double)mmx) + (double)ge;
          // register-blocked: thread owns offsets 4 tid .. 4 tid + 3; per 4 outputs one
          // broadcast LDS.128 of A and two conflict-free LDS.128 of E feed 16 FMAs
          const int kq = 4 * threadIdx.x;
          if (kq < kc) {
            const float4* G4 = reinterpret_cast<const float4*>(Gt);
            const float4* E4 = reinterpret_cast<const float4*>(U);
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            for (int q = 0; q < nt; q += 4) {  // (carrying y into the next x measured slower here)
              const float4 g = G4[q >> 2];
              const float4 x = E4[(q + kq) >> 2], y = E4[((q + kq) >> 2) + 1];
              a0 = fmaf(g.x, x.x, fmaf(g.y, x.y, fmaf(g.z, x.z, fmaf(g.w, x.w, a0))));
              a1 = fmaf(g.x, x.y, fmaf(g.y, x.z, fmaf(g.z, x.w, fmaf(g.w, y.x, a1))));
              a2 = fmaf(g.x, x.z, fmaf(g.y, x.w, fmaf(g.z, y.x, fmaf(g.w, y.y, a2))));
              a3 = fmaf(g.x, x.w, fmaf(g.y, y.x, fmaf(g.z, y.y, fmaf(g.w, y.z, a3))));
            }
            // w_i d out / d w_i convention (k_smooth_abc divides by 2^{lw2_i})
            accf[0] += (double)a0 * sm_ex2d(cexp + (double)lwf[0]);
            accf[1] += (double)a1 * sm_ex2d(cexp + (double)lwf[1]);
            accf[2] += (double)a2 * sm_ex2d(cexp + (double)lwf[2]);
            accf[3] += (double)a3 * sm_ex2d(cexp + (double)lwf[3]);
          }
          done = true;
        }
      }
      if (!done) {
#pragma unroll
      for (int c = 0; c < S_CH / S_T; ++c) {
        int k = threadIdx.x + S_T * c;
        if (k >= kc) break;
        const float lw = lwi[c];
        float a = 0.f;
        if (MODE == M_LSE && dense) {
          float a1 = 0.f;
          int q = 0;
          for (; q + 4 <= nt; q += 4) {
            const float4 g4 = *reinterpret_cast<const float4*>(Gt + q);
            const float4 m4 = *reinterpret_cast<const float4*>(Mt + q);
            a = fmaf(g4.x, ex2f(fmaf(tau2, U[q + k] - m4.x, lw)), a);
            a1 = fmaf(g4.y, ex2f(fmaf(tau2, U[q + k + 1] - m4.y, lw)), a1);
            a = fmaf(g4.z, ex2f(fmaf(tau2, U[q + k + 2] - m4.z, lw)), a);
            a1 = fmaf(g4.w, ex2f(fmaf(tau2, U[q + k + 3] - m4.w, lw)), a1);
          }
          for (; q < nt; ++q) a = fmaf(Gt[q], ex2f(fmaf(tau2, U[q + k] - Mt[q], lw)), a);
          acc[c] += (double)a + (double)a1;
          continue;
        }
        if (MODE == M_SOFT) {
          // softmax: sum_t g_t e^{tau (u - L_t)} (u - M_t) cancels terms of size
          // tau |u - M| down to d(a, b, c): every term in fp64 with the double-float M, L
          double a64 = 0.0;
          for (int q = 0; q < nt; ++q) {
            const float g = Gt[q];
            if (g == 0.f) continue;
            const double u = (double)U[q + k];
            a64 += (double)g * exp2((double)tau2 * (u - L64t[q])) * (u - M64t[q]);
          }
          acc[c] += a64 * exp2((double)lw);  // w_i d out / d w_i convention (k_smooth_abc)
          continue;
        }
        for (int q = 0; q < nt; ++q) {
          float g = Gt[q];
          if (g == 0.f) continue;
          float u = U[q + k];
          a = fmaf(g, ex2f(fmaf(tau2, u - Mt[q], lw)), a);
        }
        acc[c] += (double)a;
      }
      }
      __syncthreads();
    }
    // the CTA's partial row, combined in a fixed order (exact-path owner, then the
    // factorised-path owner of each offset): no atomics, reproducible d(a, b, c)
    for (int q = threadIdx.x; q < kc; q += S_T) red[q] = 0.0;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < S_CH / S_T; ++c) {
      const int k = threadIdx.x + S_T * c;
      if (k < kc) red[k] += (double)sg * acc[c] * (MODE == M_LSE ? (double)itau : 1.0);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = 4 * (int)threadIdx.x + r;
      if (k < kc) red[k] += (double)sg * accf[r] * (double)itau;
    }
    __syncthreads();
    double* part = p.dwpart + (long long)blockIdx.x * L + p.i_lo + k0;
    for (int q = threadIdx.x; q < kc; q += S_T) part[q] = p.lw2[p.i_lo + k0 + q] == -INFINITY ? 0.0 : red[q];
    __syncthreads();
  }
}

// dw64[i] = sum over the partial rows in a fixed order (32 offsets x 8 partial strides
// per CTA, then a fixed-shape tree): deterministic
__global__ void __launch_bounds__(1024) k_smooth_dw_reduce(const double* __restrict__ part, long long parts,
                                                           long long L, int i_lo, int i_hi, double* dw64) {
  __shared__ double s[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (i >= i_lo && i <= i_hi)
    for (long long q = w; q < parts; q += 32) acc += part[q * L + i];
  s[w][lane] = acc;
  __syncthreads();
  if (w == 0 && i < L) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) t += s[k][lane];
    dw64[i] = t;
  }
}

// ---------------------------------------------------------------------------
// d(a, b, c) from d/dw_i (fp64): w_i = relu(lo - hi - eps),
//   lo = sigmoid(c (i - a L)), hi = sigmoid(c (i - b L))   (masking.py:300-305)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sigmoid_d(double z) {
  if (z >= 0) return 1.0 / (1.0 + exp(-z));
  double ez = exp(z);
  return ez / (1.0 + ez);
}

__global__ void k_smooth_abc(const double* __restrict__ dw64, const float* __restrict__ lw2, long long L,
                             double a, double b, double c, double eps, double* d_abc) {
  __shared__ double red[3][32];
  double da = 0, db = 0, dc = 0;
  const double Lf = (double)L;
  for (long long i = threadIdx.x; i < L; i += blockDim.x) {
    double g = dw64[i];
    if (g == 0.0) continue;
    g /= exp2((double)lw2[i]);  // dw64 holds w_i d out / d w_i under the fp32 table weight
    double lo = sigmoid_d((i - a * Lf) * c);
    double hi = sigmoid_d((i - b * Lf) * c);
    if (!(lo - hi - eps > 0)) continue;  // relu gradient is 0 where the clamp is active
    double slo = lo * (1.0 - lo), shi = hi * (1.0 - hi);
    da += g * (-slo * c * Lf);
    db += g * (shi * c * Lf);
    dc += g * (slo * (i - a * Lf) - shi * (i - b * Lf));
  }
  for (int o = 16; o > 0; o >>= 1) {
    da += __shfl_xor_sync(0xffffffffu, da, o);
    db += __shfl_xor_sync(0xffffffffu, db, o);
    dc += __shfl_xor_sync(0xffffffffu, dc, o);
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = da;
    red[1][w] = db;
    red[2][w] = dc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0, s2 = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      s0 += red[0][k];
      s1 += red[1][k];
      s2 += red[2][k];
    }
    d_abc[0] += s0;
    d_abc[1] += s1;
    d_abc[2] += s2;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_smooth_fwd(int mode, SParams& p, cudaStream_t st) {
  dim3 grid((unsigned)((p.L + S_T - 1) / S_T), (unsigned)p.B);
  if (mode == M_LSE) k_smooth_fwd<M_LSE><<<grid, S_T, 0, st>>>(p);
  else k_smooth_fwd<M_SOFT><<<grid, S_T, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_smooth_bwd(int mode, SParams& p, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.gbuf, 0, sizeof(float) * p.B * p.L, st)) != cudaSuccess) return e;
  // real child positions only: the virtual pad positions (j >= L) are summed in
  // closed form by k_smooth_bwd_pad ('last') or dropped (constant padding)
  dim3 g1((unsigned)((p.L + S_T - 1) / S_T), (unsigned)p.B);
  if (mode == M_LSE) k_smooth_bwd_child<M_LSE><<<g1, S_T, 0, st>>>(p);
  else k_smooth_bwd_child<M_SOFT><<<g1, S_T, 0, st>>>(p);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (p.pad_last) {
    if (mode == M_LSE) k_smooth_bwd_pad<M_LSE><<<(unsigned)p.B, S_T, 0, st>>>(p);
    else k_smooth_bwd_pad<M_SOFT><<<(unsigned)p.B, S_T, 0, st>>>(p);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (p.dw64 != nullptr) {
    const long long parts = smooth_dw_parts(p.B);
    if (mode == M_LSE) k_smooth_bwd_w<M_LSE><<<(unsigned)parts, S_T, 0, st>>>(p);
    else k_smooth_bwd_w<M_SOFT><<<(unsigned)parts, S_T, 0, st>>>(p);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_smooth_dw_reduce<<<(unsigned)((p.L + 31) / 32), 1024, 0, st>>>(p.dwpart, parts, p.L, p.i_lo, p.i_hi,
                                                                     p.dw64);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  FGParams q;
  memset(&q, 0, sizeof(q));
  q.B = p.B;
  q.L = p.L;
  q.mp = p.mp;
  q.child = p.child;
  return launch_pointwise_vjp(mode, q, p.gbuf, st);
}

// weight table on the device (fp64, then fp32 log2): lw2[i] = log2 w_i for i in
// [i_lo, i_hi] (-inf elsewhere), lw2[L + m] = log2 sum_{i >= m} w_i — the kernel form of
// the host table (no pageable upload, so smooth formulas capture into CUDA graphs)
__global__ void __launch_bounds__(1024) k_smooth_table(double a, double b, double c, double eps, long long L,
                                                       int i_lo, int i_hi, float* __restrict__ lw2) {
  __shared__ double part[1024];
  const int tid = threadIdx.x;
  const long long per = (L + 1023) / 1024;
  const long long m0 = (long long)tid * per, m1 = min(m0 + per, L);
  const double Lf = (double)L;
  auto wgt = [&](long long i) -> double {
    if (i < i_lo || i > i_hi) return 0.0;
    const double w = sigmoid_d(((double)i - a * Lf) * c) - sigmoid_d(((double)i - b * Lf) * c) - eps;
    return w > 0.0 ? w : 0.0;
  };
  double s = 0.0;
  for (long long i = m0; i < m1; ++i) {
    const double w = wgt(i);
    lw2[i] = w > 0.0 ? (float)log2(w) : -INFINITY;
    s += w;
  }
  // exclusive suffix totals of the thread segments: warp shuffles, then the later warps
  // (fixed shape, so the same table every call)
  const int lane = tid & 31, warp = tid >> 5;
  double inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_down_sync(0xffffffffu, inc, o);
    if (lane + o < 32) inc += v;
  }
  if (lane == 0) part[warp] = inc;
  __syncthreads();
  double later = 0.0;
  for (int w = 31; w > warp; --w) later += part[w];
  const double nxt = __shfl_down_sync(0xffffffffu, inc, 1);
  double suf = later + (lane < 31 ? nxt : 0.0);
  for (long long m = m1 - 1; m >= m0; --m) {
    suf += wgt(m);
    lw2[L + m] = suf > 0.0 ? (float)log2(suf) : -INFINITY;
  }
}

cudaError_t launch_smooth_table(double a, double b, double c, double eps, long long L, int i_lo, int i_hi,
                                float* lw2, cudaStream_t st) {
  k_smooth_table<<<1, 1024, 0, st>>>(a, b, c, eps, L, i_lo, i_hi, lw2);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_smooth_abc(const double* dw64, const float* lw2, long long L, double a, double b,
                              double c, double eps, double* d_abc, cudaStream_t st) {
  k_smooth_abc<<<1, 1024, 0, st>>>(dw64, lw2, L, a, b, c, eps, d_abc);
  count_launch();
  return cudaGetLastError();
}

}  // namespace stlg
