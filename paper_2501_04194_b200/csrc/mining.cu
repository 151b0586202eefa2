// mining.cu — batched interval-mining objective on the GPU.
//
// Reference: apps.py:272-335.  For a dataset X [n, L] and a window (a, b) with
// sharpness c, `_mining_loss_var` forms the smooth-interval weights
//   w_i = relu(sigmoid(c (i - a L)) - sigmoid(c (i - b L)) - eps)     (masking.py:300-305)
// and the robustness at the trace start of "always positive over the window",
//   rho0_n = smooth_min_w(X[n, :])                                      (tape.py:360-391)
// (hard: min over the kept entries w > 0; LSE: -(1/tau) log sum w e^{-tau x};
// softmax: the w e^{-tau x}-weighted mean), then
//   loss(a, b) = mean_n relu(-rho0_n) + gamma (a - b).
// `grid_eval` (apps.py:326-335) evaluates it over an (a, b) grid one pair at a time;
// here one CTA handles one pair: the weights are formed in fp64 (as the reference
// does) into shared memory as log2 weights, each warp reduces whole rows, and the
// CTA writes the pair's loss.  With `dloss` the kernel also returns d loss / d a and
// d loss / d b (smooth modes; hard mode weights carry no gradient, tape.py:338-357),
// which `mine_interval`'s descent consumes.
#include <cfloat>

#include "kernels.cuh"

namespace stlg {

constexpr int MG_T = 256;

__device__ __forceinline__ double sigmoid_d(double z) {
  if (z >= 0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

template <int MODE>
__global__ void __launch_bounds__(MG_T) k_mining_grid(const float* __restrict__ x, long long n, int L,
                                                      long long rs, const double* __restrict__ pa,
                                                      const double* __restrict__ pb, double c, double eps,
                                                      float tau, double gamma, double* __restrict__ loss,
                                                      double* __restrict__ dloss) {
  extern __shared__ __align__(16) float msm[];
  float* lw = msm;       // log2 w_i (-inf where not kept)
  float* da = msm + L;   // d w_i / d a   (smooth modes with gradients)
  float* db = da + L;    // d w_i / d b
  __shared__ double red[3][MG_T / 32];
  const int pair = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double A = pa[pair], Bv = pb[pair];
  const bool want_grad = dloss != nullptr && MODE != M_HARD;
  int kept = 0;
  for (int i = tid; i < L; i += MG_T) {
    const double sl = sigmoid_d(c * ((double)i - A * (double)L));
    const double sh = sigmoid_d(c * ((double)i - Bv * (double)L));
    const double w = sl - sh - eps;
    lw[i] = w > 0.0 ? (float)log2(w) : -INFINITY;
    kept |= w > 0.0;
    if (want_grad) {  // relu active: dw/da = -c L sl (1 - sl), dw/db = c L sh (1 - sh)
      da[i] = w > 0.0 ? (float)(-c * (double)L * sl * (1.0 - sl)) : 0.f;
      db[i] = w > 0.0 ? (float)(c * (double)L * sh * (1.0 - sh)) : 0.f;
    }
  }
  if (!__syncthreads_or(kept)) {  // EmptyWindowError in the reference: reported as NaN
    if (tid == 0) {
      loss[pair] = __longlong_as_double(0x7ff8000000000000LL);
      if (dloss) dloss[2 * pair] = dloss[2 * pair + 1] = 0.0;
    }
    return;
  }
  const float tau2 = tau * 1.4426950408889634f, itau2 = 1.f / tau2;
  double acc = 0.0, ga = 0.0, gb = 0.0;
  for (long long row = warp; row < n; row += MG_T / 32) {
    const float* xr = x + row * rs;
    // max over the kept entries of y = -x (the reference's detached shift)
    float m = -INFINITY;
    for (int i = lane; i < L; i += 32)
      if (lw[i] > -INFINITY) m = fmaxf(m, -xr[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float rho;
    float s = 0.f, q = 0.f, sa = 0.f, sb = 0.f, qa = 0.f, qb = 0.f;
    if (MODE == M_HARD) {
      rho = -m;
    } else {
      for (int i = lane; i < L; i += 32) {
        const float l2w = lw[i];
        if (l2w > -INFINITY) {
          const float y = -xr[i];
          const float e = ex2f(fmaf(tau2, y - m, l2w));  // w e^{tau (y - m)}
          s += e;
          if (MODE == M_SOFT) q += e * (y - m);
          if (want_grad) {  // d/dw_i carries e^{tau (y - m)} without the weight itself
            const float en = ex2f(tau2 * (y - m));
            sa += en * da[i];
            sb += en * db[i];
            if (MODE == M_SOFT) {
              qa += en * (y - m) * da[i];
              qb += en * (y - m) * db[i];
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
        qa += __shfl_xor_sync(0xffffffffu, qa, o);
        qb += __shfl_xor_sync(0xffffffffu, qb, o);
      }
      const float smax = (MODE == M_LSE) ? fmaf(lg2f(s), itau2, m) : m + q / s;
      rho = -smax;
    }
    if (lane == 0 && -rho > 0.f) {  // relu(-rho) and its subgradient (tape relu: x > 0)
      acc += -(double)rho;
      if (want_grad) {
        // d(-rho)/dw_i = d smax/dw_i: LSE p_i / (tau w_i); softmax e_i (y_i - smax) / (s w_i)
        if (MODE == M_LSE) {
          ga += (double)(sa / (s * tau));
          gb += (double)(sb / (s * tau));
        } else {
          const float mu = q / s;  // smax - m
          ga += (double)((qa - mu * sa) / s);
          gb += (double)((qb - mu * sb) / s);
        }
      }
    }
  }
  if (lane == 0) {
    red[0][warp] = acc;
    red[1][warp] = ga;
    red[2][warp] = gb;
  }
  __syncthreads();
  if (tid == 0) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < MG_T / 32; ++w) {
      t0 += red[0][w];
      t1 += red[1][w];
      t2 += red[2][w];
    }
    loss[pair] = t0 / (double)n + gamma * (A - Bv);
    if (dloss) {
      dloss[2 * pair] = t1 / (double)n + gamma;
      dloss[2 * pair + 1] = t2 / (double)n - gamma;
    }
  }
}

cudaError_t launch_mining_grid(int mode, const float* x, long long n, int L, long long rs, const double* a,
                               const double* b, long long npairs, double c, double eps, float tau,
                               double gamma, double* loss, double* dloss, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  const size_t smem = (size_t)3 * L * sizeof(float);
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return;
    }
    kern<<<(unsigned)npairs, MG_T, smem, st>>>(x, n, L, rs, a, b, c, eps, tau, gamma, loss, dloss);
    e = cudaGetLastError();
  };
  if (mode == M_HARD) go(k_mining_grid<M_HARD>);
  else if (mode == M_LSE) go(k_mining_grid<M_LSE>);
  else go(k_mining_grid<M_SOFT>);
  count_launch();
  return e;
}

}  // namespace stlg
