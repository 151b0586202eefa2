// lookback.cuh — deterministic carries for row scans split over CTAs (SURVEY §2's
// "single-pass suffix scan, decoupled look-back across time tiles").
//
// A row of n tiles is scanned by n CTAs.  Each CTA draws its (row, scan index s) from a
// ticket counter (an atomic in the slot region), so every tile it depends on belongs to a
// CTA that has already started — forward progress does not rest on the hardware's block
// dispatch order.  It stages and scans its own tile, publishes the tile aggregate, and
// then folds the published aggregates of tiles 0 .. s-1 in that fixed order.  There is no
// inclusive-prefix shortcut: the carry is the same expression the sequential one-CTA walk
// evaluated, so its bits do not depend on which tiles happened to finish first (the fp64
// run sums and LSE carries stay reproducible).  One 32-byte slot per (row, tile): word 0
// the flag (zeroed by the launcher before every launch), words 1..7 the payload.  Slot
// region layout: [ticket counter slot][row-major tile slots].
#pragma once

namespace stlg {

constexpr int LB_WORDS = 8;

// this CTA's ticket (0, 1, 2, ... in the order CTAs start), broadcast to every thread
__device__ __forceinline__ int lb_ticket(unsigned* counter) {
  __shared__ int tk;
  if (threadIdx.x == 0) tk = (int)atomicAdd(counter, 1u);
  __syncthreads();
  return tk;
}

__device__ __forceinline__ void lb_store_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned lb_load_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// one thread: payload words, then the flag (release orders them)
template <int N>
__device__ __forceinline__ void lb_publish(unsigned* slot, const unsigned (&w)[N]) {
  static_assert(N < LB_WORDS, "payload too large");
#pragma unroll
  for (int i = 0; i < N; ++i) reinterpret_cast<volatile unsigned*>(slot)[1 + i] = w[i];
  lb_store_release(slot, 1u);
}

// wait for a slot and read its payload (acquire orders the payload loads after the flag)
template <int N>
__device__ __forceinline__ void lb_wait(const unsigned* slot, unsigned (&w)[N]) {
  while (lb_load_acquire(slot) == 0u) __nanosleep(32);
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = reinterpret_cast<const volatile unsigned*>(slot)[1 + i];
}

// payload of the tiles 0 .. s-1 of a row into shared memory, one slot per thread
// (all flags polled concurrently); the caller folds them in order after a barrier
template <int N>
__device__ __forceinline__ void lb_gather(const unsigned* row_slots, int s, unsigned* sh) {
  for (int j = threadIdx.x; j < s; j += blockDim.x) {
    unsigned w[N];
    lb_wait<N>(row_slots + (size_t)j * LB_WORDS, w);
#pragma unroll
    for (int i = 0; i < N; ++i) sh[j * N + i] = w[i];
  }
}

// carry of tile s: fold(x, payload words) over the slots of tiles 0 .. s-1 in scan order,
// by thread 0 after a concurrent gather of up to 64 slots at a time; every thread gets it
template <int N, typename X, typename Fold>
__device__ __forceinline__ X lb_carry(const unsigned* row_slots, int s, X x, Fold&& fold) {
  __shared__ unsigned lbw[64 * N];
  __shared__ X lbx;
  for (int j0 = 0; j0 < s; j0 += 64) {
    const int n = min(64, s - j0);
    lb_gather<N>(row_slots + (size_t)j0 * LB_WORDS, n, lbw);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 0; j < n; ++j) x = fold(x, lbw + j * N);
    __syncthreads();
  }
  if (threadIdx.x == 0) lbx = x;
  __syncthreads();
  return lbx;
}

}  // namespace stlg
