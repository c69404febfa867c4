// multiset.cuh -- work-matrix evaluation of arbitrary CSR sets (K2, C5 path).
//
// f_j = sum_v (e0d[v] - min(e0d[v], min_{s in S_j} d(v, s))) / N   (batched.py:180-240)
//
// Only (v, s) pairs with d(v, s) < e0d(v) can contribute, and for most data
// they are rare.  So:
//   1. gather the member rows (K2a) and run the direct-form screen in FLAG mode
//      (k_screen<..., MODE 2>) with the accumulator seeded by -e0d32: every pair
//      that is *possibly* closer than e0 is appended; an unflagged pair is
//      certified to contribute exactly 0 (same bound as the Greedy direct rung);
//   2. flagged pairs get their exact fp64 term t = e0d - d64 (K2b, the same
//      operation sequence as the dense kernel), keyed by (set, point);
//   3. radix sort + reduce-by-key(max) gives per (set, point) the term
//      max_s max(0, e0d - d) = e0d - min(e0d, min_s d) bit for bit;
//   4. K2c sums each set's terms with *exactly* the dense reduction structure
//      (1024-point chunks, 4 points per thread in order, the fixed 256-thread
//      tree, chunks left to right) -- zero terms are exact no-ops -- so the
//      result is bit-identical to the dense kernel k_multiset: the empty set is
//      exactly 0.0 and the full set exactly the baseline.
// If the flag buffer overflows (dense contributions, e.g. huge sets), the host
// falls back to the dense kernel.
#pragma once
#include <cstdint>

#include "kernels.cuh"

namespace ebc {

// Mbuf[m] = V32 row idx[m] (padded rows beyond nnz stay zero); set_of[m] = j.
__global__ void k_gather_members(const float* __restrict__ V32, int pitch, const int64_t* __restrict__ idx,
                                 const int64_t* __restrict__ offsets, int64_t l, int64_t nnz,
                                 float* __restrict__ Mbuf, int* __restrict__ set_of) {
  const int64_t total = nnz * pitch;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / pitch;
    const int k = (int)(i - m * pitch);
    Mbuf[i] = V32[idx[m] * pitch + k];
    if (k == 0) {
      // set of member m: last j with offsets[j] <= m (binary search)
      int64_t lo = 0, hi = l;  // invariant offsets[lo] <= m < offsets[hi]
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (offsets[mid] <= m) lo = mid; else hi = mid;
      }
      set_of[m] = (int)lo;
    }
  }
}

// Exact fp64 terms of flagged pairs; key = set * n + v, non-contributing -> ~0.
template <typename T>
__global__ void k_flag_exact(const uint2* __restrict__ pairs, const int* __restrict__ count, int cap,
                             const T* __restrict__ V, int pitch, int d, const int64_t* __restrict__ idx,
                             const int* __restrict__ set_of, const double* __restrict__ e0d, int64_t n,
                             unsigned long long* __restrict__ keys, double* __restrict__ vals) {
  const int cnt = min(*count, cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const uint2 pr = pairs[i];
    const int64_t v = pr.x, m = pr.y;
    const T* row = V + v * pitch;
    const T* mem = V + idx[m] * pitch;
    double s = 0.0;
    for (int k = 0; k < d; ++k) {  // the dense kernel's exact operation sequence
      const double t = (double)row[k] - (double)__ldg(mem + k);
      s = fma(t, t, s);
    }
    const double base = e0d[v];
    const double mn = fmin(base, s);
    const double term = base - mn;
    keys[i] = term > 0.0 ? (unsigned long long)set_of[m] * (unsigned long long)n + (unsigned long long)v
                         : ~0ull;
    vals[i] = term;
  }
}

struct DMax {
  __device__ __forceinline__ double operator()(double a, double b) const { return a > b ? a : b; }
};

// One WARP per set: the dense chunk reduction over its (sparse) terms.
// block_sum_256's tree (level s: t < s adds t + s, s = 128 .. 1) is replayed by
// one warp: lane l holds the partials of threads l + 32 m (m = 0..7); levels
// 128/64/32 pair them inside the lane (m with m + 4, m + 2, m + 1), levels
// 16..1 are the shuffle-down steps.  Every tree node is the same single fp64
// add of the same two operands as in the block form, so each chunk sum -- and
// the set's left-to-right total -- is bit-identical to the dense kernel.
__global__ void __launch_bounds__(256) k_sparse_set_sum(const unsigned long long* __restrict__ ukeys,
                                                        const double* __restrict__ uvals,
                                                        const int* __restrict__ nruns, int64_t n, int64_t l,
                                                        double inv_n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= l) return;
  const int64_t R = *nruns;
  // [r0, r1): runs with key in [j n, (j + 1) n) (lanes 0 and 1 search, then broadcast)
  int64_t found = 0;
  if (lane < 2) {
    const unsigned long long target = (unsigned long long)(j + lane) * (unsigned long long)n;
    int64_t lo = 0, hi = R;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < target) lo = mid + 1; else hi = mid;
    }
    found = lo;
  }
  const int64_t r0 = __shfl_sync(0xffffffffu, found, 0), r1 = __shfl_sync(0xffffffffu, found, 1);
  const unsigned long long base = (unsigned long long)j * (unsigned long long)n;
  double total = 0.0;
  int64_t r = r0;
  while (r < r1) {
    const int64_t ch = (int64_t)(ukeys[r] - base) / RCH;
    // runs of this chunk: [r, re) (every lane walks the same runs)
    int64_t re = r;
    while (re < r1 && (int64_t)(ukeys[re] - base) / RCH == ch) ++re;
    // thread t's accumulator (points t + 256 i, i ascending) lives in lane t % 32, slot t / 32
    double v[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t q = r; q < re; ++q) {
      const int t = (int)(((int64_t)(ukeys[q] - base) - ch * RCH) % RED_THREADS);
      if ((t & 31) == lane) {
        const int m = t >> 5;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i == m) v[i] += uvals[q];
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) v[m] += v[m + 4];  // s = 128
#pragma unroll
    for (int m = 0; m < 2; ++m) v[m] += v[m + 2];  // s = 64
    v[0] += v[1];                                   // s = 32
    double x = v[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // s = 16 .. 1
      const double y = __shfl_down_sync(0xffffffffu, x, o);
      if (lane < o) x += y;
    }
    total += __shfl_sync(0xffffffffu, x, 0);
    r = re;
  }
  if (lane == 0) out[j] = total * inv_n;
}

}  // namespace ebc
