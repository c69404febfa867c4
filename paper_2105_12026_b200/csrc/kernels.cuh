// kernels.cuh -- sm_100a kernels for the EBC Greedy / multiset hot path.
//
//   K0 k_init           d(v,e0) in fp64, cached minima, baseline partials      (ebc.py:72)
//   K1 k_screen         fused distance -> min(cm, .) -> sum over V, fp32 FFMA,  (batched.py:202-226
//                       with a per-candidate certified error bound               at the Greedy call site)
//   K3 k_finalize/k_window/k_refine/k_pick
//                       certified near-tie window, exact fp64 gains, argmax with (optimize.py:83-88)
//                       the reference tie window and lowest-index rule
//   K4 k_update         fold the chosen exemplar into cm64/cm32, f(S) in fp64    (new: cached-min)
//   K2 k_multiset       arbitrary CSR sets, fp64, work-matrix row sums           (batched.py:180-240,
//                                                                                 Alg. 2 batched.py:272-374)
//
// Determinism: no floating-point atomics.  Every sum over points uses the same
// fixed structure -- chunks of RCH points, a fixed 256-thread tree inside each
// chunk, then a left-to-right pass over chunks -- so a candidate's value never
// depends on its slot, on the launch shape or on how candidates are sharded
// across GPUs, and the empty set evaluates to exactly 0.0.
#pragma once
#include <cfloat>
#include <cuda_fp16.h>
#include <cstdint>

#include "ptx.cuh"

namespace ebc {

constexpr int RCH = 1024;         // points per reduction chunk
constexpr int RED_THREADS = 256;  // threads of every chunk-reduction block

// ---------------------------------------------------------------- reductions

// Fixed-tree sum over the 256 threads of a block; result valid in thread 0.
__device__ __forceinline__ double block_sum_256(double v, double* sbuf) {
  const int t = threadIdx.x;
  sbuf[t] = v;
  __syncthreads();
#pragma unroll
  for (int s = 128; s > 0; s >>= 1) {
    if (t < s) sbuf[t] += sbuf[t + s];
    __syncthreads();
  }
  double r = sbuf[0];
  __syncthreads();
  return r;
}

// Sequential left-to-right sum of chunk partials (one thread).  Loads go out
// 16 at a time ahead of their (still strictly ordered) adds: one memory latency
// per 16 partials instead of one per partial.
__device__ __forceinline__ double chunk_total(const double* part, int nchunks) {
  double s = 0.0;
  int c = 0;
  for (; c + 16 <= nchunks; c += 16) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __ldcg(part + c + i);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
  }
  for (; c < nchunks; ++c) s += __ldcg(part + c);
  return s;
}

// The same left-to-right sum by the last block of a grid: all threads stage
// the partials through shared memory (coalesced, one L2 round trip per 256),
// thread 0 adds them in order -- identical bits, no serial L2 latency chain.
// Called by every thread of the block; result valid in thread 0.
__device__ __forceinline__ double chunk_total_block(const double* part, int nchunks, double* sbuf) {
  double s = 0.0;
  for (int c0 = 0; c0 < nchunks; c0 += RED_THREADS) {
    const int m = min(RED_THREADS, nchunks - c0);
    if ((int)threadIdx.x < m) sbuf[threadIdx.x] = __ldcg(part + c0 + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < m; ++i) s += sbuf[i];
    __syncthreads();
  }
  return s;
}

// Order-preserving map of a double onto a signed 64-bit key (for atomicMax).
__device__ __forceinline__ long long dkey(double x) {
  long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double dkey_inv(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7fffffffffffffffLL));
}

// fp64 squared distance of stored row `row` (type T, `pitch` elements) to a
// candidate held in shared memory as fp64 -- sequential over dims.
// fp32 pre-test of an exact term max(0, cm - d64(v, c)): d32 = the fp32
// distance (fl(x - c) squared and summed with FMAs, all terms >= 0) is within
// (d + 3) 2^-24 of the exact one, so d32 (1 - (d + 4) 2^-23) > cm (1 + 2^-40)
// certifies d_exact > cm and hence d64 >= cm: the fp64 term is exactly +0.0
// (underflow and flushing only lower d32: never a false skip).  Kernels compute
// the fp64 sum only where this fails -- the same values, far fewer DFMAs.
__device__ __forceinline__ double far32_scale(int d) { return 1.0 - (double)(d + 4) * 0x1p-23; }
__device__ __forceinline__ bool far32(float d32, double ks, double cm) {
  // an overflowed fp32 sum proves nothing (cm may be beyond the fp32 range too)
  return d32 <= 3.0e38f && (double)d32 * ks > cm * (1.0 + 0x1p-40);
}

// Gram form of the same pre-test, one FFMA per coordinate: g = fl32 v.c (one
// sequential FFMA chain), nv / nc = fp32 |v|^2, |c|^2 (each within 2^-24
// relative of the exact norm), so |(nv + nc - 2 g) - d_exact| <= (d + 1) 2^-24
// (nv + nc) plus d 2^-149 per underflowed product; skip when the lower end still
// exceeds cm.  Overflow gives inf / NaN and never skips.
__device__ __forceinline__ bool far32_gram(float g, float nv, float nc, int d, double cm) {
  const double s2 = (double)nv + (double)nc;
  const double lo = s2 - 2.0 * (double)g - ((double)(d + 4) * 0x1p-24 * 1.01 * s2 + (double)(d + 4) * 0x1p-148);
  return lo > cm * (1.0 + 0x1p-40);
}

template <typename T>
__device__ __forceinline__ double dist64_row(const T* __restrict__ row, const double* cd, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = (double)row[k] - cd[k];
    s = fma(t, t, s);
  }
  return s;
}
// fp32 rows (16-byte aligned: the pitch is a multiple of 4): the same sequential
// operations, fed by 128-bit loads (a thread walks its own row; one LDG.128
// per 4 dims instead of 4 scalar loads -- K4 is HBM/latency bound).
__device__ __forceinline__ double dist64_row(const float* __restrict__ row, const double* cd, int d) {
  const float4* r4 = reinterpret_cast<const float4*>(row);
  double s = 0.0;
  int k = 0;
  for (; k + 4 <= d; k += 4) {
    const float4 x = __ldg(r4 + (k >> 2));
    double t = (double)x.x - cd[k];
    s = fma(t, t, s);
    t = (double)x.y - cd[k + 1];
    s = fma(t, t, s);
    t = (double)x.z - cd[k + 2];
    s = fma(t, t, s);
    t = (double)x.w - cd[k + 3];
    s = fma(t, t, s);
  }
  for (; k < d; ++k) {
    const double t = (double)row[k] - cd[k];
    s = fma(t, t, s);
  }
  return s;
}

// The 4 points a reduction thread owns (v0 + i * RED_THREADS, i = 0..3), their
// fp64 distances to one candidate computed as 4 interleaved chains: each chain is
// exactly dist64_row's operation sequence (bit-identical), but the 4 independent
// DFMA chains and row loads overlap (the single-chain form is latency-bound).
template <typename T>
__device__ __forceinline__ void dist64_rows4(const T* __restrict__ V, int pitch, int64_t v0, int64_t n,
                                             const double* cd, int d, double (&s)[4]) {
  const T* row[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t v = v0 + (int64_t)i * 256;
    row[i] = V + (v < n ? v : v0) * pitch;  // out-of-range points recompute row v0 (discarded)
    s[i] = 0.0;
  }
  int k = 0;
  if constexpr (sizeof(T) == 4) {
    for (; k + 4 <= d; k += 4) {
      float4 x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = __ldg(reinterpret_cast<const float4*>(row[i]) + (k >> 2));
      const double c0 = cd[k], c1 = cd[k + 1], c2 = cd[k + 2], c3 = cd[k + 3];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double t = (double)x[i].x - c0;
        s[i] = fma(t, t, s[i]);
        t = (double)x[i].y - c1;
        s[i] = fma(t, t, s[i]);
        t = (double)x[i].z - c2;
        s[i] = fma(t, t, s[i]);
        t = (double)x[i].w - c3;
        s[i] = fma(t, t, s[i]);
      }
    }
  }
  for (; k < d; ++k) {
    const double ck = cd[k];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double t = (double)row[i][k] - ck;
      s[i] = fma(t, t, s[i]);
    }
  }
}

// ---------------------------------------------------------------- per-point screen data

// pt[v] = {-cm32, tau, ip, kp}: the direct screen seeds its accumulator with
// -cm32 and uses tau = 2(d+8)u*cm32 as error quantum; the Gram screen seeds
// with ip = (cm32 - nv32)/2 and uses kp.
struct PtCoef {
  float tau_k;   // 2(d+8)u (1 + 2^-9)
  float gram_k;  // (d+4)u/2 (1 + 2^-10)
};

__device__ __forceinline__ float4 make_pt(float c32, float nv, PtCoef k) {
  return make_float4(-c32, k.tau_k * c32, (c32 - nv) * 0.5f, k.gram_k * (c32 + 2.f * nv));
}

// Tensor-screen seeds (screen_tc.cuh): per anchor a and point v,
// ip_a[v] = (cm32 - nva_a[v]) / 2 with nva_a[v] = |v - mu_a|^2 (fp64, rounded).
struct TcSeeds {
  float* ipa = nullptr;        // na x stride
  const float* nva = nullptr;  // na x stride
  int na = 0;
  int64_t stride = 0;
  // seeds folded into the MMA (one-product FP16 kinds): the origin
  // seed ip_0(v), scaled by s2 = s^2 and split into three FP16 parts, sits in K
  // columns d, d+1, d+2 of the point operand (UMMA canonical K-major layout,
  // kpad columns); the candidate operand holds 1 there
  __half* ops = nullptr;
  int kpad = 0;
  int d = 0;
  float s2 = 1.f;
};

__device__ __forceinline__ int64_t umma_off(int64_t v, int k, int kpad) {
  return (((v >> 3) * (kpad >> 3) + (k >> 3)) * 8 + (v & 7)) * 8 + (k & 7);
}

// X ~ p1 + p2 + p3 (each part the FP16 rounding of the remainder, |X| <= 2^14)
__device__ __forceinline__ void write_seed_parts(const TcSeeds& s, int64_t v, float x) {
  const __half p1 = __float2half_rn(x);
  const float r1 = x - __half2float(p1);  // exact (fp32 holds x - p1)
  const __half p2 = __float2half_rn(r1);
  const __half p3 = __float2half_rn(r1 - __half2float(p2));
  s.ops[umma_off(v, s.d, s.kpad)] = p1;
  s.ops[umma_off(v, s.d + 1, s.kpad)] = p2;
  s.ops[umma_off(v, s.d + 2, s.kpad)] = p3;
}

__device__ __forceinline__ void write_seeds(const TcSeeds& s, int64_t v, float cm32) {
  constexpr int NA_MAX = 32;
  if (s.na <= NA_MAX) {
    // all |v - mu_a|^2 loads in flight before the first store: one memory
    // latency per updated point instead of one per anchor
    float q[NA_MAX];
#pragma unroll
    for (int a = 0; a < NA_MAX; ++a)
      if (a < s.na) q[a] = __ldg(s.nva + a * s.stride + v);
#pragma unroll
    for (int a = 0; a < NA_MAX; ++a)
      if (a < s.na) s.ipa[a * s.stride + v] = (cm32 - q[a]) * 0.5f;
  } else {
    for (int a = 0; a < s.na; ++a) s.ipa[a * s.stride + v] = (cm32 - s.nva[a * s.stride + v]) * 0.5f;
  }
  if (s.ops) write_seed_parts(s, v, s.ipa[v] * s.s2);  // anchor 0 = the origin
}

// ---------------------------------------------------------------- K0: init

// Widen/pad the uploaded rows into the device layout (n_pad x pitch, zero pad).
template <typename S, typename D>
__global__ void k_pad(const S* __restrict__ src, int64_t n, int d, D* __restrict__ dst, int pitch) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = n * (int64_t)pitch;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = i / pitch;
    int k = (int)(i - v * pitch);
    dst[i] = k < d ? (D)(float)src[v * d + k] : (D)0;
  }
}
template <>
__global__ void k_pad<double, double>(const double* __restrict__ src, int64_t n, int d,
                                      double* __restrict__ dst, int pitch) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = n * (int64_t)pitch;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = i / pitch;
    int k = (int)(i - v * pitch);
    dst[i] = k < d ? src[v * d + k] : 0.0;
  }
}

// e0d[v] = d(v, e0) (fp64); nv32 = |v|^2; cm64 = e0d; pt; chunk partials of e0d.
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) k_init(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                      const double* __restrict__ e0, PtCoef pk,
                                                      double* __restrict__ e0d, double* __restrict__ cm64,
                                                      float* __restrict__ nv32, float4* __restrict__ pt,
                                                      double* __restrict__ part) {
  __shared__ double sbuf[RED_THREADS];
  __shared__ double se0[1024];
  for (int k = threadIdx.x; k < d && k < 1024; k += blockDim.x) se0[k] = e0[k];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RCH;
  double acc = 0.0;
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    int64_t v = base + threadIdx.x + (int64_t)i * RED_THREADS;
    if (v < n) {
      double t = d <= 1024 ? dist64_row(V + v * pitch, se0, d) : dist64_row(V + v * pitch, e0, d);
      e0d[v] = t;
      cm64[v] = t;
      double nv = 0.0;
      for (int k = 0; k < d; ++k) {
        const double x = (double)V[v * pitch + k];
        nv = fma(x, x, nv);
      }
      const float n32 = (float)nv;
      nv32[v] = n32;
      pt[v] = make_pt((float)t, n32, pk);
      acc += t;
    }
  }
  double s = block_sum_256(acc, sbuf);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Reset the cached minima to d(., e0) (ebc_reset / start of a Greedy run).
__global__ void k_reset(int64_t n, const double* __restrict__ e0d, const float* __restrict__ nv32, PtCoef pk,
                        double* __restrict__ cm64, float4* __restrict__ pt, unsigned char* __restrict__ selected,
                        int* __restrict__ sticky, TcSeeds seeds) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v == 0 && sticky) *sticky = 0;
  if (v < n) {
    double t = e0d[v];
    cm64[v] = t;
    pt[v] = make_pt((float)t, nv32[v], pk);
    if (seeds.ipa) write_seeds(seeds, v, (float)t);
    selected[v] = 0;
  }
}

// pt0[v] = screen data seeded with d(v, e0) (work-matrix flag screen).
__global__ void k_make_pt0(int64_t n, const double* __restrict__ e0d, const float* __restrict__ nv32, PtCoef pk,
                           float4* __restrict__ pt0) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) pt0[v] = make_pt((float)e0d[v], nv32[v], pk);
}

// max |x| over a float array (non-negative floats order like their bit patterns)
__global__ void k_absmax(const float* __restrict__ x, int64_t n, unsigned int* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(x[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

__global__ void k_set_int(int* __restrict__ p, int v) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *p = v;
}

__global__ void k_total(const double* __restrict__ part, int nchunks, double scale, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = chunk_total(part, nchunks) * scale;
}

// out = (sum of the chunk partials, left to right) / n -- ebc.py:43's division
__global__ void k_mean(const double* __restrict__ part, int nchunks, double n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = chunk_total(part, nchunks) / n;
}

// ---------------------------------------------------------------- K1: screen
//
// gain32[c] = sum_v max(0, cm32[v] - d32(v, c)) for a tile of candidates, with
// a certified bound e[c] such that |gain32 - gain_exact| <= e*infl + 8u*gain32.
//
// Layout: 256 threads = 8 warps as WP x WC = 2 x 4; inside a warp 8 lane-rows
// (points) x 4 lane-cols (candidates); each thread owns TP=4 points x TC=8
// candidates -> CTA tile = 64 points x 128 candidates.  The candidate tile is
// loaded once by the bulk-copy engine and stays in shared memory; V tiles
// (64 rows + their {-cm32, tau} pairs) stream through an mbarrier ring.
//
// Per pair the accumulator starts at -cm32[v], so after the d-dim FADD/FFMA
// chain it holds s = d32 - cm32 directly:  gain += max(-s, 0),
// err += (s < tau[v]) ? tau[v] : 0  with tau = 2(d+8)u*cm32.
// Tile geometry.  TC is fixed at 8 (the transposed butterfly below hands lane
// r the tile sum of candidate r); TP (points per thread), the warp grid and the
// ring depth are template parameters so several shapes can be instantiated.
template <int TP_, int WP_, int WC_, int STAGES_, int MINB_>
struct ScreenCfg {
  static constexpr int TP = TP_, TC = 8, LR = 8, LC = 4, WP = WP_, WC = WC_;
  static constexpr int STAGES = STAGES_, MINB = MINB_;
  static constexpr int NWARPS = WP * WC;
  static constexpr int THREADS = 32 * NWARPS;
  static constexpr int PT = WP * LR * TP;  // points per V tile
  static constexpr int CT = WC * LC * TC;  // candidates per CTA
  static size_t smem_bytes(int pitch) {
    size_t cand = (size_t)CT * pitch * sizeof(float);
    size_t stage = (size_t)PT * pitch * sizeof(float) + (size_t)PT * sizeof(float4);
    size_t ring = STAGES * stage;
    size_t red = (size_t)WP * CT * (sizeof(double) + sizeof(float));
    if (ring < red) ring = red;
    return cand + ring + (2 * STAGES + 1) * sizeof(uint64_t) + STAGES * sizeof(int) + 16;
  }
};

// Transposed butterfly over the 8 lane-rows (lane bits 0..2): on return lane r
// holds sum over the 8 rows of x[r].  Fixed order -> deterministic.
__device__ __forceinline__ float rowsum8_transposed(const float (&x)[8], int r) {
  float h[4];
  const bool up4 = (r & 4) != 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float send = up4 ? x[j] : x[j + 4];
    float keep = up4 ? x[j + 4] : x[j];
    h[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  float h2[2];
  const bool up2 = (r & 2) != 0;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float send = up2 ? h[j] : h[j + 2];
    float keep = up2 ? h[j + 2] : h[j];
    h2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  const bool up1 = (r & 1) != 0;
  float send = up1 ? h2[0] : h2[1];
  float keep = up1 ? h2[1] : h2[0];
  return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

// MODE 0: direct-form gains; 1: Gram-form gains; 2: direct-form *flags* -- append
// every (point, candidate) pair that is possibly closer than the seed distance
// (K2 work-matrix path: candidates are set members, seed = d(v, e0)).
struct FlagOut {
  uint2* pairs;      // (point, candidate row) of possibly-contributing pairs
  int* count;        // appended pairs (may exceed cap: overflow -> caller falls back)
  int cap;
  int64_t npoints;   // valid point rows
  int64_t ncands;    // valid candidate rows
};

template <class Cfg, int MODE, int PITCH>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    k_screen(const float* __restrict__ V, const float4* __restrict__ pt, int pitch_rt, int d4, int64_t cand0,
             int ntiles, int tiles_per_split, double* __restrict__ part_g, float* __restrict__ part_e,
             int64_t part_stride, float gram_kc, const int* __restrict__ level_now, int level,
             const float* __restrict__ Vc, FlagOut fo) {
  constexpr bool GRAM = MODE == 1;
  constexpr bool FLAG = MODE == 2;
  if (level_now && *level_now != level) return;  // adaptive screen: not this level's turn
  // PITCH != 0: compile-time row pitch -> every LDS address is base + immediate
  const int pitch = PITCH ? PITCH : pitch_rt;
  constexpr int TP = Cfg::TP, TC = Cfg::TC, LR = Cfg::LR, LC = Cfg::LC, WP = Cfg::WP;
  constexpr int STAGES = Cfg::STAGES, NWARPS = Cfg::NWARPS, THREADS = Cfg::THREADS;
  constexpr int PT_ = Cfg::PT, CT_ = Cfg::CT;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wp = warp % WP, wc = warp / WP;
  const int r = lane & 7, q = lane >> 3;

  const size_t cand_bytes = (size_t)CT_ * pitch * sizeof(float);
  const size_t vt_bytes = (size_t)PT_ * pitch * sizeof(float);
  const size_t pt_bytes = (size_t)PT_ * sizeof(float4);
  float* cs = reinterpret_cast<float*>(smem);
  unsigned char* stage_base = smem + cand_bytes;
  const size_t stage_bytes = vt_bytes + pt_bytes;
  size_t ring_bytes = STAGES * stage_bytes;
  const size_t red_bytes = (size_t)WP * CT_ * (sizeof(double) + sizeof(float));
  if (ring_bytes < red_bytes) ring_bytes = red_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_base + ring_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* cbar = empty + STAGES;
  int* relcnt = reinterpret_cast<int*>(cbar + 1);

  const int t0 = blockIdx.y * tiles_per_split;
  const int t1 = min(ntiles, t0 + tiles_per_split);
  const int nt = t1 - t0;
  const int64_t crow = cand0 + (int64_t)blockIdx.x * CT_;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], THREADS);
      relcnt[s] = 0;
    }
    mbar_init(cbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(cbar, (uint32_t)cand_bytes);
    bulk_g2s(cs, (Vc ? Vc : V) + crow * pitch, (uint32_t)cand_bytes, cbar);
    for (int s = 0; s < STAGES && s < nt; ++s) {
      unsigned char* st = stage_base + s * stage_bytes;
      const int64_t prow = (int64_t)(t0 + s) * PT_;
      mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
      bulk_g2s(st, V + prow * pitch, (uint32_t)vt_bytes, &full[s]);
      bulk_g2s(st + vt_bytes, pt + prow, (uint32_t)pt_bytes, &full[s]);
    }
  }

  float g[TC], e[TC];
#pragma unroll
  for (int j = 0; j < TC; ++j) { g[j] = 0.f; e[j] = 0.f; }
  double g64 = 0.0;  // this lane's fp64 total for candidate j == r (after transposed reduce)

  const float* crow_s[TC];
#pragma unroll
  for (int j = 0; j < TC; ++j) crow_s[j] = cs + (wc * (LC * TC) + q + LC * j) * pitch;

  mbar_wait(cbar, 0);
  // Gram form: per-candidate |c|^2 (fp32, sequential -- covered by kc), the
  // accumulator seed half -|c|^2/2 and the error quantum kc.
  float ic[TC], kc[TC], cnt[TC];
#pragma unroll
  for (int j = 0; j < TC; ++j) {
    ic[j] = 0.f;
    kc[j] = 0.f;
    cnt[j] = 0.f;
  }
  if (GRAM) {
#pragma unroll
    for (int j = 0; j < TC; ++j) {
      float nc = 0.f;
      for (int k4 = 0; k4 < d4; ++k4) {
        const float4 b = *reinterpret_cast<const float4*>(crow_s[j] + 4 * k4);
        nc = fmaf(b.x, b.x, nc);
        nc = fmaf(b.y, b.y, nc);
        nc = fmaf(b.z, b.z, nc);
        nc = fmaf(b.w, b.w, nc);
      }
      ic[j] = -0.5f * nc;
      kc[j] = gram_kc * nc;
    }
  }
  __syncthreads();
  // Swap adjacent dims of the resident candidate tile: an LDS.128 lands vector
  // component j in a register of parity j%2, so pairing v_k (even register)
  // with c_k now stored in the odd slot makes every FADD read one even and one
  // odd register -- no register-bank conflict (ncu: dispatch stalls).
  {
    float2* c2 = reinterpret_cast<float2*>(cs);
    const int total2 = CT_ * pitch / 2;
    for (int i = tid; i < total2; i += THREADS) {
      const float2 x = c2[i];
      c2[i] = make_float2(x.y, x.x);
    }
  }
  __syncthreads();

  for (int it = 0; it < nt; ++it) {
    const int s = it % STAGES;
    const uint32_t ph = (it / STAGES) & 1;
    mbar_wait(&full[s], ph);
    const float* vs = reinterpret_cast<const float*>(stage_base + s * stage_bytes);
    const float4* ps = reinterpret_cast<const float4*>(stage_base + s * stage_bytes + vt_bytes);

    float acc[TP][TC];
    float tau[TP];
    const float* vrow[TP];
#pragma unroll
    for (int i = 0; i < TP; ++i) {
      const int p = wp * (LR * TP) + r + LR * i;
      const float4 pp = ps[p];
      tau[i] = GRAM ? pp.w : pp.y;
      vrow[i] = vs + p * pitch;
#pragma unroll
      for (int j = 0; j < TC; ++j) acc[i][j] = GRAM ? pp.z + ic[j] : pp.x;
    }
#pragma unroll(TP >= 8 ? 1 : 2)
    for (int k4 = 0; k4 < d4; ++k4) {
      float4 a[TP], b[TC];
#pragma unroll
      for (int i = 0; i < TP; ++i) a[i] = *reinterpret_cast<const float4*>(vrow[i] + 4 * k4);
#pragma unroll
      for (int j = 0; j < TC; ++j) b[j] = *reinterpret_cast<const float4*>(crow_s[j] + 4 * k4);
      // b holds (c_{k+1}, c_k, c_{k+3}, c_{k+2}) -- see the swap above
      if (GRAM) {
        // component-outer order: each a[i].comp feeds 8 consecutive FFMAs in
        // the same operand slot (operand-reuse cache), so only b and acc are
        // read from the register banks
#pragma unroll
        for (int i = 0; i < TP; ++i) {
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = fmaf(a[i].x, b[j].y, acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < TP; ++i) {
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = fmaf(a[i].y, b[j].x, acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < TP; ++i) {
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = fmaf(a[i].z, b[j].w, acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < TP; ++i) {
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = fmaf(a[i].w, b[j].z, acc[i][j]);
        }
      }
#pragma unroll
      for (int i = 0; i < TP; ++i) {
#pragma unroll
        for (int j = 0; j < TC; ++j) {
          if (!GRAM) {
            float t;
            t = a[i].x - b[j].y; acc[i][j] = fmaf(t, t, acc[i][j]);
            t = a[i].y - b[j].x; acc[i][j] = fmaf(t, t, acc[i][j]);
            t = a[i].z - b[j].w; acc[i][j] = fmaf(t, t, acc[i][j]);
            t = a[i].w - b[j].z; acc[i][j] = fmaf(t, t, acc[i][j]);
          }
        }
      }
    }
    // Stage consumed (every LDS result has been used).  Each warp arrives on
    // the stage's `empty` mbarrier; the last warp to release it (smem counter)
    // waits on that barrier -- already complete, so no stall -- and refills the
    // stage with tile it + STAGES.  No warp ever waits for another warp's
    // progress, and the mbarrier gives the WAR ordering against the bulk copy.
    mbar_arrive(&empty[s]);  // every reading thread arrives (count = THREADS)
    __syncwarp();
    if (lane == 0) {
      const int old = atomicAdd(&relcnt[s], 1);
      if (old == NWARPS - 1) {
        relcnt[s] = 0;
        mbar_wait(&empty[s], ph);
        if (it + STAGES < nt) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          unsigned char* st = stage_base + s * stage_bytes;
          const int64_t prow = (int64_t)(t0 + it + STAGES) * PT_;
          mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
          bulk_g2s(st, V + prow * pitch, (uint32_t)vt_bytes, &full[s]);
          bulk_g2s(st + vt_bytes, pt + prow, (uint32_t)pt_bytes, &full[s]);
        }
      }
    }
    __syncwarp();

    // epilogue.  direct: acc = d32 - cm32;  Gram: acc = (cm - |v|^2 - |c|^2)/2 + v.c = t/2
    if (FLAG) {
#pragma unroll
      for (int i = 0; i < TP; ++i) {
#pragma unroll
        for (int j = 0; j < TC; ++j) {
          // rare: possibly closer than e0.  + 2^-100: an absolute floor for
          // pairs whose fp32 terms underflow (points within ~1e-15 of e0)
          if (acc[i][j] < tau[i] + 0x1p-100f) {
            const int64_t v = (int64_t)(t0 + it) * PT_ + wp * (LR * TP) + r + LR * i;
            const int64_t m = crow + wc * (LC * TC) + q + LC * j;
            if (v < fo.npoints && m < fo.ncands) {
              const int slot = atomicAdd(fo.count, 1);
              if (slot < fo.cap) fo.pairs[slot] = make_uint2((unsigned)v, (unsigned)m);
            }
          }
        }
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < TP; ++i) {
#pragma unroll
      for (int j = 0; j < TC; ++j) {
        const float sv = acc[i][j];
        if (GRAM) {
          g[j] += fmaxf(sv, 0.f);
          const float f = (sv + tau[i] > -kc[j]) ? 1.f : 0.f;
          e[j] = fmaf(f, tau[i], e[j]);
          cnt[j] += f;
        } else {
          g[j] += fmaxf(-sv, 0.f);
          e[j] = fmaf(sv < tau[i] ? 1.f : 0.f, tau[i], e[j]);
        }
      }
    }
    // fold this tile's fp32 gains into fp64 (lane r: candidate j = r)
    g64 += (double)rowsum8_transposed(g, r);
#pragma unroll
    for (int j = 0; j < TC; ++j) g[j] = 0.f;
  }

  if (FLAG) return;
  // error bound: same transposed reduce in fp32 (covered by the inflation factor)
  if (GRAM) {
#pragma unroll
    for (int j = 0; j < TC; ++j) e[j] = fmaf(kc[j], cnt[j], e[j]);
  }
  const float etot = rowsum8_transposed(e, r);
  // lane (r, q) of warp (wp, wc) now holds candidate  wc*32 + q + 4*r
  __syncthreads();  // all stages idle: reuse the ring for the cross-warp combine
  double* rg = reinterpret_cast<double*>(stage_base);
  float* re = reinterpret_cast<float*>(stage_base + WP * CT_ * sizeof(double));
  const int cl = wc * (LC * TC) + q + LC * r;
  rg[wp * CT_ + cl] = g64;
  re[wp * CT_ + cl] = etot;
  __syncthreads();
  if (tid < CT_) {
    double gs = 0.0;
    float es = 0.f;
#pragma unroll
    for (int w = 0; w < WP; ++w) {
      gs += rg[w * CT_ + tid];
      es += re[w * CT_ + tid];
    }
    const int64_t c = crow + tid;
    part_g[blockIdx.y * part_stride + c] = gs;
    part_e[blockIdx.y * part_stride + c] = es;
  }
}

// Instantiated shapes (selected at run time, EBC200_SCREEN overrides):
//   A: 4x8 per thread, 2 CTAs/SM, 64 pts x 128 cands, 2-stage ring
//   B: 8x8 per thread, 1 CTA/SM, 128 pts x 128 cands, 3-stage ring
using ScreenA = ScreenCfg<4, 2, 4, 2, 2>;
using ScreenA4 = ScreenCfg<4, 2, 4, 4, 2>;
using ScreenB = ScreenCfg<8, 2, 4, 3, 1>;

// ---------------------------------------------------------------- K3: window + refine + pick

// Combine the split partials, form the certified interval [lb, ub] and fold the
// block's largest lower bound into *maxlb (order-independent atomicMax).
__global__ void k_finalize(int64_t c0, int64_t c1, int nsplit, const double* __restrict__ part_g,
                           const float* __restrict__ part_e, int64_t part_stride, double einfl, double gcoef,
                           double gscale, const unsigned char* __restrict__ selected, double* __restrict__ ub,
                           long long* __restrict__ maxlb, const int* __restrict__ level_now, int level,
                           int ub_only = 0, const double* __restrict__ part_a = nullptr,
                           const unsigned char* __restrict__ bflag = nullptr, double* __restrict__ ubp = nullptr) {
  if (level_now && *level_now != level) return;
  __shared__ long long smax[256];
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  long long key = dkey(-INFINITY);
  // lazy step (bflag set): only the flagged 128-candidate blocks were screened;
  // the others hold stale partials and are out of the window (k_lazy_mark2)
  if (c < c1 && bflag && !bflag[(c - c0) >> 7]) {
    ub[c - c0] = -INFINITY;
  } else if (c < c1) {
    double g = 0.0, e = 0.0;
    for (int s = 0; s < nsplit; ++s) {
      g += part_g[s * part_stride + c];
      e += (double)part_e[s * part_stride + c];
    }
    g *= gscale;
    e *= gscale;
    double eps = e * einfl + gcoef * g + 1e-300;
    if (part_a) {  // all-positive tiles (k_screen_agg): certified upper bounds already
      double ga = 0.0;
      for (int s = 0; s < nsplit; ++s) ga += part_a[s * part_stride + c];
      ga *= gscale;
      g += ga;
      eps += 1e-12 * fabs(ga);
    }
    if (selected[c]) {
      ub[c - c0] = -INFINITY;
    } else {
      ub[c - c0] = g + eps;
      key = dkey(fmax(g - eps, 0.0));
      if (ubp) ubp[c - c0] = fmin(ubp[c - c0], g + eps);  // both bound the current gain
    }
  }
  smax[threadIdx.x] = key;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) smax[threadIdx.x] = max(smax[threadIdx.x], smax[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0 && !ub_only) atomicMax(maxlb, smax[0]);
}

// Upper-bound-only screens (the tensor rung: its partials are already sums of
// max(a + kq, 0), certified upper bounds with no error count): the window
// threshold is the EXACT gain of the candidate with the largest bound, which is
// a valid lower bound on the top gain.  Step 1: that candidate (lowest index
// among equal bounds).
__device__ __forceinline__ bool ub_better(double v, long long i, double bv, long long bi) {
  return v > bv || (v == bv && i < bi);
}

// Grid-wide: every block reduces a strided share of the candidates to its
// (largest bound, lowest index) pair in part/pidx, the last block to finish
// reduces those (any order gives the same pair: the comparison is a total order).
__global__ void __launch_bounds__(256) k_argmax_ub(int64_t c0, int64_t c1, const double* __restrict__ ub,
                                                   int64_t* __restrict__ topc, double* __restrict__ part,
                                                   unsigned int* __restrict__ counter,
                                                   const int* __restrict__ level_now, int level,
                                                   const unsigned char* __restrict__ selected = nullptr) {
  if (level_now && *level_now != level) return;
  __shared__ double sv[256];
  __shared__ long long si[256];
  __shared__ bool last;
  long long* pidx = reinterpret_cast<long long*>(part + gridDim.x);
  double bv = -INFINITY;
  long long bi = LLONG_MAX;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < c1; c += stride) {
    const double u = (selected && selected[c]) ? -INFINITY : ub[c - c0];
    if (u > bv) {  // ascending c per thread: the first maximum is the lowest index
      bv = u;
      bi = c;
    }
  }
  auto block_reduce = [&]() {
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s && ub_better(sv[threadIdx.x + s], si[threadIdx.x + s], sv[threadIdx.x], si[threadIdx.x])) {
        sv[threadIdx.x] = sv[threadIdx.x + s];
        si[threadIdx.x] = si[threadIdx.x + s];
      }
      __syncthreads();
    }
  };
  block_reduce();
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sv[0];
    pidx[blockIdx.x] = si[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  bv = -INFINITY;
  bi = LLONG_MAX;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const double v = __ldcg(part + b);
    const long long i = __ldcg(pidx + b);
    if (ub_better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
  __syncthreads();
  block_reduce();
  if (threadIdx.x == 0) {
    *topc = (sv[0] > -INFINITY) ? si[0] : -1;
    *counter = 0u;
  }
}

// Step 2: exact fp64 gain of topc, sum_v max(0, cm(v) - d64(v, c)) in chunk
// partials; the last block writes it as the window's lower bound (maxlb key).
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) k_gain_top(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                          const double* __restrict__ cm64,
                                                          const int64_t* __restrict__ topc,
                                                          double* __restrict__ part, unsigned int* __restrict__ counter,
                                                          long long* __restrict__ maxlb,
                                                          const int* __restrict__ level_now, int level) {
  if (level_now && *level_now != level) return;
  extern __shared__ double cd[];
  __shared__ double sbuf[RED_THREADS];
  __shared__ bool last;
  const int64_t s = *topc;
  if (s >= 0)
    for (int k = threadIdx.x; k < d; k += blockDim.x) cd[k] = (double)V[s * pitch + k];
  __syncthreads();
  double acc = 0.0;
  if (s >= 0) {
    // one point per thread, RED_THREADS points per block (a threshold, not a
    // reported value: its summation structure is free, only deterministic)
    const int64_t v = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x;
    if (v < n) {
      const double t = cm64[v] - dist64_row(V + v * pitch, cd, d);
      acc = t > 0.0 ? t : 0.0;
    }
  }
  const double bs = block_sum_256(acc, sbuf);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = bs;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const double tot = chunk_total_block(part, gridDim.x, sbuf);
    if (threadIdx.x == 0) {
      // max with the bound already there (0 after the step's reset, or the lazy
      // prologue's exact gain of the best stale bound): both are lower bounds
      *maxlb = max(*maxlb, dkey(tot));
      *counter = 0u;
    }
  }
}

// W = {c : ub_c >= max lb - margin}  (append order is irrelevant: the pick is by
// exact value and lowest index).
__global__ void k_window(int64_t c0, int64_t c1, const double* __restrict__ ub, const long long* __restrict__ maxlb,
                         double margin, int* __restrict__ wcount, int64_t* __restrict__ wlist,
                         const int* __restrict__ level_now, int level) {
  if (level_now && *level_now != level) return;
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < c1) {
    const double thr = dkey_inv(*maxlb) - margin;
    const double u = ub[c - c0];
    if (u >= thr && u > -INFINITY) {
      int slot = atomicAdd(wcount, 1);
      wlist[slot] = c;
    }
  }
}

// Adaptive screen: the screens form a ladder of decreasing speed and
// increasing precision (0 tensor-core Gram, 1 FFMA Gram, 2 direct).  After the
// pass of `level`, a window wider than `cap` moves the run to level + 1 for the
// rest of the run and clears the window state for the next pass.
__global__ void k_adapt(int* __restrict__ wcount, long long* __restrict__ maxlb, int cap, int* __restrict__ level_now,
                        int level) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (*level_now == level && *wcount > cap) {
      level_now[0] = level + 1;
      level_now[1] = level + 1;  // the run's rung (level_now[0] gates this step's kernels)
      *wcount = 0;
      *maxlb = 0;
    }
  }
}

// Every candidate of the screen range is in W (FP64 storage: no fp32 screen).
__global__ void k_window_all(int64_t c0, int64_t c1, const unsigned char* __restrict__ selected,
                             int* __restrict__ wcount, int64_t* __restrict__ wlist) {
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < c1 && !selected[c]) {
    int slot = atomicAdd(wcount, 1);
    wlist[slot] = c;
  }
}

// ---------------------------------------------------------------- threshold sieves (optimize.py:140-197)
// Every live sieve r keeps its cached minima cm_r(v) = min over S_r u {e0} of
// d64(v, .) (N doubles per slot), so a streamed element e costs one distance
// pass d64(., e) shared by all sieves plus one min/sum pass per sieve, instead
// of re-evaluating every member of every sieve.  The value of S_r u {e} is
//   sum_v (e0d(v) - min(cm_r(v), d(v, e))) / N
// with exactly k_multiset's per-point operations (fmin is exact and order-free)
// and reduction (4 points per thread in order, block_sum_256, chunk_total,
// x 1/N), so it is bit-identical to evaluating the set on the work-matrix path.

// Per point: reset the reset slots to S = {} (cm = e0d), fold commit_e into the
// commit slots, and d_e(v) = d64(v, e) for the evaluation.
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) k_sieve_points(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                              const double* __restrict__ e0d,
                                                              double* __restrict__ cm, int64_t cstride,
                                                              int64_t commit_e, const int* __restrict__ slots,
                                                              int n_commit, int n_reset, int64_t e,
                                                              double* __restrict__ de) {
  extern __shared__ double rows[];  // commit row, then e's row (fp64)
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    rows[k] = commit_e >= 0 ? (double)V[commit_e * pitch + k] : 0.0;
    rows[d + k] = e >= 0 ? (double)V[e * pitch + k] : 0.0;
  }
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  // resets first: a sieve created at the previous element may also have admitted it
  if (n_reset > 0) {
    const double b = e0d[v];
    for (int q = 0; q < n_reset; ++q) cm[(int64_t)slots[n_commit + q] * cstride + v] = b;
  }
  if (commit_e >= 0 && n_commit > 0) {
    const double dc = dist64_row(V + v * pitch, rows, d);
    for (int q = 0; q < n_commit; ++q) {
      double* c = cm + (int64_t)slots[q] * cstride + v;
      *c = fmin(*c, dc);
    }
  }
  if (e >= 0) de[v] = dist64_row(V + v * pitch, rows + d, d);
}

// part[s][chunk] for the evaluation slots (s = 0: the singleton {e}; s >= 1:
// S_r u {e} of slot eval[s - 1]), 8 per block row.
__global__ void __launch_bounds__(RED_THREADS) k_sieve_sums(int64_t n, const double* __restrict__ e0d,
                                                            const double* __restrict__ cm, int64_t cstride,
                                                            const double* __restrict__ de,
                                                            const int* __restrict__ eval, int n_eval, int nchunks,
                                                            double* __restrict__ part) {
  __shared__ double sbuf[RED_THREADS];
  const int ch = blockIdx.x;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  const int s0 = blockIdx.y * 8;
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    const int64_t v = (int64_t)ch * RCH + threadIdx.x + (int64_t)i * RED_THREADS;
    if (v < n) {
      const double base = e0d[v], dv = de[v];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int sidx = s0 + q;
        if (sidx <= n_eval) {
          const double c = sidx == 0 ? base : cm[(int64_t)eval[sidx - 1] * cstride + v];
          acc[q] += base - fmin(c, dv);
        }
      }
    }
  }
#pragma unroll 1
  for (int q = 0; q < 8; ++q) {
    if (s0 + q > n_eval) break;  // block-uniform
    const double bs = block_sum_256(acc[q], sbuf);
    if (threadIdx.x == 0) part[(int64_t)(s0 + q) * nchunks + ch] = bs;
  }
}

// ---------------------------------------------------------------- k-medoids loss (ebc.py:21-43)
// mins[v] = min over the explicit representatives [r0, r1) of the exact fp64
// direct distance (core.py:236-251), folded into the running minimum of earlier
// representative chunks (first chunk: from +inf, ebc.py:42 initial=np.inf).
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) k_kmed_min(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                          const double* __restrict__ reps, int r0, int r1,
                                                          double* __restrict__ mins, int first) {
  extern __shared__ double sr[];  // (r1 - r0) x d
  const int nr = r1 - r0;
  for (int i = threadIdx.x; i < nr * d; i += blockDim.x) sr[i] = reps[(int64_t)r0 * d + i];
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double m = first ? INFINITY : mins[v];
  for (int r = 0; r < nr; ++r) m = fmin(m, dist64_row(V + v * pitch, sr + (int64_t)r * d, d));
  mins[v] = m;
}

// part[chunk] = fixed-order sum of x over the chunk (the k_init structure:
// RCH points per block, RCH / RED_THREADS points per thread in order, the
// fixed 256-thread tree); k_total then adds the chunks left to right.
__global__ void __launch_bounds__(RED_THREADS) k_sum_chunks(const double* __restrict__ x, int64_t n,
                                                            double* __restrict__ part) {
  __shared__ double sbuf[RED_THREADS];
  const int64_t base = (int64_t)blockIdx.x * RCH;
  double acc = 0.0;
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    const int64_t v = base + threadIdx.x + (int64_t)i * RED_THREADS;
    if (v < n) acc += x[v];
  }
  const double s = block_sum_256(acc, sbuf);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ---------------------------------------------------------------- lazy Greedy (DESIGN.md §4 "Lazy steps")
// f is monotone submodular, so a candidate's gain can only shrink as S grows:
// gain_{s+1}(c) = sum_v max(0, cm_{s+1}(v) - d(v, c)) with cm only decreasing,
// and the computed fp64 sums inherit it term by term (every term is monotone in
// cm, fixed-order rounding is monotone).  ubp[c] keeps the tightest bound seen
// for c: the screen's certified upper bound (k_finalize) or its exact fp64
// gain (k_pick).  A later step needs to look only at the STALE candidates
//   ubp[c] >= lb - margin - 1e-9 |lb|,   lb = a current exact gain (below),
// every other candidate is out of the reference's tie window for certain
// (the same margin as k_window plus a rounding allowance for the different
// summation orders of the exact sums).  The lower bound comes from refining
// the RW best stale bounds first (k_lazy_topk); k_lazy_mark2 lists the stale
// set and flags its 128-candidate blocks; k_lazy_plan2 picks the mode.

__global__ void k_fill_f64(double* __restrict__ p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

constexpr int RW = 8;  // refine window group (k_refine): candidates sharing each V row read

// Lazy fast path: the LB (<= RW) candidates with the largest stale bounds
// (ubp descending, index ascending; selected ones skipped) are refined first.
// Their best exact gain is the step's lower bound lb; the stale set is a
// prefix of this order, so if the best bound OUTSIDE the batch (ub_next) is
// already below the stale threshold, the batch holds the whole stale set and
// the step is decided by that one refine (C2: almost every step after the
// first).  Grid-wide top-(LB+1): per-thread sorted lists, warp merges by
// shuffles, the last block merges the blocks' lists ((value, index) is a
// total order, so any merge order gives the same result).
constexpr int LB_MAX = RW;
constexpr int TK = LB_MAX + 1;  // entries kept per list: the batch + the best outside it
// (bound, index) as one 64-bit key: the bound rounded UP to fp32 in the high word
// (non-negative floats order like their bits), ~index in the low word (lower
// index wins ties), 0 = empty.  Rounding up keeps the batch test conservative:
// every candidate outside the batch has ubp <= its key's bound <= ub_next.
__device__ __forceinline__ unsigned long long top_key(double ub, int64_t c) {
  const float f = __double2float_ru(fmax(ub, 0.0));
  return ((unsigned long long)__float_as_uint(f) << 32) | (unsigned long long)(0xFFFFFFFFu - (unsigned)c);
}
__device__ __forceinline__ void top_insert(unsigned long long (&l)[TK], unsigned long long k) {
  if (k <= l[TK - 1]) return;
#pragma unroll
  for (int p = TK - 1; p > 0; --p) l[p] = k > l[p - 1] ? l[p - 1] : (k > l[p] ? k : l[p]);
  if (k > l[0]) l[0] = k;
}
// TK rounds of a warp max over the lanes' list heads (keys are unique); the
// winner lane pops.  Lane 0 writes the warp's sorted top-TK to out.
__device__ __forceinline__ void warp_topk(unsigned long long (&l)[TK], unsigned long long* out) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int r = 0; r < TK; ++r) {
    // the 64-bit max as two 32-bit warp reductions (high word, then the low
    // word among the lanes holding it)
    const unsigned hi = (unsigned)(l[0] >> 32), lo = (unsigned)l[0];
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const unsigned long long b = ((unsigned long long)mh << 32) | ml;
    if (lane == 0) out[r] = b;
    if (b != 0ull && l[0] == b) {
#pragma unroll
      for (int p = 0; p < TK - 1; ++p) l[p] = l[p + 1];
      l[TK - 1] = 0ull;
    }
  }
}

#ifdef EBC200_TRACE
// Development trace (tools/ub_trace.py, -DEBC200_TRACE builds only): per step,
// globaltimer stamps of the fused update's phases, min/max over blocks.
__device__ unsigned long long g_ub_trace[64][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_ub_blk[8192][4];
__device__ unsigned long long g_tk_trace[64][4];  // k_lazy_topk: start (min), scan done (max), last block, end
#define TK_TRACE_MIN(step, i) \
  if (threadIdx.x == 0 && step >= 0 && step < 64) atomicMin(&g_tk_trace[step][i], gtimer())
#define TK_TRACE_MAX(step, i) \
  if (threadIdx.x == 0 && step >= 0 && step < 64) atomicMax(&g_tk_trace[step][i], gtimer())  // one step's per-block stamps (step == 10)
#define UB_TRACE_BLK(step, i) \
  if (threadIdx.x == 0 && step == 10 && blockIdx.x < 8192) g_ub_blk[blockIdx.x][i] = gtimer()
#define UB_TRACE_MIN(step, i) \
  if (threadIdx.x == 0 && step < 64) atomicMin(&g_ub_trace[step][i], gtimer())
#define UB_TRACE_MAX(step, i) \
  if (threadIdx.x == 0 && step < 64) atomicMax(&g_ub_trace[step][i], gtimer())
#else
#define TK_TRACE_MIN(step, i)
#define TK_TRACE_MAX(step, i)
#define UB_TRACE_BLK(step, i)
#define UB_TRACE_MIN(step, i)
#define UB_TRACE_MAX(step, i)
#endif

// The rows k_update_batch keeps in shared memory, packed once per step in its
// smem layout (one bulk copy per block instead of every block walking the
// winner's and the batch's rows): [cd: the winner's row, fp64][cb: RW batch
// rows, fp64][cg: RW batch rows + the winner's, fp32, interleaved by 4 dims:
// float4 (k4, j) at k4 (RW + 1) + j][cn: their fp32 norms].  One block per
// row (RW + 1 blocks).
struct BatchPackLayout {
  size_t dbytes, cbytes, fbytes;
  __host__ __device__ BatchPackLayout(int d) {
    const size_t dp = (size_t)((d + 3) & ~3);
    dbytes = ((size_t)d * 8 + 15) & ~(size_t)15;
    cbytes = ((size_t)RW * d * 8 + 15) & ~(size_t)15;
    fbytes = (((size_t)(RW + 1) * dp + RW + 1) * 4 + 15) & ~(size_t)15;
  }
  __host__ __device__ size_t bytes() const { return dbytes + cbytes + fbytes; }
};
// The pack's rows: j < RW the batch (src[j] < 0: empty), j == RW the winner.
// Called by every thread of a block (strided over the (RW + 1) x dp floats).
struct PackArgs {
  const float* V = nullptr;
  int pitch = 0, d = 0;
  const float* nv32 = nullptr;
  unsigned char* pack = nullptr;  // nullptr: no pack
};
__device__ void batch_pack_rows(const PackArgs& a, const int64_t* src) {
  const BatchPackLayout L(a.d);
  const int d = a.d, dp = (d + 3) & ~3;
  double* cd = reinterpret_cast<double*>(a.pack);
  double* cb = reinterpret_cast<double*>(a.pack + L.dbytes);
  float* cg = reinterpret_cast<float*>(a.pack + L.dbytes + L.cbytes);
  float* cn = cg + (size_t)(RW + 1) * dp;
  const float nvj = (int)threadIdx.x <= RW && src[threadIdx.x] >= 0 ? a.nv32[src[threadIdx.x]] : 0.f;
  for (int i0 = 0; i0 < (RW + 1) * dp; i0 += 4 * (int)blockDim.x) {
    float x[4];  // four elements' loads in flight before their stores
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e * blockDim.x + threadIdx.x;
      const int j = i / dp, k = i - j * dp;
      x[e] = i < (RW + 1) * dp && src[j] >= 0 && k < d ? a.V[src[j] * a.pitch + k] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e * blockDim.x + threadIdx.x;
      if (i >= (RW + 1) * dp) break;
      const int j = i / dp, k = i - j * dp;
      cg[((k >> 2) * (RW + 1) + j) * 4 + (k & 3)] = x[e];  // interleaved by 4 dims: [dp / 4][RW + 1] float4
      if (k < d) {
        if (j == RW)
          cd[k] = (double)x[e];
        else
          cb[j * d + k] = (double)x[e];
      }
    }
  }
  if ((int)threadIdx.x <= RW) cn[threadIdx.x] = nvj;
}

// Writes the batch to wlist[0..m) (m = min(lb, unselected candidates)),
// *wcount = m and *ub_next = the (rounded-up) best bound outside it (-inf if none).
__global__ void __launch_bounds__(256) k_lazy_topk(int64_t c0, int64_t c1, const double* __restrict__ ubp,
                                                   const unsigned char* __restrict__ selected, int lb,
                                                   unsigned long long* __restrict__ part,
                                                   unsigned int* __restrict__ counter, int* __restrict__ wcount,
                                                   int64_t* __restrict__ wlist, double* __restrict__ ub_next,
                                                   PackArgs pa, const int64_t* __restrict__ best, int step) {
  __shared__ unsigned long long wt[9 * TK];  // 8 warp lists + the merged one
  __shared__ int64_t ssrc[RW + 1];           // the pack's rows (pa.pack)
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TK_TRACE_MIN(step, 0);
  pdl_launch_dependents();  // k_update_batch stages its rows while the top-k runs
  unsigned long long l[TK];
#pragma unroll
  for (int j = 0; j < TK; ++j) l[j] = 0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // four candidates' loads in flight per thread before their inserts
  int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; c + 3 * stride < c1; c += 4 * stride) {
    double u[4];
    unsigned char sl[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      u[e] = ubp[c + e * stride - c0];
      sl[e] = selected[c + e * stride];
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (!sl[e]) top_insert(l, top_key(u[e], c + e * stride - c0));
  }
  for (; c < c1; c += stride)
    if (!selected[c]) top_insert(l, top_key(ubp[c - c0], c - c0));
  warp_topk(l, wt + warp * TK);
  __syncthreads();
  TK_TRACE_MAX(step, 1);
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < TK; ++j) l[j] = 0ull;
    for (int q = lane; q < 8 * TK; q += 32) top_insert(l, wt[q]);
    warp_topk(l, part + (int64_t)blockIdx.x * TK);
    __syncwarp();
    if (lane == 0) last = ticket_acq_rel(counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  TK_TRACE_MAX(step, 2);
  const int64_t wsrc = pa.pack && threadIdx.x == 0 ? *best : -1;  // in flight during the merges
#pragma unroll
  for (int j = 0; j < TK; ++j) l[j] = 0ull;
  const int total = (int)gridDim.x * TK;
  constexpr int PT = 12;  // independent loads per thread (2 x 148 blocks x TK < 12 x 256)
  unsigned long long x[PT];
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const int q = threadIdx.x + j * blockDim.x;
    x[j] = q < total ? __ldcg(part + q) : 0ull;
  }
#pragma unroll
  for (int j = 0; j < PT; ++j) top_insert(l, x[j]);
  for (int q = threadIdx.x + PT * blockDim.x; q < total; q += blockDim.x) top_insert(l, __ldcg(part + q));
  warp_topk(l, wt + warp * TK);
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < TK; ++j) l[j] = 0ull;
    for (int q = lane; q < 8 * TK; q += 32) top_insert(l, wt[q]);
    warp_topk(l, wt + 8 * TK);
    __syncwarp();
    if (lane == 0) {
      const unsigned long long* fin = wt + 8 * TK;
      int m = 0;
      for (int j = 0; j < lb; ++j)
        if (fin[j]) {
          const int64_t c = c0 + (int64_t)(0xFFFFFFFFu - (unsigned)(fin[j] & 0xFFFFFFFFull));
          ssrc[m] = c;
          wlist[m++] = c;
        }
      for (int j = m; j < RW; ++j) ssrc[j] = -1;
      ssrc[RW] = wsrc;
      *wcount = m;
      *ub_next = fin[lb] ? (double)__uint_as_float((unsigned)(fin[lb] >> 32)) : -INFINITY;
      *counter = 0u;
    }
  }
  if (!pa.pack) return;
  // the next update's pack (k_update_batch): the winner's row and the batch's
  __syncthreads();
  batch_pack_rows(pa, ssrc);
  __syncthreads();
  TK_TRACE_MAX(step, 3);
}

// Device-sharded lazy step: the decision of the batch refine's finalize, made
// with the bound all-reduced (max) across the ranks.  Decided (-2): the batch
// is the rank's window (its exact gains are in wgain; no local pick is needed,
// the ranks exchange tie-set frontiers of their windows).
__global__ void k_lazy_decide(const long long* __restrict__ maxlb, const double* __restrict__ ub_next, double margin,
                              int* __restrict__ level, long long* __restrict__ stats,
                              cudaGraphConditionalHandle hrest) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double lb = dkey_inv(*maxlb);
    const int done = *ub_next < lb - margin - 1e-9 * fabs(lb);
    level[0] = done ? -2 : -3;
    stats[5] += done;
    if (hrest) cudaGraphSetConditional(hrest, done ? 0u : 1u);
  }
}

// Probe batch of an undecided lazy step (level[0] == -3).  The first batch is
// the top stale bounds, and on clustered data those are the neighbours of the
// centre just selected: their gains collapsed, lb comes out tiny and nearly
// every candidate stays stale (C4 steps 2-7).  Any candidate's exact gain is a
// valid lb, so a second batch is drawn for diversity: candidates are binned in
// rings of |c - s|^2 around the last selected s (two binary exponents per ring),
// the best stale bound of each ring is kept, and the np ring winners with the
// largest bounds are refined (k_refine_short, RefineFinal batch 3: lb = max).
// Which candidates are probed never affects the result, only how many stay stale.
constexpr int NRING = 128;
struct ProbeBuf {
  unsigned long long* rkey = nullptr;  // NRING ring winners (top_key), zero between steps
  unsigned int* counter = nullptr;
  int* pcount = nullptr;
  int64_t* plist = nullptr;            // RW
};
__global__ void __launch_bounds__(256) k_lazy_rings(int64_t c0, int64_t c1, const float* __restrict__ V32, int pitch,
                                                    int d, const int64_t* __restrict__ best,
                                                    const double* __restrict__ ubp,
                                                    const unsigned char* __restrict__ selected,
                                                    const int* __restrict__ level, ProbeBuf pb, int np) {
  extern __shared__ float ssv[];  // d floats: the last selected row
  __shared__ unsigned long long sk[NRING];
  __shared__ bool last;
  for (int i = threadIdx.x; i < NRING; i += blockDim.x) sk[i] = 0ull;
  const bool on = *level == -3;
  const int64_t sb = on ? *best : -1;
  if (sb >= 0)
    for (int k = threadIdx.x; k < d; k += blockDim.x) ssv[k] = V32[sb * pitch + k];
  __syncthreads();
  if (sb >= 0) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < c1; c += stride) {
      if (selected[c]) continue;
      const float4* row = reinterpret_cast<const float4*>(V32 + c * pitch);
      float a0 = 0.f, a1 = 0.f;
      int k = 0;
      for (; k + 4 <= d; k += 4) {
        const float4 q = __ldg(row + (k >> 2));
        const float x0 = q.x - ssv[k], x1 = q.y - ssv[k + 1], x2 = q.z - ssv[k + 2], x3 = q.w - ssv[k + 3];
        a0 = fmaf(x0, x0, fmaf(x1, x1, a0));
        a1 = fmaf(x2, x2, fmaf(x3, x3, a1));
      }
      for (; k < d; ++k) {
        const float x = V32[c * pitch + k] - ssv[k];
        a0 = fmaf(x, x, a0);
      }
      const int ring = (int)(__float_as_uint(a0 + a1) >> 24) & (NRING - 1);
      const unsigned long long key = top_key(ubp[c - c0], c - c0);
      if (key > sk[ring]) atomicMax(&sk[ring], key);
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < NRING; r += blockDim.x)
    if (sk[r]) atomicMax(pb.rkey + r, sk[r]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(pb.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  // warp 0: the np largest ring winners (keys are unique), rings cleared for the next step
  const int lane = threadIdx.x;
  unsigned long long l[NRING / 32];
#pragma unroll
  for (int j = 0; j < NRING / 32; ++j) {
    l[j] = __ldcg(pb.rkey + lane + 32 * j);
    pb.rkey[lane + 32 * j] = 0ull;
  }
  int m = 0;
  for (int r = 0; r < np; ++r) {
    unsigned long long b = 0ull;
#pragma unroll
    for (int j = 0; j < NRING / 32; ++j) b = l[j] > b ? l[j] : b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, b, o);
      b = x > b ? x : b;
    }
    if (b == 0ull) break;
#pragma unroll
    for (int j = 0; j < NRING / 32; ++j)
      if (l[j] == b) l[j] = 0ull;
    if (lane == 0) pb.plist[m] = c0 + (int64_t)(0xFFFFFFFFu - (unsigned)(b & 0xFFFFFFFFull));
    ++m;
  }
  if (lane == 0) {
    *pb.pcount = m;
    *pb.counter = 0u;
  }
}

// Create-time maxima in one pass (no host copies of whole arrays): [0] max e0d
// (fp64 bits), [1] max |v|^2, [2] max per-tile |v|max, [3] min block radius
// (fp32 bits; all values are non-negative, so their bits order like them).
__global__ void k_create_maxes(const double* __restrict__ e0d, const float* __restrict__ nv32, int64_t n,
                               const float* __restrict__ vmax, int64_t ntl, const float* __restrict__ rad,
                               int64_t nrad, unsigned long long* __restrict__ out) {
  unsigned long long me = 0;
  unsigned int mv = 0, mx = 0, mr = 0x7f800000u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    me = max(me, (unsigned long long)__double_as_longlong(fmax(e0d[i], 0.0)));
    mv = max(mv, __float_as_uint(fmaxf(nv32[i], 0.f)));
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vmax && i < ntl; i += stride)
    mx = max(mx, __float_as_uint(fmaxf(vmax[i], 0.f)));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rad && i < nrad; i += stride)
    mr = min(mr, __float_as_uint(fmaxf(rad[i], 0.f)));
  for (int o = 16; o > 0; o >>= 1) {
    me = max(me, __shfl_xor_sync(0xffffffffu, me, o));
    mv = max(mv, __shfl_xor_sync(0xffffffffu, mv, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mr = min(mr, __shfl_xor_sync(0xffffffffu, mr, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, me);
    atomicMax(out + 1, (unsigned long long)mv);
    atomicMax(out + 2, (unsigned long long)mx);
    atomicMin(out + 3, (unsigned long long)mr);
  }
}

// Chunk geometry for the near-centre bound (k_lazy_nearbound), once per
// context: per RCH-point chunk T its fp64 mean mu_T, radius r_T >= max |v - mu_T|
// (rounded up), |mu_T|, the sum of e0d over it, and its point count.
struct ChunkGeo {
  double* mu = nullptr;   // nchunks x d
  double* r = nullptr;    // nchunks
  double* mn = nullptr;   // nchunks: |mu_T|
  double* e0s = nullptr;  // nchunks: sum of e0d (fixed order)
  float* muf = nullptr;   // nchunks x dp: mu_T rounded to fp32 (zero padded)
  int dp = 0;
  int nchunks = 0;
};
__global__ void __launch_bounds__(256) k_chunk_geo(const float* __restrict__ V32, int pitch, int64_t n, int d,
                                                   const double* __restrict__ e0d, ChunkGeo g) {
  extern __shared__ double cmu[];  // d
  __shared__ double red[8][33];
  const int ch = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t v0 = (int64_t)ch * RCH;
  const int np = (int)min((int64_t)RCH, n - v0);
  // mean: warp w sums rows w, w + 8, ... over 32 dims at a time (coalesced)
  for (int k0 = 0; k0 < d; k0 += 32) {
    const int k = k0 + lane;
    double s = 0.0;
    if (k < d)
      for (int j = warp; j < np; j += 8) s += (double)V32[(v0 + j) * pitch + k];
    red[warp][lane] = s;
    __syncthreads();
    if (tid < 32 && k < d) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w][tid];
      cmu[k] = t / (double)np;
      g.mu[(int64_t)ch * d + k] = cmu[k];
    }
    __syncthreads();
  }
  for (int k = tid; k < g.dp; k += blockDim.x) g.muf[(int64_t)ch * g.dp + k] = k < d ? (float)cmu[k] : 0.f;
  double rmax = 0.0, es = 0.0;
  for (int j = tid; j < np; j += blockDim.x) {
    double q = 0.0;
    for (int k = 0; k < d; ++k) {
      const double x = (double)V32[(v0 + j) * pitch + k] - cmu[k];
      q = fma(x, x, q);
    }
    rmax = fmax(rmax, q);
    es += e0d[v0 + j];
  }
  for (int o = 16; o > 0; o >>= 1) {
    rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    es += __shfl_xor_sync(0xffffffffu, es, o);
  }
  if (lane == 0) {
    red[warp][0] = rmax;
    red[warp][1] = es;
  }
  __syncthreads();
  if (tid == 0) {
    double m = 0.0, e = 0.0;
    for (int w = 0; w < 8; ++w) {
      m = fmax(m, red[w][0]);
      e += red[w][1];
    }
    g.r[ch] = sqrt(m) * (1.0 + 1e-9);
    g.e0s[ch] = e;
    double q = 0.0;
    for (int k = 0; k < d; ++k) q = fma(cmu[k], cmu[k], q);
    g.mn[ch] = sqrt(q) * (1.0 + 1e-9);
  }
}

// Near-centre bound of an undecided lazy step (level[0] == -3), for every stale
// candidate c (ubp >= the stale threshold).  With s the centre just selected,
// cm(v) <= d(v, s), so
//   gain(c) = sum_v max(0, cm(v) - d(v, c)) <= sum_v min(cm(v), max(0, d(v, s) - d(v, c)))
// and d(v, s) - d(v, c) = 2 v.u + |s|^2 - |c|^2 (u = c - s) is linear in v: over
// a chunk T, v.u <= mu_T.u + r_T |u|.  Hence
//   gain(c) <= sum_T min(CM_T, n_T max(0, 2 mu_T.u + 2 r_T |u| + |s|^2 - |c|^2 + m_T))
// with CM_T = sum of cm over T (= sum e0d - the update's chunk partial) and m_T
// covering the fp64 roundings of d64 and of this evaluation.  Candidates next
// to s (whose gains just collapsed -- on clustered data a whole cluster) get a
// bound far below lb and leave the stale set without a screen; the bound is
// stored in ubp (it bounds every later gain too).  A candidate whose partial
// sum already reaches the threshold stops early and stays stale.
constexpr int NB_CPB = 64;  // candidates per block (4 chunk groups of 64 threads)
// The dot mu_T.u runs in fp32 (mu_T rounded to fp32 in muf, u = fl32(c - s)):
// |error| <= (d + 4) 2^-24 |u| |mu_T| (products, partial sums, both roundings),
// added to the bound.  Each candidate visits the chunks starting at its own
// (on index-ordered clustered data its own cluster first, where a candidate far
// from s reaches the threshold after a few chunks and stops).
// Chunks are staged through shared memory NB_TILE at a time (fp32 means, the
// per-chunk scalars, this step's CM_T), so the inner loop is shared-memory
// broadcasts and FMAs; the block stops when every candidate has stopped.
constexpr int NB_TILE = 64;
template <int DR>  // DR > 0: u in DR registers (d <= DR); 0: u in shared memory
__global__ void __launch_bounds__(256) k_lazy_nearbound(int64_t c0, int64_t c1, const float* __restrict__ V32,
                                                        int pitch, int d, const int64_t* __restrict__ best,
                                                        double* __restrict__ ubp,
                                                        const unsigned char* __restrict__ selected,
                                                        const long long* __restrict__ maxlb, double margin,
                                                        const int* __restrict__ level, ChunkGeo g,
                                                        const double* __restrict__ fpart, int64_t n) {
  extern __shared__ float nbs[];  // s[dp], mu tile [NB_TILE][dp], then (DR == 0) u[d][NB_CPB]
  __shared__ double part[4][NB_CPB];
  __shared__ double tr[NB_TILE], tm[NB_TILE], tcm[NB_TILE], tn[NB_TILE];
  __shared__ int stop[NB_CPB];
  if (*level != -3) return;
  const int tid = threadIdx.x, j = tid & (NB_CPB - 1), grp = tid >> 6;
  const int dp = g.dp;
  const int64_t c = c0 + (int64_t)blockIdx.x * NB_CPB + j;
  const double lb = dkey_inv(*maxlb);
  const double thr = lb - margin - 1e-9 * fabs(lb);
  const bool stale = c < c1 && !selected[c] && ubp[c - c0] >= thr;
  if (!__syncthreads_or(stale)) return;
  const int64_t sb = *best;
  float* sv = nbs;
  float* mt = nbs + dp;
  float* us = mt + NB_TILE * dp;
  for (int k = tid; k < d; k += blockDim.x) sv[k] = V32[sb * pitch + k];
  if (tid < NB_CPB) stop[tid] = 0;
  __syncthreads();
  // u = fl32(c - s) (registers or smem), |u| from the exact differences, |c|^2, |s|^2
  float ur[DR > 0 ? DR : 1];
  double q = 0.0, cc = 0.0, s2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const float x = stale ? V32[c * pitch + k] : 0.f;
    const double du = (double)x - (double)sv[k];
    q = fma(du, du, q);
    cc = fma((double)x, (double)x, cc);
    s2 = fma((double)sv[k], (double)sv[k], s2);
    const float uf = x - sv[k];
    if constexpr (DR > 0) {
#pragma unroll
      for (int r = 0; r < DR; ++r)
        if (r == k) ur[r] = uf;
    } else if (grp == 0) {
      us[k * NB_CPB + j] = uf;
    }
  }
  if constexpr (DR > 0) {
#pragma unroll
    for (int r = 0; r < DR; ++r)
      if (r >= d) ur[r] = 0.f;
  }
  if (!stale && grp == 0) stop[j] = 1;
  const double un = sqrt(q) * (1.0 + 1e-12);
  const double mrel = 2.0 * (4e-12 + 1e-15 * (double)(d + 1));  // (a + b)^2 <= 2 a^2 + 2 b^2
  const double snc = fmax(sqrt(s2), sqrt(cc)) + un;
  const double cst = s2 - cc + mrel * snc * snc;  // per candidate
  const double kdot = 2.0 * (double)(d + 4) * 0x1p-24 * 1.01 * un;
  const double un2 = 2.0 * un;
  const int tstart = (int)min((int64_t)g.nchunks - 1, max((int64_t)0, (c0 + (int64_t)blockIdx.x * NB_CPB) / RCH));
  double acc = 0.0;
  bool mystop = !stale;
  for (int i0 = 0; i0 < g.nchunks; i0 += NB_TILE) {
    const int nt = min(NB_TILE, g.nchunks - i0);
    __syncthreads();  // previous tile consumed; stop flags visible
    if (__syncthreads_and(stop[j] != 0)) break;
    for (int e = tid; e < nt * dp; e += blockDim.x) {
      const int ti = e / dp, k = e - ti * dp;
      int T = tstart + i0 + ti;
      if (T >= g.nchunks) T -= g.nchunks;
      mt[e] = __ldg(g.muf + (int64_t)T * dp + k);
    }
    if (tid < nt) {
      int T = tstart + i0 + tid;
      if (T >= g.nchunks) T -= g.nchunks;
      const double rT = g.r[T], mnT = g.mn[T], e0s = g.e0s[T];
      tr[tid] = rT;
      tm[tid] = mnT;
      tcm[tid] = e0s - __ldcg(fpart + T) + 1e-12 * e0s;
      tn[tid] = (double)min((int64_t)RCH, n - (int64_t)T * RCH);
    }
    __syncthreads();
    if (mystop || stop[j]) continue;
    for (int ti = grp; ti < nt; ti += 4) {
      const float* mu = mt + ti * dp;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      if constexpr (DR > 0) {
#pragma unroll
        for (int k = 0; k < DR; k += 4) {
          if (k >= dp) break;
          const float4 m4 = *reinterpret_cast<const float4*>(mu + k);
          a0 = fmaf(ur[k], m4.x, a0);
          a1 = fmaf(ur[k + 1], m4.y, a1);
          a2 = fmaf(ur[k + 2], m4.z, a2);
          a3 = fmaf(ur[k + 3], m4.w, a3);
        }
      } else {
        for (int k = 0; k < d; ++k) a0 = fmaf(us[k * NB_CPB + j], mu[k], a0);
      }
      const float dot = (a0 + a1) + (a2 + a3);
      const double rT = tr[ti], mnT = tm[ti];
      const double MT = mnT + rT;
      const double ell = fma(2.0, (double)dot, fma(rT, un2, fma(mnT, kdot, fma(mrel * MT, MT, cst))));
      if (ell > 0.0) acc += fmin(tcm[ti], tn[ti] * ell);
    }
    if (acc >= thr) {  // cannot leave the stale set: stop every group of the candidate
      mystop = true;
      stop[j] = 1;
    }
  }
  __syncthreads();
  part[grp][j] = acc;
  __syncthreads();
  if (grp == 0 && stale && !stop[j]) {
    const double b = (((part[0][j] + part[1][j]) + part[2][j]) + part[3][j]) * (1.0 + 1e-12);
    if (b < ubp[c - c0]) ubp[c - c0] = b;
  }
}

// Undecided lazy step (level[0] == -3): list the stale candidates
// ubp[c] >= lb - margin - 1e-9 |lb| (lb = *maxlb, the batch's best exact gain)
// in slist (count *scount) and flag their 128-candidate blocks.
// The stale set in INDEX ORDER (three passes: per-256-block counts, one-block
// scan, ordered writes) -- a gathered re-screen packs neighbouring candidates
// into the same 128-candidate block, which keeps the block anchors close and
// the tile pruning effective.
__device__ __forceinline__ bool lazy_is_stale(int64_t c, int64_t c0, int64_t c1, const double* __restrict__ ubp,
                                              const unsigned char* __restrict__ selected, double thr) {
  return c < c1 && !selected[c] && ubp[c - c0] >= thr;
}

__global__ void __launch_bounds__(256) k_lazy_mark2(int64_t c0, int64_t c1, const double* __restrict__ ubp,
                                                    const unsigned char* __restrict__ selected,
                                                    const long long* __restrict__ maxlb, double margin,
                                                    int* __restrict__ bcnt, unsigned char* __restrict__ bflag,
                                                    const int* __restrict__ level) {
  __shared__ int wsum[8];
  if (*level != -3) return;
  const double lb = dkey_inv(*maxlb);
  const double thr = lb - margin - 1e-9 * fabs(lb);
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool stale = lazy_is_stale(c, c0, c1, ubp, selected, thr);
  if (stale) bflag[(c - c0) >> 7] = 1;
  const unsigned bal = __ballot_sync(0xffffffffu, stale);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += wsum[w];
    bcnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_lazy_scan(int* __restrict__ bcnt, int nb, int* __restrict__ scount,
                                                    const int* __restrict__ level) {
  __shared__ int sx[1024];
  __shared__ int carry;
  if (*level != -3) return;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int x = b < nb ? bcnt[b] : 0;
    sx[threadIdx.x] = x;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive scan (Hillis-Steele)
      const int y = threadIdx.x >= o ? sx[threadIdx.x - o] : 0;
      __syncthreads();
      sx[threadIdx.x] += y;
      __syncthreads();
    }
    if (b < nb) bcnt[b] = carry + sx[threadIdx.x] - x;  // exclusive offset, in place
    __syncthreads();
    if (threadIdx.x == 0) carry += sx[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *scount = carry;
}

__global__ void __launch_bounds__(256) k_lazy_write(int64_t c0, int64_t c1, const double* __restrict__ ubp,
                                                    const unsigned char* __restrict__ selected,
                                                    const long long* __restrict__ maxlb, double margin,
                                                    const int* __restrict__ boff, int64_t* __restrict__ slist,
                                                    const int* __restrict__ level) {
  __shared__ int wsum[8];
  if (*level != -3) return;
  const double lb = dkey_inv(*maxlb);
  const double thr = lb - margin - 1e-9 * fabs(lb);
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool stale = lazy_is_stale(c, c0, c1, ubp, selected, thr);
  const unsigned bal = __ballot_sync(0xffffffffu, stale);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int off = boff[blockIdx.x];
  for (int w = 0; w < warp; ++w) off += wsum[w];
  if (stale) slist[off + __popc(bal & ((1u << lane) - 1u))] = c;
}

// Mode of an undecided lazy step (level[0] == -3), written to level[0]:
//   -1  few stale candidates (<= cap, or no screen): they are the window of
//       the second refine (copied into wlist);
//   rung  many: the flagged blocks are re-screened and the screen builds the
//       window (hs: the screen's conditional graph node, when captured).
// stats: [5] lazy steps decided without a screen, [6] candidates re-examined.
constexpr int L_GATHER = 8;  // level[0] of a gathered re-screen (matches no rung: the block screens skip)
__global__ void __launch_bounds__(256) k_lazy_plan2(const int* __restrict__ scount,
                                                    const int64_t* __restrict__ slist, int cap,
                                                    int* __restrict__ wcount, int64_t* __restrict__ wlist,
                                                    int* __restrict__ level, long long* __restrict__ stats,
                                                    cudaGraphConditionalHandle hs,
                                                    const unsigned char* __restrict__ bflag = nullptr, int nblocks = 0,
                                                    int gather_cap = 0, int gather_rung = -1,
                                                    cudaGraphConditionalHandle hg = 0) {
  __shared__ int nfl;
  if (level[0] != -3) return;
  const int cnt = *scount;
  const bool few = cnt <= cap;
  if (few)
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) wlist[i] = slist[i];
  // gathered re-screen: the stale set compacted into fresh 128-candidate blocks
  // when the flagged blocks are less than half full (scattered stale sets)
  if (threadIdx.x == 0) nfl = 0;
  __syncthreads();
  bool gather = false;
  if (!few && gather_cap > 0 && cnt <= gather_cap && level[1] == gather_rung) {
    int m = 0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) m += bflag[b] != 0;
    atomicAdd(&nfl, m);
    __syncthreads();
    gather = (int64_t)nfl * 128 > 2 * (int64_t)cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    stats[6] += cnt;
    stats[5] += few ? 1 : 0;  // decided without a screen
    level[0] = few ? -1 : (gather ? L_GATHER : level[1]);
    *wcount = few ? cnt : 0;
    if (hs) cudaGraphSetConditional(hs, (few || gather) ? 0u : 1u);
    if (hg) cudaGraphSetConditional(hg, gather ? 1u : 0u);
  }
}

// Gathered re-screen: the stale candidates' rows packed into Vg (rows past the
// count up to the block boundary zeroed), ub = -inf for every candidate (the
// gathered finalize writes the re-screened ones).
__global__ void k_gather_rows(const float* __restrict__ V32, int pitch, const int64_t* __restrict__ slist,
                              const int* __restrict__ scount, int cap, float* __restrict__ Vg,
                              double* __restrict__ ub, int64_t ncand, const int* __restrict__ level_now, int level) {
  if (*level_now != level) return;
  const int cnt = min(*scount, cap);
  const int64_t rows = ((int64_t)cnt + 127) / 128 * 128;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * pitch; i += stride) {
    const int64_t r = i / pitch;
    const int k = (int)(i - r * pitch);
    Vg[i] = r < cnt ? V32[slist[r] * pitch + k] : 0.f;
  }
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncand; c += stride) ub[c] = -INFINITY;
}

// Bounds of the gathered candidates (k_finalize's ub-only formula per slot).
__global__ void k_finalize_gathered(const int* __restrict__ scount, const int64_t* __restrict__ slist, int64_t c0,
                                    int nsplit, const double* __restrict__ part_g, const float* __restrict__ part_e,
                                    int64_t part_stride, double einfl, double gcoef, double gscale,
                                    const unsigned char* __restrict__ selected, double* __restrict__ ub,
                                    double* __restrict__ ubp, const int* __restrict__ level_now, int level) {
  if (*level_now != level) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *scount) return;
  const int64_t c = slist[i];
  double g = 0.0, e = 0.0;
  for (int s = 0; s < nsplit; ++s) {
    g += part_g[s * part_stride + i];
    e += (double)part_e[s * part_stride + i];
  }
  g *= gscale;
  e *= gscale;
  const double eps = e * einfl + gcoef * g + 1e-300;
  if (selected[c]) {
    ub[c - c0] = -INFINITY;
  } else {
    ub[c - c0] = g + eps;
    ubp[c - c0] = fmin(ubp[c - c0], g + eps);
  }
}

// Exact fp64 gain partials.  The nchunks point chunks are cut into ng fixed
// groups (ng depends only on n).  A unit is (window group of RW candidates,
// chunk group): every V row it reads is used for RW candidates (L2 traffic /RW).
// Per candidate and chunk, each thread sums its 4 points in order, then the
// 256 per-thread partials are reduced by one warp in a fixed order (8
// sequential per lane, then a butterfly); chunks are added left to right into
// part_r[w*ng + grp].  A candidate's value never depends on its RW neighbours,
// its slot in the window, or the number of ranks.

// Certified tile-pair pruning: every point of tile t is at least rho - R from
// every candidate of the block (triangle inequality through the anchor), so
// when (rho - R)^2 > max cm over the tile no pair can contribute or count.
// Explicit roundings (no contraction) so every role of a CTA agrees bit for bit.
__device__ __forceinline__ bool tile_prunable(float rho, float rad, float cmx) {
  const float gap = __fsub_rn(rho, rad);
  return gap > 0.f && __fmul_rn(__fmul_rn(gap, gap), 0.99999f) > cmx;
}

// Exact chunk skipping for the refine (tensor-screen anchors, screen_tc.cuh):
// a chunk whose every point tile is certified out of reach of candidate c
// ((rho_a[tile] - |c - mu_a|)^2 > max cm over the tile, same test as the
// screen's tile-pair pruning) has every term max(0, cm - d) exactly 0, so
// skipping it leaves the fixed-order fp64 sums bit for bit unchanged.
struct RefinePrune {
  const float* rho = nullptr;  // na x kpstride (nullptr: off)
  int64_t kpstride = 0;
  const float* cmx = nullptr;  // per point tile, current step
  const int* tile_anchor = nullptr;
  const float* anchors = nullptr;
  int apitch = 0;
  int np = 128;                // points per tile
  const float* crad = nullptr; // per candidate |c - mu_anchor| rounded up (k_cand_rad, at create)
};

// crad[c] = |c - mu_a|, a = the anchor of c's 128-row block, in fp64 and rounded
// up (the refine's pruning radius; computed once at create instead of per unit).
template <typename T>
__global__ void k_cand_rad(const T* __restrict__ V, int pitch, int64_t n, int d, const int* __restrict__ tile_anchor,
                           const float* __restrict__ anchors, int apitch, float* __restrict__ crad) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const float* mu = anchors + (int64_t)tile_anchor[c >> 7] * apitch;
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double x = (double)V[c * pitch + k] - (double)mu[k];
    r2 = fma(x, x, r2);
  }
  crad[c] = __double2float_ru(sqrt(r2) * (1.0 + 1e-12));
}

// The pick, folded into the refine's last block (the block whose ticket
// completes the grid): exact gains of the window, the reference argmax rule
// (optimize.py:83-85: top = max value; window = 1e-12 max(1,|top|); best =
// lowest index with value >= top - window; value = f(S) + gain/N) and, with
// `commit`, the selection.  A lazy first batch (`batch`) first decides whether
// it holds the whole stale set (best bound outside it below the threshold):
// if so it picks and marks the step decided (level[0] = -2), otherwise it
// marks it undecided (-3) and leaves the pick to the second refine.
struct RefineFinal {
  unsigned int* counter = nullptr;  // nullptr: no finalize (the caller picks)
  double* wgain = nullptr;
  double inv_n = 0.0;
  const double* cur = nullptr;
  int64_t* best = nullptr;
  int commit = 0, step = 0;
  unsigned char* selected = nullptr;
  int64_t* sel_out = nullptr;
  long long* stats = nullptr;   // [0] window sum [1] max [2] rung [3] steps [5] decided lazy steps [7] lazy steps
  int* level = nullptr;         // [0] this step's gate, [1] the run's rung
  double* ubp = nullptr;        // lazy bounds: exact gains of the window
  int64_t c0 = 0;
  int batch = 0;
  const double* ub_next = nullptr;
  double margin = 0.0;
  long long* maxlb = nullptr;
  int* scount = nullptr;                 // zeroed for the undecided path
  cudaGraphConditionalHandle hrest = 0;  // the undecided-step conditional node (graph capture)
};

// nt: the participating threads (the first nt of the block; every thread of
// the block must call it -- it synchronises the block)
// pre: (optional) the wc x ng partials already in shared memory (the caller
// computed them there); otherwise they are read from part_r.
__device__ void refine_finalize_n(const RefineFinal& F, int wc, const int64_t* __restrict__ wlist,
                                  const double* __restrict__ part_r, int ng, double* sred, long long* sidx,
                                  int nt, const double* pre = nullptr, const double* fsm = nullptr) {
  const int tid = threadIdx.x;
  const bool on = tid < nt;
  // thread 0's reads of the step state go out first (no latency on the tail)
  long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0}, lvl1 = -1, mlb = 0;
  double ubn = 0.0;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) st[i] = F.stats[i];
    if (F.level) lvl1 = F.level[1];
    if (F.batch == 1) ubn = *F.ub_next;
    if (F.batch == 3) mlb = *F.maxlb;
  }
  const double f = fsm ? *fsm : *F.cur;
  double top = -INFINITY, gmax = 0.0, mine = 0.0;
  // short windows: every partial loaded by the whole block first (one memory
  // round trip), then each candidate's left-to-right sum from shared memory --
  // the same additions in the same order as chunk_total
  const bool staged = wc <= nt && (pre || (int64_t)wc * ng <= 2 * (int64_t)nt);
  if (staged && !pre) {
    for (int i = tid; i < wc * ng && on; i += nt) sred[i] = __ldcg(part_r + i);
    __syncthreads();
  }
  const double* sp = pre ? pre : sred;
  double gs = 0.0;
  if (staged && tid < wc)
    for (int q = 0; q < ng; ++q) gs += sp[tid * ng + q];
  __syncthreads();
  for (int w = tid; w < wc && on; w += nt) {
    const double gsum = staged ? gs : chunk_total(part_r + (int64_t)w * ng, ng);
    mine = gsum;  // staged: w == tid, read back below without a memory round trip
    F.wgain[w] = gsum;
    if (F.ubp) F.ubp[wlist[w] - F.c0] = gsum;  // the exact gain bounds every later one (submodularity)
    top = fmax(top, __dadd_rn(f, __dmul_rn(gsum, F.inv_n)));  // no FMA contraction: host pick() matches
    gmax = fmax(gmax, gsum);
  }
  if (on) {
    sred[tid] = top;
    sred[nt + tid] = gmax;
  }
  __syncthreads();
  for (int st = nt / 2; st > 0; st >>= 1) {
    if (tid < st) {
      sred[tid] = fmax(sred[tid], sred[tid + st]);
      sred[nt + tid] = fmax(sred[nt + tid], sred[nt + tid + st]);
    }
    __syncthreads();
  }
  top = sred[0];
  if (F.batch == 3) {  // probe batch (k_lazy_rings): raises lb, decides nothing
    if (tid == 0 && wc > 0) {
      const long long k = dkey(sred[nt]);
      if (k > mlb) *F.maxlb = k;
      F.stats[6] = st[6] + wc;
    }
    return;
  }
  if (F.batch == 2) {  // sharded: the decision waits for the global bound (k_lazy_decide)
    if (tid == 0) {
      *F.maxlb = dkey(sred[nt]);
      F.stats[7] = st[7] + 1;
      F.stats[6] = st[6] + wc;
      F.level[0] = -3;
      *F.scount = 0;  // for the undecided path
    }
    return;
  }
  if (F.batch) {
    __shared__ int sdone;
    if (tid == 0) {
      const double lb = sred[nt];
      const int done = ubn < lb - F.margin - 1e-9 * fabs(lb);
      *F.maxlb = dkey(lb);
      F.stats[7] = st[7] + 1;
      F.stats[5] = st[5] + done;
      F.stats[6] = st[6] + wc;
      F.level[0] = done ? -2 : -3;
      *F.scount = 0;
      if (F.hrest) cudaGraphSetConditional(F.hrest, done ? 0u : 1u);
      sdone = done;
    }
    __syncthreads();
    if (!sdone) return;
  }
  const double window = 1e-12 * fmax(1.0, fabs(top));
  long long bi = LLONG_MAX;
  for (int w = tid; w < wc && on; w += nt) {
    const double val = __dadd_rn(f, __dmul_rn(staged ? mine : F.wgain[w], F.inv_n));
    if (val >= top - window) bi = min(bi, (long long)wlist[w]);
  }
  if (on) sidx[tid] = bi;
  __syncthreads();
  for (int st = nt / 2; st > 0; st >>= 1) {
    if (tid < st) sidx[tid] = min(sidx[tid], sidx[tid + st]);
    __syncthreads();
  }
  if (tid == 0) {
    const long long b = sidx[0] == LLONG_MAX ? -1 : sidx[0];
    *F.best = b;
    F.stats[0] = st[0] + wc;
    F.stats[1] = max(st[1], (long long)wc);
    F.stats[2] = lvl1;
    F.stats[3] = st[3] + 1;
    if (F.commit && b >= 0) {
      F.selected[b] = 1;
      F.sel_out[F.step] = b;
    }
  }
}

// refine_finalize_n for a window of at most 32 candidates whose exact gains
// are in shared memory (gs[w]) and f(S) at *fsm: the same decisions and
// writes, on ONE warp (shuffle reductions, no block barriers).  Called by
// every lane of one warp.
__device__ void refine_finalize_warp(const RefineFinal& F, int wc, const int64_t* __restrict__ wlist,
                                     const double* gs, const double* fsm) {
  const int lane = threadIdx.x & 31;
  long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0}, lvl1 = -1, mlb = 0;
  double ubn = 0.0;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) st[i] = F.stats[i];
    if (F.level) lvl1 = F.level[1];
    if (F.batch == 1) ubn = *F.ub_next;
    if (F.batch == 3) mlb = *F.maxlb;
  }
  const double f = *fsm;
  const bool on = lane < wc;
  const double g = on ? gs[lane] : 0.0;
  const int64_t c = on ? wlist[lane] : 0;
  if (on) {
    F.wgain[lane] = g;
    if (F.ubp) F.ubp[c - F.c0] = g;  // the exact gain bounds every later one (submodularity)
  }
  double top = on ? __dadd_rn(f, __dmul_rn(g, F.inv_n)) : -INFINITY;  // no FMA contraction: host pick() matches
  double gmax = on ? fmax(0.0, g) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    top = fmax(top, __shfl_xor_sync(0xffffffffu, top, o));
    gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  }
  if (F.batch == 3) {  // probe batch (k_lazy_rings): raises lb, decides nothing
    if (lane == 0 && wc > 0) {
      const long long k = dkey(gmax);
      if (k > mlb) *F.maxlb = k;
      F.stats[6] = st[6] + wc;
    }
    return;
  }
  if (F.batch == 2) {  // sharded: the decision waits for the global bound (k_lazy_decide)
    if (lane == 0) {
      *F.maxlb = dkey(gmax);
      F.stats[7] = st[7] + 1;
      F.stats[6] = st[6] + wc;
      F.level[0] = -3;
      *F.scount = 0;
    }
    return;
  }
  if (F.batch) {
    int done = 0;
    if (lane == 0) {
      const double lb = gmax;
      done = ubn < lb - F.margin - 1e-9 * fabs(lb);
      *F.maxlb = dkey(lb);
      F.stats[7] = st[7] + 1;
      F.stats[5] = st[5] + done;
      F.stats[6] = st[6] + wc;
      F.level[0] = done ? -2 : -3;
      *F.scount = 0;
      if (F.hrest) cudaGraphSetConditional(F.hrest, done ? 0u : 1u);
    }
    if (!__shfl_sync(0xffffffffu, done, 0)) return;
  }
  const double window = 1e-12 * fmax(1.0, fabs(top));
  long long bi = on && __dadd_rn(f, __dmul_rn(g, F.inv_n)) >= top - window ? (long long)c : LLONG_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bi = min(bi, (long long)__shfl_xor_sync(0xffffffffu, bi, o));
  if (lane == 0) {
    const long long b = bi == LLONG_MAX ? -1 : bi;
    *F.best = b;
    F.stats[0] = st[0] + wc;
    F.stats[1] = max(st[1], (long long)wc);
    F.stats[2] = lvl1;
    F.stats[3] = st[3] + 1;
    if (F.commit && b >= 0) {
      F.selected[b] = 1;
      F.sel_out[F.step] = b;
    }
  }
}

__device__ __forceinline__ void refine_finalize(const RefineFinal& F, int wc, const int64_t* __restrict__ wlist,
                                                const double* __restrict__ part_r, int ng, double* sred,
                                                long long* sidx) {
  refine_finalize_n(F, wc, wlist, part_r, ng, sred, sidx, blockDim.x);
}

template <typename T, bool BIGD>
__global__ void __launch_bounds__(RED_THREADS) k_refine(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                        const double* __restrict__ cm64,
                                                        const int* __restrict__ wcount,
                                                        const int64_t* __restrict__ wlist, int nchunks, int ng,
                                                        double* __restrict__ part_r, RefinePrune pr,
                                                        const int* __restrict__ skip_level, RefineFinal fin) {
  if (skip_level && *skip_level == -2) return;  // lazy step already decided by the first batch
  extern __shared__ double cd[];  // RW * d doubles (BIGD: candidates read through L1 instead)
  __shared__ double red[RW][RED_THREADS];
  __shared__ int64_t cidx[RW];
  __shared__ double tot[RW];
  __shared__ float crad[RW];   // |c - mu_anchor| rounded up (pruning)
  __shared__ int canc[RW];
  __shared__ int live[RW];     // candidate j has a reachable tile in this chunk
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpg = (nchunks + ng - 1) / ng;
  const int wc = *wcount;
  const int ngroups = (wc + RW - 1) / RW;
  const int64_t units = (int64_t)ngroups * ng;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int wg = (int)(u / ng);
    const int grp = (int)(u - (int64_t)wg * ng);
    const int nw = min(RW, wc - wg * RW);
    __syncthreads();
    if (!BIGD) {
      for (int i = tid; i < RW * d; i += blockDim.x) {
        const int j = i / d, k = i - j * d;
        cd[i] = j < nw ? (double)V[wlist[wg * RW + j] * pitch + k] : 0.0;
      }
    }
    if (tid < RW) {
      tot[tid] = 0.0;
      cidx[tid] = tid < nw ? wlist[wg * RW + tid] : wlist[wg * RW];
      if (pr.rho) {
        const int64_t c = cidx[tid];
        canc[tid] = pr.tile_anchor[c >> 7];
        crad[tid] = pr.crad[c];
      }
    }
    __syncthreads();
    const int ch1 = min(nchunks, (grp + 1) * cpg);
    for (int ch = grp * cpg; ch < ch1; ++ch) {
      if (tid < RW) {
        int lv = tid < nw;
        if (lv && pr.rho) {
          lv = 0;
          const int tpc = RCH / pr.np;
          const float* rho = pr.rho + (int64_t)canc[tid] * pr.kpstride;
          for (int q = 0; q < tpc; ++q) {
            const int64_t t = (int64_t)ch * tpc + q;
            if (t * pr.np < n && !tile_prunable(rho[t], crad[tid], pr.cmx[t])) lv = 1;
          }
        }
        live[tid] = lv;
      }
      __syncthreads();
      bool any = false;
#pragma unroll
      for (int j = 0; j < RW; ++j) any |= live[j] != 0;
      double acc[RW];
#pragma unroll
      for (int j = 0; j < RW; ++j) acc[j] = 0.0;
      const int64_t v0 = (int64_t)ch * RCH + tid;
      if (v0 < n && any) {
        // the thread's 4 points as 4 interleaved chains per candidate: each
        // (point, candidate) chain is the same sequential fp64 operation
        // sequence as before (bit-identical), the 4 x RW chains overlap
        unsigned lm = 0;  // block-uniform: a short window / unreachable chunk does not pay
#pragma unroll
        for (int j = 0; j < RW; ++j) lm |= (live[j] ? 1u : 0u) << j;
        const T* row[4];
        double s[4][RW];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t v = v0 + (int64_t)i * RED_THREADS;
          row[i] = V + (v < n ? v : v0) * pitch;
#pragma unroll
          for (int j = 0; j < RW; ++j) s[i][j] = 0.0;
        }
        auto step = [&](int k, const double (&x)[4]) {
#pragma unroll
          for (int j = 0; j < RW; ++j) {
            if (lm >> j & 1u) {
              const double cv = BIGD ? (double)__ldg(V + cidx[j] * pitch + k) : cd[j * d + k];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const double t = x[i] - cv;
                s[i][j] = fma(t, t, s[i][j]);
              }
            }
          }
        };
        int k = 0;
        if constexpr (sizeof(T) == 4) {
          // fp32 rows are 16-byte aligned (pitch % 4 == 0): one LDG.128 per row
          // and 4 dims; 8 dims per iteration keep the 8 loads of the four rows
          // in flight together (the refine of a short window is latency-bound)
          for (; k + 8 <= d; k += 8) {
            float4 q[4], r[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              q[i] = __ldg(reinterpret_cast<const float4*>(row[i]) + (k >> 2));
              r[i] = __ldg(reinterpret_cast<const float4*>(row[i]) + (k >> 2) + 1);
            }
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].x;
            step(k, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].y;
            step(k + 1, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].z;
            step(k + 2, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].w;
            step(k + 3, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)r[i].x;
            step(k + 4, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)r[i].y;
            step(k + 5, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)r[i].z;
            step(k + 6, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)r[i].w;
            step(k + 7, x);
          }
          for (; k + 4 <= d; k += 4) {
            float4 q[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) q[i] = __ldg(reinterpret_cast<const float4*>(row[i]) + (k >> 2));
            double x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].x;
            step(k, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].y;
            step(k + 1, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].z;
            step(k + 2, x);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (double)q[i].w;
            step(k + 3, x);
          }
        }
        for (; k < d; ++k) {
          double x[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) x[i] = (double)row[i][k];
          step(k, x);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t v = v0 + (int64_t)i * RED_THREADS;
          if (v < n) {
            const double c = cm64[v];
#pragma unroll
            for (int j = 0; j < RW; ++j) {
              const double t = c - s[i][j];
              if (lm >> j & 1u) acc[j] += t > 0.0 ? t : 0.0;
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < RW; ++j) red[j][tid] = acc[j];
      __syncthreads();
      {
        // warp `warp` reduces candidate j = warp (RW == 8 warps)
        double x = 0.0;
#pragma unroll
        for (int q = 0; q < RED_THREADS / 32; ++q) x += red[warp][lane * (RED_THREADS / 32) + q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) tot[warp] += x;
      }
      __syncthreads();
    }
    if (tid < nw) part_r[(int64_t)(wg * RW + tid) * ng + grp] = tot[tid];
  }
  if (!fin.counter) return;
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(fin.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid == 0) *fin.counter = 0u;
  refine_finalize(fin, wc, wlist, part_r, ng, &red[0][0], reinterpret_cast<long long*>(&red[2][0]));
}
static_assert(RW == RED_THREADS / 32, "one reducing warp per window candidate");

// Refine of a short window (<= RW candidates: the lazy first batch).  The
// classic k_refine gives each (window group, chunk group) unit to a 256-thread
// block (4 points per thread, the row loads on its critical path), so a short
// window runs latency-bound on nchunks blocks.  Here every point is one thread
// and every chunk is SHORT_SPLIT blocks of RED_THREADS (all SMs stream V):
// term(v, j) = max(0, cm(v) - d64(v, c_j)) with the same sequential fp64
// operations per (point, candidate) (certified-unreachable tiles give 0,
// exactly what the classic computes there), written to xt; the block taking a
// chunk's last ticket replays the classic chunk reduction -- thread t adds the
// terms of points t, t+256, t+512, t+768 in order, the same 8-sequential +
// butterfly warp sums -- and the chunk sums are combined by the last chunk in
// the classic order (chunks of a group left to right, then the groups):
// bit-identical partials, so both refines serve any candidate.
constexpr int SHORT_THREADS = RED_THREADS;
constexpr int SHORT_SPLIT = RCH / RED_THREADS;  // blocks per chunk
struct ShortBufs {
  double* xt = nullptr;              // RW x n_pad terms
  int64_t xstride = 0;               // n_pad
  unsigned int* chunk_ticket = nullptr;  // nchunks (zero between launches)
};
// STAGE: the block's 256 rows and cm values arrive by two bulk copies on one
// mbarrier (one request in flight per block instead of a row walk per thread).
template <typename T, bool STAGE>
__global__ void __launch_bounds__(SHORT_THREADS) k_refine_short(const T* __restrict__ V, int pitch, int64_t n,
                                                                int d, const double* __restrict__ cm64,
                                                                const int* __restrict__ wcount,
                                                                const int64_t* __restrict__ wlist, int nchunks,
                                                                int ng, double* __restrict__ xch,
                                                                double* __restrict__ part_r, RefinePrune pr,
                                                                RefineFinal fin, ShortBufs sb) {
  // dynamic smem: STAGE ? [rows 256 x pitch T][cm 256 doubles] : [], then cd: RW * d doubles,
  // then (fp32 rows) cf: RW * d floats for the far32 pre-test
  extern __shared__ __align__(128) unsigned char rs_smem[];
  const size_t stage_bytes = STAGE ? (size_t)RED_THREADS * pitch * sizeof(T) + RED_THREADS * sizeof(double) : 0;
  double* cd = reinterpret_cast<double*>(rs_smem + stage_bytes);
  float* cf = reinterpret_cast<float*>(cd + RW * d);
  __shared__ uint64_t sfull;
  __shared__ double red[RW][RED_THREADS];
  __shared__ int lmask[RED_THREADS / 64];  // live candidates per point tile of this block
  __shared__ int flag;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wc = min(RW, *wcount);
  const int ch = blockIdx.x / SHORT_SPLIT, qb = blockIdx.x - ch * SHORT_SPLIT;
  const int64_t bs = (int64_t)ch * RCH + (int64_t)qb * RED_THREADS;
  if (STAGE && tid == 0) {
    mbar_init(&sfull, 1);
    fence_mbar_init();
    if (bs < n && wc > 0) {  // rows < n_pad: always a whole slice
      const uint32_t rb = (uint32_t)RED_THREADS * pitch * sizeof(T);
      mbar_arrive_expect_tx(&sfull, rb + RED_THREADS * 8);
      bulk_g2s(rs_smem, V + bs * pitch, rb, &sfull);
      bulk_g2s(rs_smem + rb, cm64 + bs, RED_THREADS * 8, &sfull);
    }
  }
  for (int i = tid; i < RW * d; i += blockDim.x) {
    const int j = i / d, k = i - j * d;
    const T x = j < wc ? V[wlist[j] * pitch + k] : (T)0;
    cd[i] = (double)x;
    if constexpr (sizeof(T) == 4) cf[i] = (float)x;
  }
  const int64_t b0 = (int64_t)ch * RCH + (int64_t)qb * RED_THREADS;  // first point of this block
  const int tpb = RED_THREADS / pr.np;                                // point tiles per block (np <= 256)
  if (tid < max(tpb, 1)) {
    unsigned m = (1u << wc) - 1u;
    const int64_t t = b0 / pr.np + tid;
    if (pr.rho && t * pr.np < n) {
      m = 0;
      for (int j = 0; j < wc; ++j) {
        const int64_t c = wlist[j];
        const float* rho = pr.rho + (int64_t)pr.tile_anchor[c >> 7] * pr.kpstride;
        if (!tile_prunable(rho[t], pr.crad[c], pr.cmx[t])) m |= 1u << j;
      }
    }
    lmask[tid] = (int)m;
  }
  __syncthreads();
  const int64_t v = b0 + tid;
  unsigned lm = (unsigned)lmask[tpb > 0 ? tid / pr.np : 0];
  if (STAGE && bs < n && wc > 0) mbar_wait(&sfull, 0);
  const double c = v < n ? (STAGE ? reinterpret_cast<const double*>(rs_smem + (size_t)RED_THREADS * pitch *
                                                                              sizeof(T))[tid]
                                  : cm64[v])
                         : 0.0;
  double s[RW];
#pragma unroll
  for (int j = 0; j < RW; ++j) s[j] = 0.0;
  if constexpr (sizeof(T) == 4) {
    // far32 pre-test: only candidates that may be closer than cm get the fp64 sum
    if (v < n && lm) {
      const float4* r4 = STAGE ? reinterpret_cast<const float4*>(reinterpret_cast<const float*>(rs_smem) +
                                                                 (size_t)tid * pitch)
                               : reinterpret_cast<const float4*>(V + v * pitch);
      float q32[RW];
#pragma unroll
      for (int j = 0; j < RW; ++j) q32[j] = 0.f;
      int k = 0;
      for (; k + 4 <= d; k += 4) {
        const float4 q = STAGE ? r4[k >> 2] : __ldg(r4 + (k >> 2));
#pragma unroll
        for (int j = 0; j < RW; ++j)
          if (lm >> j & 1u) {
            const float* cj = cf + j * d + k;
            float x = q.x - cj[0];
            q32[j] = fmaf(x, x, q32[j]);
            x = q.y - cj[1];
            q32[j] = fmaf(x, x, q32[j]);
            x = q.z - cj[2];
            q32[j] = fmaf(x, x, q32[j]);
            x = q.w - cj[3];
            q32[j] = fmaf(x, x, q32[j]);
          }
      }
      for (; k < d; ++k) {
        const float xr = reinterpret_cast<const float*>(r4)[k];
#pragma unroll
        for (int j = 0; j < RW; ++j)
          if (lm >> j & 1u) {
            const float x = xr - cf[j * d + k];
            q32[j] = fmaf(x, x, q32[j]);
          }
      }
      const double ks = far32_scale(d);
#pragma unroll
      for (int j = 0; j < RW; ++j)
        if ((lm >> j & 1u) && far32(q32[j], ks, c)) lm &= ~(1u << j);
    }
  }
  if (v < n && lm) {
    const T* row = STAGE ? reinterpret_cast<const T*>(rs_smem) + (size_t)tid * pitch : V + v * pitch;
    auto step = [&](int k, double x) {
#pragma unroll
      for (int j = 0; j < RW; ++j)
        if (lm >> j & 1u) {
          const double t = x - cd[j * d + k];
          s[j] = fma(t, t, s[j]);
        }
    };
    int k = 0;
    if constexpr (sizeof(T) == 4) {
      for (; k + 16 <= d; k += 16) {  // 4 x LDG.128 in flight
        float4 q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          q[i] = STAGE ? reinterpret_cast<const float4*>(row)[(k >> 2) + i]
                       : __ldg(reinterpret_cast<const float4*>(row) + (k >> 2) + i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          step(k + 4 * i, (double)q[i].x);
          step(k + 4 * i + 1, (double)q[i].y);
          step(k + 4 * i + 2, (double)q[i].z);
          step(k + 4 * i + 3, (double)q[i].w);
        }
      }
      for (; k + 4 <= d; k += 4) {
        const float4 q = STAGE ? reinterpret_cast<const float4*>(row)[k >> 2]
                               : __ldg(reinterpret_cast<const float4*>(row) + (k >> 2));
        step(k, (double)q.x);
        step(k + 1, (double)q.y);
        step(k + 2, (double)q.z);
        step(k + 3, (double)q.w);
      }
    }
    for (; k < d; ++k) step(k, (double)row[k]);
  }
  if (v < n) {
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      const double t = c - s[j];
      if (j < wc) sb.xt[(int64_t)j * sb.xstride + v] = (lm >> j & 1u) && t > 0.0 ? t : 0.0;
    }
  }
  // the block taking the chunk's last ticket reduces it
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    flag = atomicAdd(sb.chunk_ticket + ch, 1u) == (unsigned)(SHORT_SPLIT - 1);
  }
  __syncthreads();
  if (!flag) return;
  __threadfence();
  // the classic reduction: thread t adds the terms of points t, t+256, t+512, t+768 in order
#pragma unroll
  for (int j = 0; j < RW; ++j) {
    double acc = 0.0;
    if (j < wc)
#pragma unroll
      for (int i = 0; i < RCH / RED_THREADS; ++i) {
        const int64_t w = (int64_t)ch * RCH + tid + i * RED_THREADS;
        if (w < n) acc += __ldcg(sb.xt + (int64_t)j * sb.xstride + w);
      }
    red[j][tid] = acc;
  }
  __syncthreads();
  if (warp < RW) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < RED_THREADS / 32; ++q) x += red[warp][lane * (RED_THREADS / 32) + q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && warp < wc) xch[(int64_t)warp * nchunks + ch] = x;
  }
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    sb.chunk_ticket[ch] = 0u;
    __threadfence();
    last = atomicAdd(fin.counter, 1u) == (unsigned)nchunks - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid == 0) *fin.counter = 0u;
  // group partials in the classic order: tot = 0; tot += chunk sums left to right
  const int cpg = (nchunks + ng - 1) / ng;
  for (int i = tid; i < wc * ng; i += blockDim.x) {
    const int w = i / ng, grp = i - w * ng;
    double tot = 0.0;
    const int c1 = min(nchunks, (grp + 1) * cpg);
    for (int q = grp * cpg; q < c1; ++q) tot += __ldcg(xch + (int64_t)w * nchunks + q);
    part_r[(int64_t)w * ng + grp] = tot;
  }
  __syncthreads();
  refine_finalize_n(fin, wc, wlist, part_r, ng, &red[0][0], reinterpret_cast<long long*>(&red[2][0]), RED_THREADS);
}

// ---------------------------------------------------------------- sharded exchange
// One rank's contribution to the global argmax.  Its local tie set
// T_r = {w in window : value_w >= top_r - 1e-12 max(1, |top_r|)} holds every
// candidate of the rank the reference rule can pick (the global threshold is
// >= every local one: top - window(top) is monotone in top, optimize.py:83-85).
// Of T_r only the index-ordered Pareto frontier is sent: c is kept iff every
// candidate of T_r with a lower index has a strictly lower value.  The global
// winner (lowest index with value >= the global threshold) is never dominated
// -- a dominating candidate would be eligible with a lower index -- so the
// union of the frontiers decides exactly as the union of the T_r would.  Exact
// duplicates collapse to their lowest index, so the frontier is almost always
// one entry.  Records: rec[0] = {count, 0}, rec[1 + i] = {index, exact gain}
// in increasing index (and value) order; a frontier longer than TIE_CAP is
// reported as count TIE_CAP + 1 (the caller falls back to the host exchange),
// never truncated silently.  TIE_CAP + 1 records = 128 B per rank and step.
constexpr int TIE_CAP = 7;

__global__ void __launch_bounds__(1024) k_tie_records(const int* __restrict__ wcount,
                                                      const int64_t* __restrict__ wlist,
                                                      const double* __restrict__ wgain, double inv_n,
                                                      const double* __restrict__ cur, double2* __restrict__ rec) {
  __shared__ double smax[1024];
  __shared__ long long sidx[1024];
  __shared__ double sgain[1024];
  const int t = threadIdx.x;
  const int wc = *wcount;
  const double f = *cur;
  double top = -INFINITY;
  for (int w = t; w < wc; w += blockDim.x) top = fmax(top, __dadd_rn(f, __dmul_rn(wgain[w], inv_n)));
  smax[t] = top;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) smax[t] = fmax(smax[t], smax[t + s]);
    __syncthreads();
  }
  top = smax[0];
  const double thr = top - 1e-12 * fmax(1.0, fabs(top));
  double prev = -INFINITY;  // value of the last frontier entry
  int cnt = 0;
  for (int it = 0; it <= TIE_CAP; ++it) {
    // next frontier entry: the lowest index whose value beats the previous entry
    long long bi = LLONG_MAX;
    double bg = 0.0;
    for (int w = t; w < wc; w += blockDim.x) {
      const double g = wgain[w];
      const double val = __dadd_rn(f, __dmul_rn(g, inv_n));
      const long long id = (long long)wlist[w];
      if (val >= thr && val > prev && id < bi) {
        bi = id;
        bg = g;
      }
    }
    sidx[t] = bi;
    sgain[t] = bg;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (t < s && sidx[t + s] < sidx[t]) {
        sidx[t] = sidx[t + s];
        sgain[t] = sgain[t + s];
      }
      __syncthreads();
    }
    bi = sidx[0];
    bg = sgain[0];
    __syncthreads();
    if (bi == LLONG_MAX) break;
    if (it == TIE_CAP) {
      cnt = TIE_CAP + 1;  // overflow: reported, not truncated
      break;
    }
    if (t == 0) rec[1 + it] = make_double2((double)bi, bg);
    cnt = it + 1;
    prev = __dadd_rn(f, __dmul_rn(bg, inv_n));
  }
  if (t == 0) rec[0] = make_double2((double)cnt, 0.0);
}

// Global pick over the all-gathered records of `world` ranks (identical input
// on every rank -> identical winner): top value, reference tie window, lowest
// index.  Marks the winner selected and records it as step `step`.
__global__ void __launch_bounds__(1024) k_pick_global(const double2* __restrict__ all, int world, double inv_n,
                                                      const double* __restrict__ cur, int64_t* __restrict__ best,
                                                      unsigned char* __restrict__ selected,
                                                      int64_t* __restrict__ sel_out, int step, int* __restrict__ err) {
  __shared__ double smax[1024];
  __shared__ long long smin[1024];
  const double f = *cur;
  double top = -INFINITY;
  for (int r = 0; r < world; ++r) {
    const double2* rr = all + (int64_t)r * (TIE_CAP + 1);
    const int cnt = (int)rr[0].x;
    if (cnt > TIE_CAP && threadIdx.x == 0) *err |= 1;
    for (int i = threadIdx.x; i < min(cnt, TIE_CAP); i += blockDim.x)
      top = fmax(top, __dadd_rn(f, __dmul_rn(rr[1 + i].y, inv_n)));
  }
  smax[threadIdx.x] = top;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
    __syncthreads();
  }
  top = smax[0];
  const double thr = top - 1e-12 * fmax(1.0, fabs(top));
  long long bi = LLONG_MAX;
  for (int r = 0; r < world; ++r) {
    const double2* rr = all + (int64_t)r * (TIE_CAP + 1);
    const int cnt = min((int)rr[0].x, TIE_CAP);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      if (__dadd_rn(f, __dmul_rn(rr[1 + i].y, inv_n)) >= thr) bi = min(bi, (long long)rr[1 + i].x);
  }
  smin[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) smin[threadIdx.x] = min(smin[threadIdx.x], smin[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const long long b = smin[0] == LLONG_MAX ? -1 : smin[0];
    *best = b;
    if (b >= 0) selected[b] = 1;
    if (sel_out) sel_out[step] = b;
  }
}

// End-of-run consistency guard of the sharded Greedy: a 64-bit hash of the k
// selected indices and the bits of their values and gains; every rank
// all-gathers the hashes and flags (err bit 2) any rank that disagrees.
__global__ void k_sel_hash(const int64_t* __restrict__ sel, const double* __restrict__ val,
                           const double* __restrict__ gain, int k, unsigned long long* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long h = 0xcbf29ce484222325ull;  // FNV-1a over 64-bit words
  auto mix = [&](unsigned long long x) {
    for (int b = 0; b < 8; ++b) {
      h ^= (x >> (8 * b)) & 0xffull;
      h *= 0x100000001b3ull;
    }
  };
  for (int s = 0; s < k; ++s) {
    mix((unsigned long long)sel[s]);
    mix((unsigned long long)__double_as_longlong(val[s]));
    mix((unsigned long long)__double_as_longlong(gain[s]));
  }
  *out = h;
}

__global__ void k_sel_hash_check(const unsigned long long* __restrict__ all, int world, int* __restrict__ err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int r = 1; r < world; ++r)
    if (all[r] != all[0]) *err |= 2;
}

// ---------------------------------------------------------------- K4: cached-min update

// cm64 = min(cm64, d64(., s)); pt = {-cm32, tau}; chunk partials of (e0d - cm64).
// The last block to finish turns the partials into f(S) and the step record.
// STAGE (fp32 rows, pitch <= UPDATE_STAGE_PITCH): each 256-point slice of the
// chunk is a contiguous run of rows; the block copies it into shared memory
// with coalesced 128-bit loads (the HBM-bound part of K4), then every thread
// computes its own point's distance from shared memory (LDS.128, conflict-free
// for an odd number of float4 per row) -- the same fp64 operation sequence.
constexpr int UPDATE_STAGE_PITCH = 132;

__device__ __forceinline__ double dist64_smem_row(const float* row, const double* cd, int d) {
  const float4* r4 = reinterpret_cast<const float4*>(row);
  double s = 0.0;
  int k = 0;
  for (; k + 4 <= d; k += 4) {
    const float4 x = r4[k >> 2];
    double t = (double)x.x - cd[k];
    s = fma(t, t, s);
    t = (double)x.y - cd[k + 1];
    s = fma(t, t, s);
    t = (double)x.z - cd[k + 2];
    s = fma(t, t, s);
    t = (double)x.w - cd[k + 3];
    s = fma(t, t, s);
  }
  for (; k < d; ++k) {
    const double t = (double)row[k] - cd[k];
    s = fma(t, t, s);
  }
  return s;
}

template <typename T>
__global__ void __launch_bounds__(RED_THREADS) k_update(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                        const int64_t* __restrict__ best, PtCoef pk,
                                                        const double* __restrict__ e0d, const float* __restrict__ nv32,
                                                        double* __restrict__ cm64, float4* __restrict__ pt,
                                                        TcSeeds seeds,
                                                        double* __restrict__ fpart,
                                                        unsigned int* __restrict__ counter, double inv_n,
                                                        double* __restrict__ cur, double* __restrict__ val_out,
                                                        double* __restrict__ gain_out, int step) {
  extern __shared__ double cd[];
  __shared__ double sbuf[RED_THREADS];
  __shared__ bool last;
  const int64_t s = *best;
  if (s < 0) return;
  for (int k = threadIdx.x; k < d; k += blockDim.x) cd[k] = (double)V[s * pitch + k];
  __syncthreads();
  double acc = 0.0;
  // the thread's 4 distances first (independent rows: their loads overlap),
  // then the updates and the sum in the fixed point order
  double tv[RCH / RED_THREADS];
#pragma unroll
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    const int64_t v = (int64_t)blockIdx.x * RCH + threadIdx.x + (int64_t)i * RED_THREADS;
    tv[i] = v < n ? dist64_row(V + v * pitch, cd, d) : 0.0;
  }
#pragma unroll
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    const int64_t v = (int64_t)blockIdx.x * RCH + threadIdx.x + (int64_t)i * RED_THREADS;
    if (v < n) {
      const double t = tv[i];
      double m = cm64[v];
      if (t < m) {
        m = t;
        cm64[v] = m;
        pt[v] = make_pt((float)m, nv32[v], pk);
        if (seeds.ipa) write_seeds(seeds, v, (float)m);
      }
      acc += e0d[v] - m;
    }
  }
  const double bs = block_sum_256(acc, sbuf);
  if (threadIdx.x == 0) {
    fpart[blockIdx.x] = bs;
    __threadfence();
    const unsigned int ticket = atomicAdd(counter, 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const double fnew = chunk_total_block(fpart, gridDim.x, sbuf) * inv_n;
    if (threadIdx.x == 0) {
      const double fold = *cur;
      if (val_out) val_out[step] = fnew;
      if (gain_out) gain_out[step] = fnew - fold;
      *cur = fnew;
      *counter = 0u;
    }
  }
}


// K4 for fp32 grounds, split in two so the HBM-bound part gets a wide grid:
// (a) k_update_terms -- one point per thread, 256-row slices of V staged in
//     shared memory with coalesced 128-bit loads (pitch <= UPDATE_STAGE_PITCH),
//     cached-min / seed updates, term[v] = e0d[v] - cm[v];
// (b) k_update_reduce -- the fixed chunk reduction of the terms (4 points per
//     thread in order, 256-thread tree, chunks left to right): bit-identical
//     to the fused kernel above.
template <bool STAGE>
__global__ void __launch_bounds__(RED_THREADS) k_update_terms(const float* __restrict__ V, int pitch, int64_t n,
                                                              int d, const int64_t* __restrict__ best, PtCoef pk,
                                                              const double* __restrict__ e0d,
                                                              const float* __restrict__ nv32,
                                                              double* __restrict__ cm64, float4* __restrict__ pt,
                                                              TcSeeds seeds, double* __restrict__ terms) {
  extern __shared__ double cd[];
  const int64_t s = *best;
  if (s < 0) return;
  for (int k = threadIdx.x; k < d; k += blockDim.x) cd[k] = (double)V[s * pitch + k];
  const int64_t v0 = (int64_t)blockIdx.x * RED_THREADS;
  const int64_t v = v0 + threadIdx.x;
  double t = 0.0;
  if constexpr (STAGE) {
    float* stage = reinterpret_cast<float*>(cd + ((d + 1) & ~1));  // 16-byte aligned after the candidate
    const int rows = (int)(n - v0 < RED_THREADS ? n - v0 : RED_THREADS);
    const float4* src = reinterpret_cast<const float4*>(V + v0 * pitch);
    float4* dst = reinterpret_cast<float4*>(stage);
    const int q4 = rows * (pitch >> 2);
    for (int q = threadIdx.x; q < q4; q += RED_THREADS) dst[q] = __ldcs(src + q);
    __syncthreads();
    if (v < n) t = dist64_smem_row(stage + threadIdx.x * pitch, cd, d);
  } else {
    __syncthreads();
    if (v < n) t = dist64_row(V + v * pitch, cd, d);
  }
  if (v < n) {
    double m = cm64[v];
    if (t < m) {
      m = t;
      cm64[v] = m;
      pt[v] = make_pt((float)m, nv32[v], pk);
      if (seeds.ipa) write_seeds(seeds, v, (float)m);
    }
    terms[v] = e0d[v] - m;
  }
}

__global__ void __launch_bounds__(RED_THREADS) k_update_reduce(const double* __restrict__ terms, int64_t n,
                                                               double* __restrict__ fpart,
                                                               unsigned int* __restrict__ counter, double inv_n,
                                                               double* __restrict__ cur, double* __restrict__ val_out,
                                                               double* __restrict__ gain_out, int step,
                                                               const int64_t* __restrict__ best) {
  __shared__ double sbuf[RED_THREADS];
  __shared__ bool last;
  if (*best < 0) return;
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    const int64_t v = (int64_t)blockIdx.x * RCH + threadIdx.x + (int64_t)i * RED_THREADS;
    if (v < n) acc += terms[v];
  }
  const double bs = block_sum_256(acc, sbuf);
  if (threadIdx.x == 0) {
    fpart[blockIdx.x] = bs;
    __threadfence();
    const unsigned int ticket = atomicAdd(counter, 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const double fnew = chunk_total_block(fpart, gridDim.x, sbuf) * inv_n;
    if (threadIdx.x == 0) {
      const double fold = *cur;
      if (val_out) val_out[step] = fnew;
      if (gain_out) gain_out[step] = fnew - fold;
      *cur = fnew;
      *counter = 0u;
    }
  }
}

// K4 fused (fp32 grounds): ONE launch per step streams V once and produces
// f(S) with exactly the fixed reduction structure of k_update_reduce.
//
// * One block per slice of UF_ROWS = 256 consecutive rows, one row per thread.
//   The slice (contiguous in HBM), its cm64 run and its e0d run arrive by three
//   cp.async.bulk copies on one mbarrier -- no register staging; several
//   blocks per SM keep ~200 KB per SM in flight.
// * Per row: the fp64 distance to the winner s in dist64_smem_row's operation
//   order, cm64 / pt / anchored-seed refresh for points whose minimum changed,
//   term[v] = e0d[v] - cm64[v] (to L2).
// * Chunk c (RCH = 1024 points = 4 slices): the block taking the chunk's last
//   ticket sums its terms in k_update_reduce's fixed order (thread u adds terms
//   u, u+256, u+512, u+768 left to right, then block_sum_256's tree) --
//   bit-identical; the block completing the last chunk adds the chunk partials
//   left to right (chunk_total_block) and records f(S).  Tickets are reset by
//   their last taker, so graph replays need no memset.
constexpr int UF_ROWS = RED_THREADS;
static_assert(RCH % UF_ROWS == 0, "a chunk is a whole number of slices");

struct UpdateCounters {
  unsigned int* chunk_ticket;  // nchunks
  unsigned int* chunks_done;   // 1
};

// UFR = rows per slice = threads per block (64, 128 or 256).  Smaller slices
// mean more, smaller blocks per SM, so one block's copy overlaps another's
// compute (the 256-row form waits for its 110 KB slice at C2 and runs 1.3
// waves of 2 blocks per SM).  A chunk's sum is always the 256-thread structure
// of k_update_reduce: with UFR < 256 every thread plays 256 / UFR of its
// virtual threads, the same additions in the same order.
template <int UFR>
__global__ void __launch_bounds__(UFR) k_update_fused(
    const float* __restrict__ V, int pitch, int64_t n, int d, const int64_t* __restrict__ best, PtCoef pk,
    const double* __restrict__ e0d, const float* __restrict__ nv32, double* __restrict__ cm64,
    float4* __restrict__ pt, TcSeeds seeds, double* __restrict__ terms, double* __restrict__ fpart,
    UpdateCounters ctr, double inv_n, double* __restrict__ cur, double* __restrict__ val_out,
    double* __restrict__ gain_out, int step) {
  static_assert(RED_THREADS % UFR == 0 && RCH % UFR == 0, "slices tile the chunk reduction");
  constexpr int VT = RED_THREADS / UFR;  // virtual reduction threads per thread
  extern __shared__ __align__(16) unsigned char uf_smem[];
  __shared__ uint64_t full;
  __shared__ double sbuf[RED_THREADS];
  __shared__ int flag;
  const int64_t s = *best;
  if (s < 0) return;
  const int t = threadIdx.x;
  const int id = blockIdx.x;
  const int nslices = gridDim.x;
  const int nchunks = (int)((n + RCH - 1) / RCH);
  // rows < n_pad: always a full slice; cm64 / e0d are allocated n_pad long
  const uint32_t row_bytes = (uint32_t)UFR * pitch * 4;
  double* cd = reinterpret_cast<double*>(uf_smem);
  float* cdf = reinterpret_cast<float*>(uf_smem + (((size_t)d * 8 + 15) & ~(size_t)15));  // fp32 copy
  unsigned char* stage = uf_smem + (((size_t)d * 8 + 15) & ~(size_t)15) + (((size_t)((d + 3) & ~3) * 4 + 15) & ~(size_t)15);
  if (t == 0) {
    mbar_init(&full, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&full, row_bytes + 2 * UFR * 8);
    bulk_g2s(stage, V + (int64_t)id * UFR * pitch, row_bytes, &full);
    bulk_g2s(stage + row_bytes, cm64 + (int64_t)id * UFR, UFR * 8, &full);
    bulk_g2s(stage + row_bytes + UFR * 8, e0d + (int64_t)id * UFR, UFR * 8, &full);
  }
  for (int k = t; k < d; k += UFR) {
    const float x = V[s * pitch + k];
    cd[k] = (double)x;
    cdf[k] = x;
  }
  __syncthreads();
  mbar_wait(&full, 0);
  const int64_t v = (int64_t)id * UFR + t;
  if (v < n) {
    const float* row = reinterpret_cast<const float*>(stage) + (size_t)t * pitch;
    double m = reinterpret_cast<const double*>(stage + row_bytes)[t];
    // far32 pre-test: the fp64 distance only where the winner may be closer than cm
    float q32 = 0.f;
    {
      const float4* r4 = reinterpret_cast<const float4*>(row);
      int k = 0;
      float qa = 0.f, qb = 0.f;
      for (; k + 4 <= d; k += 4) {
        const float4 q = r4[k >> 2];
        float x = q.x - cdf[k];
        qa = fmaf(x, x, qa);
        x = q.y - cdf[k + 1];
        qb = fmaf(x, x, qb);
        x = q.z - cdf[k + 2];
        qa = fmaf(x, x, qa);
        x = q.w - cdf[k + 3];
        qb = fmaf(x, x, qb);
      }
      for (; k < d; ++k) {
        const float x = row[k] - cdf[k];
        qa = fmaf(x, x, qa);
      }
      q32 = qa + qb;
    }
    if (!far32(q32, far32_scale(d), m)) {
      const double dist = dist64_smem_row(row, cd, d);
      if (dist < m) {
        m = dist;
        cm64[v] = m;
        pt[v] = make_pt((float)m, nv32[v], pk);
        if (seeds.ipa) write_seeds(seeds, v, (float)m);
      }
    }
    terms[v] = reinterpret_cast<const double*>(stage + row_bytes + UFR * 8)[t] - m;
  }
  __syncthreads();
  const int c = id / (RCH / UFR);
  if (t == 0) {
    const int in_chunk = min(RCH / UFR, nslices - c * (RCH / UFR));
    flag = ticket_acq_rel(ctr.chunk_ticket + c) == (unsigned int)(in_chunk - 1);
  }
  __syncthreads();
  if (!flag) return;
  // virtual thread u = t + q UFR: its 4 points u, u+256, u+512, u+768 in order
#pragma unroll
  for (int q = 0; q < VT; ++q) {
    const int u = t + q * UFR;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < RCH / RED_THREADS; ++i) {
      const int64_t w = (int64_t)c * RCH + u + (int64_t)i * RED_THREADS;
      if (w < n) acc += __ldcg(terms + w);
    }
    sbuf[u] = acc;
  }
  __syncthreads();
  // block_sum_256's tree over the virtual threads
#pragma unroll
  for (int st = RED_THREADS / 2; st > 0; st >>= 1) {
    for (int u = t; u < st; u += UFR) sbuf[u] += sbuf[u + st];
    __syncthreads();
  }
  const double bs = sbuf[0];
  __syncthreads();
  if (t == 0) {
    ctr.chunk_ticket[c] = 0u;
    fpart[c] = bs;
    flag = ticket_acq_rel(ctr.chunks_done) == (unsigned int)(nchunks - 1);
  }
  __syncthreads();
  if (!flag) return;
  // chunk partials left to right (chunk_total_block with this block's width)
  double fsum = 0.0;
  for (int c0 = 0; c0 < nchunks; c0 += UFR) {
    const int m = min(UFR, nchunks - c0);
    if (t < m) sbuf[t] = __ldcg(fpart + c0 + t);
    __syncthreads();
    if (t == 0)
      for (int i = 0; i < m; ++i) fsum += sbuf[i];
    __syncthreads();
  }
  const double fnew = fsum * inv_n;
  if (t == 0) {
    const double fold = *cur;
    if (val_out) val_out[step] = fnew;
    if (gain_out) gain_out[step] = fnew - fold;
    *cur = fnew;
    *ctr.chunks_done = 0u;
  }
}

// K4 fused with the NEXT lazy step's first batch (DESIGN.md §4 "update + batch"):
// each 256-row slice is staged once (bulk copies, as k_update_fused) and serves
// both the winner's distances -> cm (k_update_fused's operations) and, with the
// NEW cm, the batch candidates' terms (k_refine_short's operations: the
// sequential fp64 sum per (point, candidate), max(0, cm - d)).  A chunk's last
// ticket taker sums its f(S) terms (k_update_reduce's order) and its batch terms
// (the classic chunk reduction); the block completing the last chunk records
// f(S), then the batch's group partials and finalize, which decides the next
// step reading the f(S) it just wrote -- the same values as the two launches.
struct BatchArgs {
  const int* wcount = nullptr;
  const int64_t* wlist = nullptr;
  double* xch = nullptr;     // RW x nchunks chunk sums
  double* part_r = nullptr;  // RW x ng group partials
  int ng = 1;
  ShortBufs sb;              // xt terms (the per-chunk tickets are the update's)
  RefineFinal fin;
};

// fp32 Gram dots of one row (this lane's float4 range [k4b, k4e)) with the
// first NB batch rows and the winner (g[RW]) of the interleaved pack: packed
// FFMA2 on (even, odd) dim pairs, no per-candidate predicates (NB is a
// template argument).  far32_gram's bound holds for any summation order.
template <int NB>
__device__ __forceinline__ void gram_dots(const float4* __restrict__ r4, const float4* __restrict__ cgi, int k4b,
                                          int k4e, float (&g)[RW + 1]) {
  float2 a[NB + 1];
#pragma unroll
  for (int j = 0; j <= NB; ++j) a[j] = make_float2(0.f, 0.f);
  for (int k4 = k4b; k4 < k4e; ++k4) {
    const float4 q = r4[k4];
    const float2 q0 = make_float2(q.x, q.y), q1 = make_float2(q.z, q.w);
    const float4* c = cgi + k4 * (RW + 1);
#pragma unroll
    for (int j = 0; j <= NB; ++j) {
      const float4 c4 = c[j == NB ? RW : j];
      a[j] = __ffma2_rn(q0, make_float2(c4.x, c4.y), a[j]);
      a[j] = __ffma2_rn(q1, make_float2(c4.z, c4.w), a[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) g[j] = a[j].x + a[j].y;
  g[RW] = a[NB].x + a[NB].y;
}

// UFR rows per slice (64, 128 or 256; k_update_fused's virtual reduction
// threads).  Dynamic smem: the winner's row and the batch rows (fp64), then the
// slice stage, which the chunk reductions reuse once every row is consumed.
template <int UFR>
__global__ void __launch_bounds__(2 * UFR, UFR == 64 ? 5 : 3) k_update_batch(
    const float* __restrict__ V, int pitch, int64_t n, int d, const int64_t* __restrict__ best, PtCoef pk,
    const double* __restrict__ e0d, const float* __restrict__ nv32, double* __restrict__ cm64,
    float4* __restrict__ pt, TcSeeds seeds, double* __restrict__ terms, double* __restrict__ fpart,
    UpdateCounters ctr, double inv_n, double* __restrict__ cur, double* __restrict__ val_out,
    double* __restrict__ gain_out, int step, BatchArgs ba, const unsigned char* __restrict__ pack) {
  // two threads per row (a pair of adjacent lanes): each takes half of the fp32
  // Gram dots (combined by a shuffle: the far32_gram bound holds for any
  // summation order), the even lane the winner's exact distance, and the
  // batch's exact terms are split between the pair (candidate j on lane j & 1)
  constexpr int NT = 2 * UFR;
  static_assert(RED_THREADS % NT == 0 && RCH % UFR == 0 && UFR >= 64, "slices tile the chunk reduction");
  constexpr int VT = RED_THREADS / NT;
  constexpr int HW = RW / 2;  // batch candidates per lane
  extern __shared__ __align__(16) unsigned char uf_smem[];
  __shared__ uint64_t full;
  __shared__ int flag;
  const int64_t s = *best;
  if (s < 0) return;
  UB_TRACE_MIN(step, 0);
  UB_TRACE_MAX(step, 1);
  UB_TRACE_BLK(step, 0);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int r = t >> 1, p = t & 1;
  const unsigned pm = 3u << (lane & 30);  // the pair's lanes (the pair always branches together)
  const int id = blockIdx.x;
  const int nslices = gridDim.x;
  const int nchunks = (int)((n + RCH - 1) / RCH);
  const uint32_t row_bytes = (uint32_t)UFR * pitch * 4;
  const int dp = (d + 3) & ~3;
  const BatchPackLayout L(d);
  double* cd = reinterpret_cast<double*>(uf_smem);                     // the winner's row
  double* cb = reinterpret_cast<double*>(uf_smem + L.dbytes);          // the batch rows (RW x d)
  float* cg = reinterpret_cast<float*>(uf_smem + L.dbytes + L.cbytes);  // fp32 rows (RW batch + the winner), stride dp
  float* cn = cg + (size_t)(RW + 1) * dp;                               // their fp32 norms
  unsigned char* stage = uf_smem + L.bytes();
  double (*red)[RED_THREADS] = reinterpret_cast<double (*)[RED_THREADS]>(stage);  // after the rows
  double* sbuf = reinterpret_cast<double*>(stage) + RW * RED_THREADS;
  // launched as a programmatic dependent of k_lazy_topk (PDL): the rows, cm
  // and e0d do not depend on it and are staged while it runs; the pack and the
  // batch count are its output (after pdl_wait)
  if (t == 0) {
    mbar_init(&full, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&full, row_bytes + 2 * UFR * 8 + (uint32_t)L.bytes());
    bulk_g2s(stage, V + (int64_t)id * UFR * pitch, row_bytes, &full);
    bulk_g2s(stage + row_bytes, cm64 + (int64_t)id * UFR, UFR * 8, &full);
    bulk_g2s(stage + row_bytes + UFR * 8, e0d + (int64_t)id * UFR, UFR * 8, &full);
  }
  const int64_t v = (int64_t)id * UFR + r;
  const float nv = v < n ? nv32[v] : 0.f;  // in flight during the bulk copies
  pdl_wait();
  if (t == 0) bulk_g2s(uf_smem, pack, (uint32_t)L.bytes(), &full);
  const int wc = min(RW, *ba.wcount);
  __syncthreads();
  mbar_wait(&full, 0);
  UB_TRACE_MAX(step, 2);
  UB_TRACE_BLK(step, 1);
  if (v < n) {
    const float* row = reinterpret_cast<const float*>(stage) + (size_t)r * pitch;
    const float4* r4 = reinterpret_cast<const float4*>(row);
    // Gram-form fp32 pre-tests (far32_gram) for the winner and the batch: this
    // lane's half of the dims, then the pair's sum
    float g[RW + 1];
#pragma unroll
    for (int j = 0; j <= RW; ++j) g[j] = 0.f;
    const int h4 = (dp / 4 + 1) >> 1;
    const int k4b = p ? h4 : 0, k4e = p ? dp / 4 : h4;
    const float4* cgi = reinterpret_cast<const float4*>(cg);
    switch (wc) {
      case 0: gram_dots<0>(r4, cgi, k4b, k4e, g); break;
      case 1: gram_dots<1>(r4, cgi, k4b, k4e, g); break;
      case 2: gram_dots<2>(r4, cgi, k4b, k4e, g); break;
      case 3: gram_dots<3>(r4, cgi, k4b, k4e, g); break;
      case 4: gram_dots<4>(r4, cgi, k4b, k4e, g); break;
      case 5: gram_dots<5>(r4, cgi, k4b, k4e, g); break;
      case 6: gram_dots<6>(r4, cgi, k4b, k4e, g); break;
      case 7: gram_dots<7>(r4, cgi, k4b, k4e, g); break;
      default: gram_dots<RW>(r4, cgi, k4b, k4e, g); break;
    }
#pragma unroll
    for (int j = 0; j <= RW; ++j) g[j] += __shfl_xor_sync(pm, g[j], 1);
    double m = reinterpret_cast<const double*>(stage + row_bytes)[r];
    if (!far32_gram(g[RW], nv, cn[RW], d, m)) {
      double dist = 0.0;
      if (p == 0) dist = dist64_smem_row(row, cd, d);
      dist = __shfl_sync(pm, dist, lane & 30);  // the even lane's value to both
      if (dist < m) {
        m = dist;
        if (p == 0) {
          cm64[v] = m;
          pt[v] = make_pt((float)m, nv, pk);
          if (seeds.ipa) write_seeds(seeds, v, (float)m);
        }
      }
    }
    if (p == 0) terms[v] = reinterpret_cast<const double*>(stage + row_bytes + UFR * 8)[r] - m;
    // the batch's terms with the new minimum (k_refine_short's operation order),
    // fp64 only where the pre-test cannot rule the term out; candidate
    // j = 2 i + p on this lane
    unsigned lm = 0;
#pragma unroll
    for (int i = 0; i < HW; ++i) {
      const int j = 2 * i + p;
      if (j < wc && !far32_gram(g[j], nv, cn[j], d, m)) lm |= 1u << i;
    }
    double sj[HW];
#pragma unroll
    for (int i = 0; i < HW; ++i) sj[i] = 0.0;
    if (lm) {
      auto step_k = [&](int k, double x) {
#pragma unroll
        for (int i = 0; i < HW; ++i)
          if (lm >> i & 1u) {
            const double tt = x - cb[(2 * i + p) * d + k];
            sj[i] = fma(tt, tt, sj[i]);
          }
      };
      int k = 0;
      for (; k + 4 <= d; k += 4) {
        const float4 q = r4[k >> 2];
        step_k(k, (double)q.x);
        step_k(k + 1, (double)q.y);
        step_k(k + 2, (double)q.z);
        step_k(k + 3, (double)q.w);
      }
      for (; k < d; ++k) step_k(k, (double)row[k]);
    }
#pragma unroll
    for (int i = 0; i < HW; ++i) {
      const int j = 2 * i + p;
      if (j < wc) {
        const double tt = m - sj[i];
        ba.sb.xt[(int64_t)j * ba.sb.xstride + v] = (lm >> i & 1u) && tt > 0.0 ? tt : 0.0;
      }
    }
  }
  __syncthreads();  // every row consumed: the stage is reused below
  UB_TRACE_MAX(step, 3);
  UB_TRACE_BLK(step, 2);
#ifdef EBC200_TRACE
  if (threadIdx.x == 0 && step == 10 && blockIdx.x < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_ub_blk[blockIdx.x][3] = smid;
  }
#endif
  const int c = id / (RCH / UFR);
  if (t == 0) {
    const int in_chunk = min(RCH / UFR, nslices - c * (RCH / UFR));
    flag = ticket_acq_rel(ctr.chunk_ticket + c) == (unsigned int)(in_chunk - 1);
  }
  __syncthreads();
  if (!flag) return;
  // virtual thread u = t + q NT: the f(S) terms of points u, u+256, u+512, u+768
  // in order (k_update_reduce), and the batch terms likewise (k_refine_short);
  // every load of a virtual thread is issued before its adds
  constexpr int PPT = RCH / RED_THREADS;
#pragma unroll 1
  for (int q = 0; q < VT; ++q) {
    const int u = t + q * NT;
    double x[RW + 1][PPT];
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
      const int64_t w = (int64_t)c * RCH + u + (int64_t)i * RED_THREADS;
      x[0][i] = w < n ? __ldcg(terms + w) : 0.0;
#pragma unroll
      for (int j = 0; j < RW; ++j) x[j + 1][i] = w < n && j < wc ? __ldcg(ba.sb.xt + (int64_t)j * ba.sb.xstride + w) : 0.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < PPT; ++i)
      if ((int64_t)c * RCH + u + (int64_t)i * RED_THREADS < n) acc += x[0][i];
    sbuf[u] = acc;
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      double bj = 0.0;
#pragma unroll
      for (int i = 0; i < PPT; ++i)
        if (j < wc && (int64_t)c * RCH + u + (int64_t)i * RED_THREADS < n) bj += x[j + 1][i];
      red[j][u] = bj;
    }
  }
  __syncthreads();
  // block_sum_256's tree over the virtual threads
#pragma unroll
  for (int st = RED_THREADS / 2; st > 0; st >>= 1) {
    for (int u = t; u < st; u += NT) sbuf[u] += sbuf[u + st];
    __syncthreads();
  }
  for (int wj = warp; wj < RW; wj += NT / 32) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < RED_THREADS / 32; ++q) x += red[wj][lane * (RED_THREADS / 32) + q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && wj < wc) ba.xch[(int64_t)wj * nchunks + c] = x;
  }
  const double bs = sbuf[0];
  __syncthreads();
  if (t == 0) {
    ctr.chunk_ticket[c] = 0u;
    fpart[c] = bs;
    flag = ticket_acq_rel(ctr.chunks_done) == (unsigned int)(nchunks - 1);
  }
  __syncthreads();
  if (!flag) return;
  UB_TRACE_MAX(step, 4);
  // The last block: f(S) = the chunk partials left to right (chunk_total_block)
  // and each batch candidate's exact gain = its group partials (chunks
  // [g cpg, (g+1) cpg) left to right) summed left to right, in the same order
  // as the separate passes (identical bits).  Group partials of several chunks
  // are summed in parallel first; the chunk partials are streamed through
  // shared memory in tiles of RED_THREADS, one memory round trip per tile:
  // thread 32 sums f(S), thread j < wc candidate j (with one chunk per group,
  // cpg == 1, 0.0 + x == x, so the group step is a plain add).
  double fold = 0.0;
  if (t == 0) fold = *cur;
  double* tb = reinterpret_cast<double*>(stage);  // (RW + 1) x RED_THREADS tile
  double* tot_s = tb + (RW + 1) * RED_THREADS;     // wc exact gains, then f(S)
  const int ng = ba.ng;
  const int cpg = (nchunks + ng - 1) / ng;
  double* grp = tb + RED_THREADS;  // cpg > 1: wc x ng group partials (ng <= 256: batch_fusable)
  if (cpg > 1)
    for (int i = t; i < wc * ng; i += NT) {
      const int w = i / ng, gi = i - w * ng;
      const int q1 = min(nchunks, (gi + 1) * cpg);
      const double* src = ba.xch + (int64_t)w * nchunks;
      double tot = 0.0;
      int q = gi * cpg;
      for (; q + 8 <= q1; q += 8) {
        double x8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x8[e] = __ldcg(src + q + e);
#pragma unroll
        for (int e = 0; e < 8; ++e) tot += x8[e];
      }
      for (; q < q1; ++q) tot += __ldcg(src + q);
      grp[i] = tot;
    }
  double fsum = 0.0, gtot = 0.0;
  for (int c0 = 0; c0 < nchunks; c0 += RED_THREADS) {
    const int m = min(RED_THREADS, nchunks - c0);
    const int rows_in = cpg == 1 ? wc : 0;
#pragma unroll
    for (int rr = 0; rr <= RW; ++rr)
#pragma unroll
      for (int q = 0; q < RED_THREADS / NT; ++q) {
        const int cc = t + q * NT;
        if (cc < m && rr <= rows_in)
          tb[rr * RED_THREADS + cc] =
              rr == 0 ? __ldcg(fpart + c0 + cc) : __ldcg(ba.xch + (int64_t)(rr - 1) * nchunks + c0 + cc);
      }
    __syncthreads();
    if (t == 32) {
      int i = 0;
      for (; i + 8 <= m; i += 8) {
        double x8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x8[e] = tb[i + e];
#pragma unroll
        for (int e = 0; e < 8; ++e) fsum += x8[e];
      }
      for (; i < m; ++i) fsum += tb[i];
    }
    if (t < rows_in) {
      const double* row = tb + (t + 1) * RED_THREADS;
      int i = 0;
      for (; i + 8 <= m; i += 8) {
        double x8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) x8[e] = row[i + e];
#pragma unroll
        for (int e = 0; e < 8; ++e) gtot += x8[e];
      }
      for (; i < m; ++i) gtot += row[i];
    }
    __syncthreads();
  }
  if (cpg > 1 && t < wc) {
    const double* gp = grp + t * ng;
    int i = 0;
    for (; i + 8 <= ng; i += 8) {
      double x8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x8[e] = gp[i + e];
#pragma unroll
      for (int e = 0; e < 8; ++e) gtot += x8[e];
    }
    for (; i < ng; ++i) gtot += gp[i];
  }
  if (t < wc) tot_s[t] = gtot;
  if (t == 32) tot_s[RW] = fsum * inv_n;
  __syncthreads();
  const double fnew = tot_s[RW];
  if (t == 0) {
    if (val_out) val_out[step] = fnew;
    if (gain_out) gain_out[step] = fnew - fold;
    *cur = fnew;
    *ctr.chunks_done = 0u;
  }
  UB_TRACE_MAX(step, 5);
  // the batch's finalize on the exact gains, f(S) from shared memory, on warp 0
  if (warp == 0) refine_finalize_warp(ba.fin, wc, ba.wlist, tot_s, tot_s + RW);
  UB_TRACE_MAX(step, 6);
}

// ---------------------------------------------------------------- K2: multiset (work matrix)

// part[j*nchunks + ch] = sum over chunk ch of (e0d[v] - min(e0d[v], min_{s in S_j} d64(v, s))).
// One block per (chunk, set); members are read through L1 (broadcast across the block).
template <typename T>
__global__ void __launch_bounds__(RED_THREADS) k_multiset(const T* __restrict__ V, int pitch, int64_t n, int d,
                                                          const double* __restrict__ e0d,
                                                          const int64_t* __restrict__ offsets,
                                                          const int64_t* __restrict__ idx, int64_t set0,
                                                          int nchunks, double* __restrict__ part) {
  __shared__ double sbuf[RED_THREADS];
  const int ch = blockIdx.x;
  const int64_t j = set0 + blockIdx.y;
  const int64_t m0 = offsets[j], m1 = offsets[j + 1];
  double acc = 0.0;
  for (int i = 0; i < RCH / RED_THREADS; ++i) {
    const int64_t v = (int64_t)ch * RCH + threadIdx.x + (int64_t)i * RED_THREADS;
    if (v < n) {
      const double base = e0d[v];
      double m = base;
      const T* row = V + v * pitch;
      for (int64_t p = m0; p < m1; ++p) {
        const T* mem = V + idx[p] * pitch;
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
          const double t = (double)row[k] - (double)__ldg(mem + k);
          s = fma(t, t, s);
        }
        m = fmin(m, s);
      }
      acc += base - m;
    }
  }
  const double bs = block_sum_256(acc, sbuf);
  if (threadIdx.x == 0) part[blockIdx.y * (int64_t)nchunks + ch] = bs;
}

__global__ void k_multiset_final(const double* __restrict__ part, int64_t l, int nchunks, double inv_n,
                                 double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < l) out[j] = chunk_total(part + j * nchunks, nchunks) * inv_n;
}

}  // namespace ebc
