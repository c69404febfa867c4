// screen_tc.cuh -- tcgen05 (5th-gen tensor core) Gram-form candidate screen.
//
// Same contract as k_screen<Cfg, GRAM=true> (kernels.cuh): for a tile of 128
// candidates, accumulate over all points gain/2 = sum_v max(0, t/2) with
// t/2 = (cm - |v|^2 - |c|^2)/2 + v.c, plus a certified error bound -- but the
// dot products v.c come from tcgen05.mma (kind::tf32) instead of FFMA:
//
//   v.c ~= hi(v).hi(c) + hi(v).lo(c) + lo(v).hi(c)      ("3xTF32")
//
// with hi = x truncated to TF32 and lo = x - hi, so every product carries
// ~2^-20 relative error and the fp32 accumulation in TMEM adds at most
// (3 Kpad + 16) 2^-23 relative to sum |v_k c_k| (DESIGN.md §4 "tensor screen").
//
// CTA = 6 warps:  warp 0 = bulk-copy producer + TMEM allocator,
//                 warp 1 = MMA issuer (one elected lane),
//                 warps 2..5 = epilogue, one candidate per thread (= TMEM lane).
// Operands are staged by the bulk-copy engine straight from pre-split,
// UMMA-canonical copies of V (K-major, no swizzle: 8-row x 16-byte core
// matrices, LBO = 128 B between K chunks, SBO = Kpad*32 B between row groups),
// so no thread touches operand data.  Accumulators: 2 TMEM buffers of NP
// columns (M = 128 lanes = candidates, N = NP points), double-buffered against
// the epilogue; V tiles: 2-stage smem ring.
#pragma once
#include <cstdint>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace ebc {
namespace tc {

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// smem matrix descriptor: K-major, SWIZZLE_NONE, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor: kind::tf32, D fp32, A/B tf32, both K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::f16 with BF16 A/B, fp32 D, both K-major
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::f16 with FP16 A/B (format 0), fp32 D, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Operand kinds of the tensor screen.
//   KIND_TF32: 3xTF32 split (kind::tf32), KIND_BF16: 3-product BF16 split
//   (kind::f16), KIND_F16: FP16-stored grounds, one exact FP16 product per
//   element (fp16 x fp16 has 22 significant bits: exact in the fp32 accumulator),
//   KIND_F16R: fp32 grounds scaled by s = 2^e and ROUNDED to fp16, one product
//   per element: relative operand error 2^-11 each, so the certified bound is
//   ~2^-10 |v| |c'| per pair (vs ~2^-16 for the BF16 split) at a third of the
//   MMA work -- the first rung when the BF16 split is MMA-bound (large d).
enum { KIND_TF32 = 0, KIND_BF16 = 1, KIND_F16 = 2, KIND_F16R = 3 };
__host__ __device__ constexpr bool one_product(int kind) { return kind == KIND_F16 || kind == KIND_F16R; }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 64 consecutive accumulator columns of this warp's lanes, one wait.
__device__ __forceinline__ void ld64(uint32_t taddr, float (&v)[64]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, "
      "%36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, "
      "%57, %58, %59, %60, %61, %62, %63}, [%64];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int W>
__device__ __forceinline__ void ldcols(uint32_t taddr, float (&v)[W]) {
  if constexpr (W == 64) {
    ld64(taddr, v);
  } else if constexpr (W == 16) {
    ld16(taddr, v);
  } else {
    static_assert(W % 32 == 0, "columns per thread: multiple of 32");
#pragma unroll
    for (int h = 0; h < W / 32; ++h) {
      float t[32];
      ld32(taddr + 32 * h, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[32 * h + i] = t[i];
    }
  }
}

constexpr int M = 128;        // candidates per CTA (UMMA M)
#ifndef EBC200_EPI_FADD2
#define EBC200_EPI_FADD2 1
#endif
#ifndef EBC200_SPEC
#define EBC200_SPEC 1  // speculative slow path in the split-rung epilogue (k_screen_tc)
#endif
#ifndef EBC200_EPI_WARPGROUPS
#define EBC200_EPI_WARPGROUPS 2
#endif
constexpr int EPI_WARPGROUPS = EBC200_EPI_WARPGROUPS;  // epilogue warpgroups (slices of the point columns)
constexpr int MMA_WARPS = 3;       // one issuing warp per accumulator buffer (tiles round-robin)
constexpr int EPI_WARP0 = 1 + MMA_WARPS;
constexpr int THREADS = 32 * EPI_WARP0 + 128 * EPI_WARPGROUPS;  // producer + MMA warps + epilogue
// accumulator buffers: BF16 operands (A = 2 x 56 columns) leave room for 3 x 128
// fp32 accumulators in the 512 TMEM columns, TF32 (A = 2 x 128) for 2
template <int KIND>
struct TmemMap {
  static constexpr bool W16 = KIND != KIND_TF32;  // 16-bit operands: 2 elements per TMEM column
  static constexpr int NB = W16 ? 3 : 2;
  static constexpr uint32_t ALO = W16 ? 64 : 128;
  static constexpr uint32_t ACC = W16 ? 128 : 256;
  static constexpr int PARTS = one_product(KIND) ? 1 : 2;  // operand parts per point tile
  static constexpr int ES = W16 ? 2 : 4;                  // operand element bytes
};
constexpr int MAX_STAGES = 4;
// TMEM columns: A_hi [0,128), A_lo [128,256), accumulators [256 + b*NP, ...)
constexpr uint32_t COL_AHI = 0, COL_ALO = 128, COL_ACC = 256, TMEM_COLS = 512;

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0)
      : "memory");
}

// The three 3xTF32 products of one K step in a single asm block: hi.hi (sets
// or accumulates), hi.lo, lo.hi.  One statement = one issue sequence.
__device__ __forceinline__ void mma3_tf32_ts(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi,
                                             uint64_t b_lo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 q, %6, %6;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, {%7, %7, %7, %7}, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, {%7, %7, %7, %7}, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, {%7, %7, %7, %7}, q;\n\t}\n" ::"r"(tmem_d),
      "r"(a_hi), "r"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(acc), "r"(0)
      : "memory");
}

// One FP16 product per K step (KIND_F16).
__device__ __forceinline__ void mma1_f16_ts(uint32_t tmem_d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0)
      : "memory");
}

// Same for the BF16 split (kind::f16, K = 16 per instruction).
__device__ __forceinline__ void mma3_bf16_ts(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi,
                                             uint64_t b_lo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 q, %6, %6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, {%7, %7, %7, %7}, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, {%7, %7, %7, %7}, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, {%7, %7, %7, %7}, q;\n\t}\n" ::"r"(tmem_d),
      "r"(a_hi), "r"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(acc), "r"(0)
      : "memory");
}

__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

inline int stages_for(int kpad, int np, int es = 4, int parts = 2, size_t list_bytes = 0) {
  const size_t stage = (size_t)parts * np * kpad * es;
  const size_t budget = 220 * 1024 - list_bytes;
  int st = (int)(budget / stage);
  return st > MAX_STAGES ? MAX_STAGES : st;
}

// the kept-tile list (uint16 per point tile of the CTA's split) follows the barriers
__host__ __device__ constexpr size_t list_bytes_for(int tps) { return ((size_t)tps * 2 + 15) / 16 * 16; }

inline size_t smem_bytes(int kpad, int np, int es = 4, int parts = 2, size_t list_bytes = 0) {
  const size_t stage = (size_t)parts * np * kpad * es;  // B_hi (, B_lo)
  size_t ring = stages_for(kpad, np, es, parts, list_bytes) * stage;
  const size_t xchg = EPI_WARPGROUPS * 128 * (sizeof(double) + sizeof(float));  // slice exchange reuses the ring
  if (ring < xchg) ring = xchg;
  return ring + (2 * MAX_STAGES + 8) * sizeof(uint64_t) + 64 + list_bytes;
}

}  // namespace tc

// Split V into TF32 hi/lo parts in the UMMA canonical K-major blocked layout:
// element (v, k) at ((v/8 * KC + k/4) * 8 + v%8) * 4 + k%4, KC = kpad/4.
__global__ void k_split_tf32(const float* __restrict__ V32, int pitch, int64_t nrows, int d, int kpad,
                             float* __restrict__ hi, float* __restrict__ lo) {
  const int KC = kpad / 4;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = nrows * kpad;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / kpad;
    const int k = (int)(i - v * kpad);
    const float x = k < d ? V32[v * pitch + k] : 0.f;
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    const float l = x - h;  // exact
    const int64_t off = (((v >> 3) * KC + (k >> 2)) * 8 + (v & 7)) * 4 + (k & 3);
    hi[off] = h;
    lo[off] = l;
  }
}

// BF16 split: x = h + m + l, h = bf16(x), m = bf16(x - h); the screen uses h, m.
// Layout as above with 8-element (16-byte) chunks: element (v, k) at
// ((v/8 * KC + k/8) * 8 + v%8) * 8 + k%8, KC = kpad/8.
__global__ void k_split_bf16(const float* __restrict__ V32, int pitch, int64_t nrows, int d, int kpad,
                             __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int KC = kpad / 8;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = nrows * kpad;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / kpad;
    const int k = (int)(i - v * kpad);
    const float x = k < d ? V32[v * pitch + k] : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 m = __float2bfloat16_rn(x - __bfloat162float(h));
    const int64_t off = (((v >> 3) * KC + (k >> 3)) * 8 + (v & 7)) * 8 + (k & 7);
    hi[off] = h;
    lo[off] = m;
  }
}

// FP16 grounds: V (exactly widened to fp32) back to fp16, same blocked layout
// (scale 1: exact).  KIND_F16R: fp16(scale * x), scale a power of two.
__global__ void k_split_f16(const float* __restrict__ V32, int pitch, int64_t nrows, int d, int kpad,
                            __half* __restrict__ hi, float scale = 1.f) {
  const int KC = kpad / 8;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = nrows * kpad;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / kpad;
    const int k = (int)(i - v * kpad);
    const float x = k < d ? V32[v * pitch + k] : 0.f;
    const int64_t off = (((v >> 3) * KC + (k >> 3)) * 8 + (v & 7)) * 8 + (k & 7);
    hi[off] = __float2half_rn(x * scale);
  }
}

// ---------------------------------------------------------------- anchors
// The tensor screen computes v.c' with c' = c - mu_a, mu_a the anchor of the
// candidate tile (anchor 0 = the origin, the plain Gram form).  Its error scales
// with |v| |c'| instead of |v|^2 + |c|^2, so clustered data (C4) keeps narrow
// windows.  Anchors: farthest-point sampling from the origin; each 128-candidate
// block takes the anchor that minimises max |c - mu_a|.  Every choice is valid --
// the bounds use each candidate's own |c'| -- the choice only sets their width.

__device__ __forceinline__ unsigned long long fps_key(float dist, int64_t v) {
  return ((unsigned long long)__float_as_uint(fmaxf(dist, 0.f)) << 32) | (0xFFFFFFFFull - (unsigned long long)v);
}

// Step a of farthest-point sampling: anchor a is the origin (a = 0) or the
// point keyed in keys[a]; fold it into mind and key the next farthest point.
__global__ void k_fps_step(const float* __restrict__ V32, int pitch, int64_t n, int d, int a, int na,
                           float* __restrict__ mind, unsigned long long* __restrict__ keys,
                           float* __restrict__ anchors, int apitch) {
  __shared__ unsigned long long sk[32];
  int64_t src = -1;
  if (a > 0) src = (int64_t)(0xFFFFFFFFull - (keys[a] & 0xFFFFFFFFull));
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < apitch; k += blockDim.x)
      anchors[(int64_t)a * apitch + k] = (src >= 0 && k < d) ? V32[src * pitch + k] : 0.f;
  unsigned long long best = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    float t = 0.f;
    const float* row = V32 + v * pitch;
    if (src >= 0) {
      const float* mu = V32 + src * pitch;
      for (int k = 0; k < d; ++k) {
        const float x = row[k] - mu[k];
        t = fmaf(x, x, t);
      }
    } else {
      for (int k = 0; k < d; ++k) t = fmaf(row[k], row[k], t);
    }
    const float m = a == 0 ? t : fminf(mind[v], t);
    mind[v] = m;
    const unsigned long long key = fps_key(m, v);
    best = key > best ? key : best;
  }
  if (a + 1 >= na) return;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffff, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) sk[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = sk[w] > best ? sk[w] : best;
    atomicMax(&keys[a + 1], best);
  }
}

// All of farthest-point sampling in one cooperative launch: the same per-step
// arithmetic and keys as k_fps_step (so the same anchors), one grid barrier per
// anchor instead of one launch per anchor.  bar: two zeroed words.
__device__ __forceinline__ void fps_grid_barrier(unsigned int* bar, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int nb = gridDim.x;
    if (atomicAdd(bar, 1u) == nb - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*(volatile unsigned int*)(bar + 1) == gen) __nanosleep(32);
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}
__global__ void __launch_bounds__(256) k_fps_all(const float* __restrict__ V32, int pitch, int64_t n, int d, int na,
                                                 float* __restrict__ mind, unsigned long long* __restrict__ keys,
                                                 float* __restrict__ anchors, int apitch, unsigned int* bar) {
  extern __shared__ float fmu[];  // (d + 3) / 4 * 4: the current anchor, zero padded
  __shared__ unsigned long long sk[8];
  unsigned int gen = *(volatile unsigned int*)(bar + 1);
  for (int a = 0; a < na; ++a) {
    int64_t src = -1;
    if (a > 0) src = (int64_t)(0xFFFFFFFFull - (__ldcg(keys + a) & 0xFFFFFFFFull));
    for (int k = threadIdx.x; k < (d + 3) / 4 * 4; k += blockDim.x) {
      const float x = src >= 0 && k < d ? V32[src * pitch + k] : 0.f;
      fmu[k] = x;
      if (blockIdx.x == 0 && k < d) anchors[(int64_t)a * apitch + k] = x;
    }
    if (blockIdx.x == 0)
      for (int k = d + threadIdx.x; k < apitch; k += blockDim.x) anchors[(int64_t)a * apitch + k] = 0.f;
    __syncthreads();
    unsigned long long best = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
      // rows are 16-byte aligned (pitch % 4 == 0, zero-padded past d, fmu too):
      // four independent partial sums over 128-bit loads (any order is fine --
      // anchors only steer the bounds, every choice is certified)
      const float4* row4 = reinterpret_cast<const float4*>(V32 + v * pitch);
      float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
      for (int k4 = 0; k4 < (d + 3) / 4; ++k4) {
        const float4 r = __ldg(row4 + k4);
        const float x0 = r.x - fmu[4 * k4], x1 = r.y - fmu[4 * k4 + 1];
        const float x2 = r.z - fmu[4 * k4 + 2], x3 = r.w - fmu[4 * k4 + 3];
        t0 = fmaf(x0, x0, t0);
        t1 = fmaf(x1, x1, t1);
        t2 = fmaf(x2, x2, t2);
        t3 = fmaf(x3, x3, t3);
      }
      const float t = (t0 + t1) + (t2 + t3);
      const float m = a == 0 ? t : fminf(mind[v], t);
      mind[v] = m;
      const unsigned long long key = fps_key(m, v);
      best = key > best ? key : best;
    }
    if (a + 1 >= na) break;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffff, best, o);
      best = other > best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) sk[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = sk[w] > best ? sk[w] : best;
      atomicMax(&keys[a + 1], best);
    }
    fps_grid_barrier(bar, gen);
  }
}

// nva[a][v] = |v - mu_a|^2 (fp64 sum, rounded to fp32) for every anchor.
__global__ void k_nva(const float* __restrict__ V32, int pitch, int64_t n, int d, const float* __restrict__ anchors,
                      int apitch, int na, float* __restrict__ nva, int64_t stride) {
  const int64_t total = (int64_t)na * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(i / n);
    const int64_t v = i - (int64_t)a * n;
    const float* row = V32 + v * pitch;
    const float* mu = anchors + (int64_t)a * apitch;
    double t = 0.0;
    for (int k = 0; k < d; ++k) {
      const double x = (double)row[k] - (double)mu[k];
      t = fma(x, x, t);
    }
    nva[a * stride + v] = (float)t;
  }
}

// The same values, one thread per point for every anchor at once (anchors
// staged in shared memory; the per-(anchor, point) fp64 sum in the same order).
constexpr int NA_ALL = 32;
__global__ void __launch_bounds__(128) k_nva_all(const float* __restrict__ V32, int pitch, int64_t n, int d,
                                                 const float* __restrict__ anchors, int apitch, int na,
                                                 float* __restrict__ nva, int64_t stride) {
  extern __shared__ double amd[];  // na x dp anchors in fp64 (converted once), zero padded (dp = d rounded
                                   // up to 4; rows are zero padded too, so the extra terms add exactly 0)
  const int dp = (d + 3) / 4 * 4;
  for (int i = threadIdx.x; i < na * dp; i += blockDim.x) {
    const int a = i / dp, k = i - a * dp;
    amd[i] = k < d ? (double)anchors[(int64_t)a * apitch + k] : 0.0;
  }
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double acc[NA_ALL];
#pragma unroll
  for (int a = 0; a < NA_ALL; ++a) acc[a] = 0.0;
  const float4* row4 = reinterpret_cast<const float4*>(V32 + v * pitch);
  for (int k4 = 0; k4 < dp / 4; ++k4) {
    const float4 r = __ldg(row4 + k4);
    const double r0 = r.x, r1 = r.y, r2 = r.z, r3 = r.w;
#pragma unroll
    for (int a = 0; a < NA_ALL; ++a)
      if (a < na) {
        const double2 m01 = *reinterpret_cast<const double2*>(amd + a * dp + 4 * k4);
        const double2 m23 = *reinterpret_cast<const double2*>(amd + a * dp + 4 * k4 + 2);
        double t = r0 - m01.x;
        acc[a] = fma(t, t, acc[a]);
        t = r1 - m01.y;
        acc[a] = fma(t, t, acc[a]);
        t = r2 - m23.x;
        acc[a] = fma(t, t, acc[a]);
        t = r3 - m23.y;
        acc[a] = fma(t, t, acc[a]);
      }
  }
#pragma unroll
  for (int a = 0; a < NA_ALL; ++a)
    if (a < na) nva[a * stride + v] = (float)acc[a];
}

// Per 128-candidate block: the anchor minimising max_c |c - mu_a|^2 (ties: lower a).
// na <= NA_ALL: every thread sums its candidate against all anchors at once
// (anchors in shared memory, dynamic smem na x d floats); larger na loops.
__global__ void __launch_bounds__(128) k_tile_anchor(const float* __restrict__ V32, int pitch, int64_t n, int d,
                                                     const float* __restrict__ anchors, int apitch, int na,
                                                     int* __restrict__ tile_anchor, float* __restrict__ tile_rad,
                                                     int staged, const int* __restrict__ n_dev = nullptr,
                                                     const int* __restrict__ level_now = nullptr, int level = 0) {
  // n_dev: a device-side row count (gathered lazy re-screens; blocks past it exit)
  if (level_now && *level_now != level) return;
  if (n_dev) n = min(n, (int64_t)*n_dev);
  if ((int64_t)blockIdx.x * 128 >= n) return;
  extern __shared__ float tmu[];  // na x d (na <= NA_ALL)
  __shared__ float wm[4][NA_ALL];
  __shared__ float wmax[4];
  const int64_t c = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float best = INFINITY;
  int besta = 0;
  if (staged) {  // host: na <= NA_ALL and na x dp floats of dynamic smem
    // anchors zero padded to dp (rows are zero padded too: the extra terms add
    // exactly 0, so the sums equal the looped form's)
    const int dp = (d + 3) / 4 * 4;
    for (int i = threadIdx.x; i < na * dp; i += blockDim.x) {
      const int a = i / dp, k = i - a * dp;
      tmu[i] = k < d ? anchors[(int64_t)a * apitch + k] : 0.f;
    }
    __syncthreads();
    float t[NA_ALL];
#pragma unroll
    for (int a = 0; a < NA_ALL; ++a) t[a] = 0.f;
    if (c < n) {
      const float4* row4 = reinterpret_cast<const float4*>(V32 + c * pitch);
      for (int k4 = 0; k4 < dp / 4; ++k4) {
        const float4 r = __ldg(row4 + k4);
#pragma unroll
        for (int a = 0; a < NA_ALL; ++a)
          if (a < na) {
            const float4 m = *reinterpret_cast<const float4*>(tmu + a * dp + 4 * k4);
            float x = r.x - m.x;
            t[a] = fmaf(x, x, t[a]);
            x = r.y - m.y;
            t[a] = fmaf(x, x, t[a]);
            x = r.z - m.z;
            t[a] = fmaf(x, x, t[a]);
            x = r.w - m.w;
            t[a] = fmaf(x, x, t[a]);
          }
      }
    }
#pragma unroll
    for (int a = 0; a < NA_ALL; ++a) {
      float m = t[a];
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
      if (lane == 0) wm[warp][a] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int a = 0; a < na; ++a) {
        const float m = fmaxf(fmaxf(wm[0][a], wm[1][a]), fmaxf(wm[2][a], wm[3][a]));
        if (m < best) {
          best = m;
          besta = a;
        }
      }
  } else {
    for (int a = 0; a < na; ++a) {
      float t = 0.f;
      if (c < n) {
        const float* row = V32 + c * pitch;
        const float* mu = anchors + (int64_t)a * apitch;
        for (int k = 0; k < d; ++k) {
          const float x = row[k] - mu[k];
          t = fmaf(x, x, t);
        }
      }
      for (int o = 16; o > 0; o >>= 1) t = fmaxf(t, __shfl_xor_sync(0xffffffff, t, o));
      if (lane == 0) wmax[warp] = t;
      __syncthreads();
      const float m = fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3]));
      if (m < best) {
        best = m;
        besta = a;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    tile_anchor[blockIdx.x] = besta;
    // R = max_c |c - mu| rounded up (fp32 sum error (d+2)u << 1e-5)
    if (tile_rad) tile_rad[blockIdx.x] = sqrtf(best) * (1.f + 1e-5f) + 1e-30f;
  }
}

// Seeds from the cached minima for every anchor; padded points get -1e30 so
// they can never contribute (a = S + ip + ic stays hugely negative).
__global__ void k_seed_ipa(const double* __restrict__ cm64, int64_t n, int64_t n_pad, TcSeeds seeds) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) {
    write_seeds(seeds, v, (float)cm64[v]);
  } else if (v < n_pad) {
    for (int a = 0; a < seeds.na; ++a) seeds.ipa[a * seeds.stride + v] = -1e30f;
    // MMA seeds: -2^14 / s2 <= -(max |ip|), far below any -kq (the candidate side
    // of the origin form, ic = -|c|^2/2, is <= 0)
    if (seeds.ops) write_seed_parts(seeds, v, -16384.f);
  }
}

// kpmax[a][t] = max over the NP points of tile t of kp = KP (cm32 + nva_a) at
// reset (cm = d(., e0)); cm only decreases within a run, so it bounds every step.
// vmax[t] = max |v| over the tile (rounded up).
__global__ void k_tile_kpmax(const double* __restrict__ e0d, const float* __restrict__ nv32,
                             const float* __restrict__ nva, int64_t stride, int na, int64_t n, int64_t ntiles,
                             int np, float kp_coef, float* __restrict__ kpmax, float* __restrict__ vmax,
                             float* __restrict__ rho, float* __restrict__ rhomax = nullptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)na * ntiles) return;
  const int a = (int)(i / ntiles);
  const int64_t t = i - (int64_t)a * ntiles;
  float m = 0.f, vm = 0.f, rm = INFINITY, rx = 0.f;
  for (int j = 0; j < np; ++j) {
    const int64_t v = t * np + j;
    if (v < n) {
      const float q = nva[a * stride + v];
      m = fmaxf(m, kp_coef * ((float)e0d[v] + q));
      vm = fmaxf(vm, nv32[v]);
      rm = fminf(rm, q);
      rx = fmaxf(rx, q);
    }
  }
  // rhomax = max_v |v - mu_a| rounded up (all-positive tile test, k_screen_agg)
  if (rhomax) rhomax[a * ntiles + t] = sqrtf(rx) * (1.f + 1e-5f) + 1e-30f;
  kpmax[a * ntiles + t] = m * (1.f + 1e-6f);
  if (a == 0) vmax[t] = sqrtf(vm) * (1.f + 1e-5f);
  // rho = min_v |v - mu_a| rounded down (nva is the fp64 value rounded to fp32)
  rho[a * ntiles + t] = sqrtf(rm) * (1.f - 1e-5f);
}

// cmx[t] = max over the tile's points of the cached minimum (rounded up).
__global__ void k_tile_cmmax(const double* __restrict__ cm64, int64_t n, int64_t ntiles, int np,
                             float* __restrict__ cmx, float* __restrict__ cmn = nullptr) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  double m = 0.0, mn = INFINITY;
  for (int j = lane; j < np; j += 32) {
    const int64_t v = t * np + j;
    if (v < n) {
      m = fmax(m, cm64[v]);
      mn = fmin(mn, cm64[v]);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffff, m, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffff, mn, o));
  }
  if (lane == 0) {
    cmx[t] = __double2float_ru(m);
    if (cmn) cmn[t] = __double2float_rd(mn);  // min cm over the tile, rounded down
  }
}

// ---------------------------------------------------------------- all-positive tiles
// A (candidate block, point tile) pair whose every pair is certified to have
// d(v, c) < cm(v) -- (max_v |v - mu| + max_c |c - mu|)^2 < min_v cm(v), the
// triangle inequality through the block's anchor -- has max(0, a) = a for every
// pair, so its contribution to the gain is the LINEAR sum
//   sum_v a_v = sum_v ip_mu(v) + c'.(sum_v v) + n_t ic
// computed from per-tile aggregates (k_screen_agg) instead of 128 x 128 MMA
// terms.  Early Greedy steps on clustered data (C4) are dominated by such
// tiles: at step 0 cm = |v|^2 exceeds every inter-regime distance.
__device__ __forceinline__ bool tile_allpos(float rhomax, float rad, float cmn) {
  const float r = __fadd_ru(rhomax, rad);
  return __fmul_ru(__fmul_ru(r, r), 1.00001f) < cmn;
}

// vsum[t][k] = sum of the tile's (real) points, fp64 accumulation rounded to
// fp32; vsn[t] = |vsum[t]| rounded up.  One block per tile.
// rhomin[t] = min over anchors of rhomax[a][t] (the any-block screen of k_tile_ipsum)
__global__ void k_tile_rhomin(const float* __restrict__ rhomax, int na, int64_t ntiles, float* __restrict__ rhomin) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  float m = INFINITY;
  for (int a = 0; a < na; ++a) m = fminf(m, rhomax[a * ntiles + t]);
  rhomin[t] = m;
}

__global__ void k_tile_vsum(const float* __restrict__ V32, int pitch, int64_t n, int d, int np,
                            float* __restrict__ vsum, float* __restrict__ vsn) {
  __shared__ double nrm[32];
  const int64_t t = blockIdx.x;
  double q = 0.0;
  for (int k = threadIdx.x; k < pitch; k += blockDim.x) {
    double acc = 0.0;
    if (k < d)
      for (int j = 0; j < np; ++j) {
        const int64_t v = t * np + j;
        if (v < n) acc += (double)V32[v * pitch + k];
      }
    const float f = (float)acc;
    vsum[t * pitch + k] = f;
    q += (double)f * (double)f;
  }
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  if ((threadIdx.x & 31) == 0) nrm[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += nrm[w];
    vsn[t] = (float)(sqrt(tot) * (1.0 + 1e-6)) + 1e-30f;
  }
}

// ipsum[a][t] = sum over the tile's real points of the fp32 seeds ip_a(v) (fp64,
// fixed order).  One warp per (anchor, tile).
// Only tiles that can be all-positive for SOME block are summed: tile_allpos is
// monotone in (rhomax, rad), so (min over anchors of rhomax[a][t], min block
// radius) failing it rules the tile out for every block (its ipsum is never
// read); *anyflag records whether any tile passed (k_screen_agg exits early
// otherwise -- the late steps of a run).
__global__ void k_tile_ipsum(const float* __restrict__ ipa, int64_t stride, int na, int64_t n, int64_t ntiles,
                             int np, double* __restrict__ ipsum, const float* __restrict__ rhomin, float radmin,
                             const float* __restrict__ cmn, int* __restrict__ anyflag,
                             const int* __restrict__ level_now = nullptr) {
  if (level_now && *level_now < 0) return;  // lazy step decided without a screen
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)na * ntiles) return;
  const int a = (int)(w / ntiles);
  const int64_t t = w - (int64_t)a * ntiles;
  if (!tile_allpos(rhomin[t], radmin, cmn[t])) return;
  if (a == 0 && lane == 0) atomicOr(anyflag, 1);
  double s = 0.0;
  for (int j = lane; j < np; j += 32) {
    const int64_t v = t * np + j;
    if (v < n) s += (double)ipa[a * stride + v];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if (lane == 0) ipsum[w] = s;
}

// tile_prunable (kernels.cuh): the certified tile-pair test shared with k_refine.

// Anchor data of the tensor screen (kernel argument).
struct TcAnchors {
  const float* mu;          // na x apitch
  int apitch;
  const int* tile_anchor;   // per 128-row block of candidates
  const float* ipa;         // na x ipstride seeds
  int64_t ipstride;
  const float* kpmax;       // na x kpstride
  int64_t kpstride;
  const float* vmax;        // per point tile
  float kc;                 // kc = kc_coef (|mu| |c'| + |c'|^2)
  float kx;                 // per pair MMA term kx |v|max |c'|
  // tile-pair pruning (nullptr: off): rho[a][t] = min_v |v - mu_a|, rad[block]
  // = max_c |c - mu_a|, cmx[t] = max cm over the tile (current step)
  const float* rho;
  const float* rad;
  const float* cmx;
  int list_cap;             // uint16 entries reserved for the kept-tile list
  int kq_cap;               // float2 {kpmax, vmax} entries staged in smem per CTA (0: read per tile)
  unsigned long long* work; // if set: += executed (candidate block, point tile) pairs
  // all-positive tiles handled by k_screen_agg (nullptr: off): rhomax[a][t] =
  // max_v |v - mu_a|, cmn[t] = min cm over the tile (current step)
  const float* rhomax = nullptr;
  const float* cmn = nullptr;
  // KIND_F16R: operands are fp16(oscale * x), the accumulator holds oscale^2 v.c';
  // keta = sqrt(d) x (fp16 subnormal half-spacing 2^-25) / oscale x 1.02, the
  // absolute underflow term of the operand rounding (per |c'| and per |v|max)
  float oscale = 1.f;
  float sinv2 = 1.f;
  float keta = 0.f;
  float keta2 = 0.f;  // d eta^2
  // MS: the per-tile seed/final-add quantum kpmax is scaled by kpscale to cover
  // the in-MMA fp32 accumulation of the seed parts ((kpad + 24) 2^-23 |ip|)
  float kpscale = 1.f;
  // lazy step (kernels.cuh k_lazy_mark): screen only the 128-candidate blocks
  // flagged here (nullptr: every block); indexed by (crow - cand0) >> 7
  const unsigned char* bflag = nullptr;
  const int* ncand_dev = nullptr;  // gathered candidates (Vc rows): CTAs of blocks past the count exit
};

// One CTA: candidates [cand0 + 128*bx, +128) x V tiles [t0, t1) of NP points.
// A (candidates, hi and lo) lives in TMEM for the CTA's life (MMA "TS" form:
// the tensor core reads only the B tiles from shared memory); B tiles stream
// through a STAGES-deep bulk-copy ring released by the MMA commit alone; the
// per-point seed/quantum {ip, kp} is read by the epilogue through L1.
// FLAG: work-matrix flag screen (multiset.cuh) -- candidates are the gathered
// member rows Vc, seeds are the reset state (cm = d(., e0)), and every pair that
// is possibly closer than e0 (a > -kq) is appended to fo instead of summed.
// MS: seeds folded into the MMA (one-product FP16 kinds; TcSeeds): K columns
// d..d+2 of the point operand hold the scaled origin seed in three FP16 parts,
// the candidate operand holds 1 there, so the accumulator is s^2 (ip_0 + v.c)
// and the epilogue neither loads nor adds seeds.  Origin anchor only.
// MB = 2 (one-product kinds with folded seeds only, NP = 64): the CTA screens
// TWO candidate blocks against each 64-point tile -- A of block h in TMEM
// columns [64h, 64h + 56), its three accumulators at 128 + (3h + b) 64 -- so every
// point tile fetched from L2 serves 256 candidates (half the L2 -> SM traffic
// per pair); epilogue warpgroup h owns block h.  Per-tile host arrays are at
// 128-point granularity (index >> 1).
template <int NP, int KIND, bool FLAG = false, bool MS = false, int MB = 1>
__global__ void __launch_bounds__(tc::THREADS, 1)
    k_screen_tc(const float* __restrict__ V32, int pitch, int d, const unsigned char* __restrict__ Vhi,
                const unsigned char* __restrict__ Vlo, TcAnchors an,
                int kpad, int stages, int64_t cand0, int ntiles, int tiles_per_split, double* __restrict__ part_g,
                float* __restrict__ part_e, int64_t part_stride, const int* __restrict__ level_now,
                int level, const float* __restrict__ Vc = nullptr, FlagOut fo = FlagOut{}) {
  using namespace tc;
  if (level_now && *level_now != level) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  using TM = TmemMap<KIND>;
  constexpr bool BF = TM::W16;  // 16-bit operands (BF16 split or FP16)
  constexpr int ES = TM::ES;    // operand element bytes
  const uint32_t b_bytes = (uint32_t)NP * kpad * ES;
  const uint32_t stage_bytes = TM::PARTS * b_bytes;
  unsigned char* stage0 = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* full = bars;                   // [stages] operands landed
  uint64_t* sempty = bars + MAX_STAGES;    // [stages] operands consumed (MMA commit)
  uint64_t* tfull = bars + 2 * MAX_STAGES;       // [3] accumulator ready
  uint64_t* tempty = bars + 2 * MAX_STAGES + 3;  // [3] accumulator drained (all epilogue threads)
  uint64_t* aready = bars + 2 * MAX_STAGES + 6;  // A written to TMEM (all epilogue threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * MAX_STAGES + 7);

  const int t0 = blockIdx.y * tiles_per_split;
  const int t1 = min(ntiles, t0 + tiles_per_split);
  const int nt = t1 - t0;
  static_assert(MB == 1 || (MB == 2 && NP == 64 && MS && !FLAG && EPI_WARPGROUPS == 2), "two-block CTA shape");
  constexpr int TSH = MB == 2 ? 1 : 0;  // per-tile host arrays: 128-point tiles
  const int64_t crow = cand0 + (int64_t)blockIdx.x * M * MB;
  if (an.bflag) {  // CTA-uniform: exits before any barrier or TMEM allocation
    const int64_t b0 = (int64_t)blockIdx.x * MB;
    if (!an.bflag[b0] && (MB == 1 || !an.bflag[b0 + 1])) return;
  }
  if (an.ncand_dev && crow >= (int64_t)*an.ncand_dev) return;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sempty[s], 1);
    }
    for (int b = 0; b < 3; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128 * EPI_WARPGROUPS);
    }
    mbar_init(aready, 128 * EPI_WARPGROUPS);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  // kept point tiles of this CTA (certified tile-pair pruning, tile_prunable):
  // every role walks the same compacted list, built once by all threads
  // per-tile error-quantum inputs {kpmax[anchor][t], vmax[t]} of the CTA's tile
  // range, staged once so the epilogue's per-tile quantum is a shared-memory read
  float2* kqs = reinterpret_cast<float2*>(smem + (size_t)stages * stage_bytes + (2 * MAX_STAGES + 8) * sizeof(uint64_t) + 64);
  const bool kq_staged = nt <= an.kq_cap;
  if (kq_staged) {
    const int a0 = MS ? 0 : an.tile_anchor[crow >> 7];
    const float* kpg = an.kpmax + (int64_t)a0 * an.kpstride;
    for (int i = tid; i < nt; i += THREADS) kqs[i] = make_float2(kpg[(t0 + i) >> TSH], an.vmax[(t0 + i) >> TSH]);
    __syncthreads();  // kq_staged is uniform over the CTA
  }
  uint16_t* tlist = nullptr;
  int ntk = nt;
  if (an.rho && nt <= an.list_cap) {
    __shared__ int wsum[THREADS / 32];
    tlist = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(kqs) + (size_t)an.kq_cap * sizeof(float2));
    const float rad = an.rad[crow >> 7];
    const float* rho = an.rho + (int64_t)an.tile_anchor[crow >> 7] * an.kpstride;
    int base = 0;
    for (int c0i = 0; c0i < nt; c0i += THREADS) {
      const int i = c0i + tid;
      bool keep = i < nt && !tile_prunable(rho[t0 + i], rad, an.cmx[t0 + i]);
      if (keep && an.rhomax)  // summed from aggregates by k_screen_agg instead
        keep = !tile_allpos(an.rhomax[(int64_t)an.tile_anchor[crow >> 7] * an.kpstride + t0 + i], rad, an.cmn[t0 + i]);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) wsum[warp] = __popc(bal);
      __syncthreads();
      int off = base, tot = 0;
#pragma unroll 1
      for (int w = 0; w < THREADS / 32; ++w) {
        off += w < warp ? wsum[w] : 0;
        tot += wsum[w];
      }
      if (keep) tlist[off + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)i;
      base += tot;
      __syncthreads();
    }
    ntk = base;
  }
  auto TL = [&](int k) -> int { return tlist ? (int)tlist[k] : k; };
  if (an.work && tid == 0) atomicAdd(an.work, (unsigned long long)ntk);

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      for (int it = 0; it < ntk; ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(&sempty[s], ((it / stages) - 1) & 1);
        unsigned char* st = stage0 + s * stage_bytes;
        const int64_t prow = (int64_t)(t0 + TL(it)) * NP;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        bulk_g2s(st, Vhi + prow * kpad * ES, b_bytes, &full[s]);
        if (TM::PARTS == 2) bulk_g2s(st + b_bytes, Vlo + prow * kpad * ES, b_bytes, &full[s]);
      }
    }
  } else if (warp < EPI_WARP0) {
    // ---------------- MMA issuers: warp 1 + b issues the tiles that use
    // accumulator buffer b, so one warp's barrier waits and register set-up
    // overlap the other's queued MMAs.  The whole warp walks the loop
    // (warp-uniform operands stay in uniform registers), one elected lane issues.
    constexpr uint32_t idesc =
        one_product(KIND) ? idesc_f16(M, NP) : (KIND == KIND_BF16 ? idesc_bf16(M, NP) : idesc_tf32(M, NP));
    const uint32_t sbo = (uint32_t)kpad * 8 * ES;  // 8 rows x kpad elements
    const int ksteps = kpad / (BF ? 16 : 8);       // 32 bytes of K per instruction
    constexpr int NB = TM::NB;
    const int b = warp - 1;
    const uint32_t dt = tmem + TM::ACC + (uint32_t)(b * NP);
    const uint32_t dt2 = tmem + TM::ACC + (uint32_t)((NB + b) * NP);  // MB = 2: block 1's buffer b
    const uint32_t ahi = tmem + COL_AHI, alo = tmem + TM::ALO;
    mbar_wait(aready, 0);
    fence_after();
    for (int it = b; it < ntk && b < NB; it += NB) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      if (it >= NB) mbar_wait(&tempty[b], ((it / NB) - 1) & 1);
      fence_after();
      const uint32_t bhi = smem_u32(stage0 + s * stage_bytes);
      // descriptors built once per tile; K step j advances the start-address
      // field by 256 B (= 16 in 16-byte units) and A by 8 TMEM columns
      const uint64_t dhi = sdesc(bhi, 128, sbo);
      const uint64_t dlo = sdesc(bhi + b_bytes, 128, sbo);
      if (elect_one()) {
#pragma unroll 4
        for (int j = 0; j < ksteps; ++j) {
          if (one_product(KIND)) {
            mma1_f16_ts(dt, ahi + 8 * j, dhi + 16 * j, idesc, j > 0);
            if (MB == 2) mma1_f16_ts(dt2, ahi + 64 + 8 * j, dhi + 16 * j, idesc, j > 0);
          }
          else if (KIND == KIND_BF16)
            mma3_bf16_ts(dt, ahi + 8 * j, alo + 8 * j, dhi + 16 * j, dlo + 16 * j, idesc, j > 0);
          else
            mma3_tf32_ts(dt, ahi + 8 * j, alo + 8 * j, dhi + 16 * j, dlo + 16 * j, idesc, j > 0);
        }
        commit(&sempty[s]);  // operands consumed -> producer may refill
        commit(&tfull[b]);   // accumulator ready for the epilogue
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: EPI_WARPGROUPS x 4 warps; thread = candidate
    // (TMEM lane) x one slice of the tile's point columns
    const int q = warp & 3;                    // TMEM lane quadrant of this warp
    const int half = (warp - EPI_WARP0) >> 2;  // which slice of the NP columns
    constexpr int SLICE = MB == 2 ? NP : NP / EPI_WARPGROUPS;
    const int cl = q * 32 + lane;
    const int64_t c = crow + (MB == 2 ? (int64_t)half * M : 0) + cl;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int anc = MS ? 0 : an.tile_anchor[crow >> 7];  // anchor of this candidate block
    const float* mu = an.mu + (int64_t)anc * an.apitch;
    float cn2 = 0.f, mc = 0.f, mn2 = 0.f;
    {
      // A of this candidate into TMEM: slice 0 writes hi [0,128), the last slice lo [128,256)
      const float* row = (Vc ? Vc : V32) + c * pitch;  // Vc: gathered candidate rows
      const bool do_hi = MB == 2 || half == 0, do_lo = TM::PARTS == 2 && half == EPI_WARPGROUPS - 1;
      auto cprime = [&](int k) -> float {  // c' = fl(c - mu), accumulating |c'|^2, mu.c', |mu|^2
        if (k >= d) return 0.f;
        const float m = mu[k];
        const float x = row[k] - m;
        cn2 = fmaf(x, x, cn2);
        mc = fmaf(m, x, mc);
        mn2 = fmaf(m, m, mn2);
        return x;
      };
#pragma unroll 1
      for (int blk = 0; blk < (BF ? 2 : 4); ++blk) {
        uint32_t rh[32], rl[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (one_product(KIND)) {
            // KIND_F16: origin anchor only (c' = c, exactly fp16, oscale 1);
            // KIND_F16R: fp16(oscale c'), the rounding is in the bound
            const int k = blk * 64 + 2 * i;
            const float x0 = cprime(k), x1 = cprime(k + 1);
            // MS: 1 in the seed columns d..d+2
            const float y0 = (MS && k >= d && k < d + 3) ? 1.f : x0 * an.oscale;
            const float y1 = (MS && k + 1 >= d && k + 1 < d + 3) ? 1.f : x1 * an.oscale;
            rh[i] = (uint32_t)__half_as_ushort(__float2half_rn(y0)) |
                    ((uint32_t)__half_as_ushort(__float2half_rn(y1)) << 16);
            rl[i] = 0u;
          } else if (BF) {
            // column = packed pair (k = 2i, 2i+1), low half = even k
            const int k = blk * 64 + 2 * i;
            const float x0 = cprime(k), x1 = cprime(k + 1);
            const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
            const __nv_bfloat16 m0 = __float2bfloat16_rn(x0 - __bfloat162float(h0));
            const __nv_bfloat16 m1 = __float2bfloat16_rn(x1 - __bfloat162float(h1));
            rh[i] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
            rl[i] = (uint32_t)__bfloat16_as_ushort(m0) | ((uint32_t)__bfloat16_as_ushort(m1) << 16);
          } else {
            const int k = blk * 32 + i;
            const float x = cprime(k);
            const uint32_t h = __float_as_uint(x) & 0xFFFFE000u;
            rh[i] = h;
            rl[i] = __float_as_uint(x - __uint_as_float(h));
          }
        }
        if (do_hi) st32(tmem + lane_off + COL_AHI + (MB == 2 ? half * 64 : 0) + blk * 32, rh);
        if (do_lo) st32(tmem + lane_off + TM::ALO + blk * 32, rl);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_before();
      mbar_arrive(aready);
    }
    // t/2 = ip_a(v) + v.c' + ic, ic = -(mu.c' + |c'|^2/2); per-pair error bound
    // kpmax[a][tile] + kc + kx |v|max(tile) |c'|  (DESIGN.md §4 "anchored tensor screen")
    const float cn = sqrtf(cn2) * (1.f + 1e-5f);
    const float ic = -(mc + 0.5f * cn2);
    const float kc = fmaf(an.keta, cn, an.kc * (sqrtf(mn2) * (1.f + 1e-5f) * cn + cn2)) + an.keta2;
    const float kxc = fmaf(an.kx, cn, an.keta);
    const float* ipa = an.ipa + (int64_t)anc * an.ipstride;
    const float* kpa = an.kpmax + (int64_t)anc * an.kpstride;
    double g64 = 0.0;
    float e = 0.f;
    constexpr int NB = TM::NB;
    constexpr int SW = SLICE;  // accumulator columns per thread and tile
    // this slice's point seeds ip, software-pipelined one tile ahead: tile it+1's
    // loads are issued as soon as tile it's seed add has consumed the registers,
    // so their L2 latency hides behind the rest of tile it's epilogue
    float ipv[MS ? 1 : SW];
    auto load_seeds = [&](int itn) {
      if constexpr (!MS) {
        const float4* pp4 = reinterpret_cast<const float4*>(ipa + (int64_t)(t0 + TL(itn)) * NP + half * SLICE);
#pragma unroll
        for (int i = 0; i < SW / 4; ++i) {
          const float4 p = __ldg(pp4 + i);
          ipv[4 * i] = p.x;
          ipv[4 * i + 1] = p.y;
          ipv[4 * i + 2] = p.z;
          ipv[4 * i + 3] = p.w;
        }
      }
    };
    if (ntk > 0) load_seeds(0);
    // speculative slow path (split / FP16 kinds without folded seeds): after a
    // tile with a positive term the next tile skips the early-out max tree and
    // goes straight to the sum -- identical result (an all-zero tile adds +0.0),
    // 0.5 fewer issue slots per pair on clustered data (C4: 99.8% of the
    // warp-tiles take the slow path)
    constexpr bool SPEC = EBC200_SPEC && !FLAG && !MS;
    bool spec = false;
    for (int it = 0; it < ntk; ++it) {
      const int b = it % NB;
      const int tt = t0 + TL(it);  // point tile
      // one error quantum per tile: kpmax = max_v kp over the tile (bounds every
      // pair's kp_v; computed at reset, cm only decreases within a run)
      float kpt, vmt;
      if (kq_staged) {
        const float2 q2 = kqs[tt - t0];
        kpt = q2.x;
        vmt = q2.y;
      } else {
        kpt = kpa[tt >> TSH];
        vmt = __ldg(an.vmax + (tt >> TSH));
      }
      mbar_wait(&tfull[b], (it / NB) & 1);
      fence_after();
      float S[SW];
      ldcols<SW>(tmem + lane_off + TM::ACC +
                 (uint32_t)(MB == 2 ? (half * NB + b) * NP : b * NP + half * SLICE), S);
      fence_before();
      mbar_arrive(&tempty[b]);  // this thread's columns of the buffer are in registers
      // the quantum is formed only now: its inputs share a load scoreboard with
      // the seed loads, and an FFMA scheduled before the tcgen05.ld held the
      // load's issue behind them (ncu, C4: 13% of stall samples).  vmt + 0*S[0]
      // (exactly vmt: S is finite) makes the FFMA depend on the TMEM load.
      const float vmt_after = __fadd_rn(vmt, __fmul_rn(S[0], 0.f));
      const float kq = fmaf(kpt, an.kpscale, fmaf(kxc, vmt_after, kc));
      // FLAG: possibly closer than e0 iff a > -kq - 2^-100 (absolute floor for
      // pairs whose products underflow: points within ~1e-15 of e0)
      const float thr = -kq - 0x1p-100f;
      const float icq = ic + kq;       // bound: a + kq = b + icq
      // b = S + ip per pair, a = b + ic.  fl(b + ic) is monotone in b, so
      // max_i a_i = fl(max_i b_i + ic): when that is <= thr (< 0) every pair
      // adds exactly 0 to the gain and to the count, and the tile is skipped --
      // the common case (few points are closer to a candidate than to the summary).
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if constexpr (MS) {
        // the accumulator already holds s^2 b: the max tree runs on it raw and
        // max_i fl(S_i s^-2 + icq) = fl(max_i S_i s^-2 + icq) (exact power of two)
      } else {
#if EBC200_EPI_FADD2
      if (KIND == KIND_F16R) {
        // S sinv2 is exact (power of two): fl(S sinv2 + ip) in one packed FFMA2
        const float2 sv2 = make_float2(an.sinv2, an.sinv2);
#pragma unroll
        for (int i = 0; i < SW; i += 2) {
          const float2 r = __ffma2_rn(make_float2(S[i], S[i + 1]), sv2, make_float2(ipv[i], ipv[i + 1]));
          S[i] = r.x;
          S[i + 1] = r.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < SW; i += 2) {  // packed FADD2: half the issue slots
          const float2 r = __fadd2_rn(make_float2(S[i], S[i + 1]), make_float2(ipv[i], ipv[i + 1]));
          S[i] = r.x;
          S[i + 1] = r.y;
        }
      }
#else
      if (KIND == KIND_F16R)
#pragma unroll
        for (int i = 0; i < SW; ++i) S[i] *= an.sinv2;
#pragma unroll
      for (int i = 0; i < SW; ++i) S[i] += ipv[i];
#endif
      if (it + 1 < ntk) load_seeds(it + 1);  // ipv is free again
      }
      if (!(SPEC && spec)) {
#pragma unroll
        for (int i = 0; i < SW; i += 8) {
          m4[(i / 8) & 3] = fmaxf(m4[(i / 8) & 3], fmaxf(fmaxf(S[i], S[i + 1]), S[i + 2]));
          m4[(i / 8) & 3] = fmaxf(m4[(i / 8) & 3], fmaxf(fmaxf(S[i + 3], S[i + 4]), S[i + 5]));
          m4[(i / 8) & 3] = fmaxf(m4[(i / 8) & 3], fmaxf(S[i + 6], S[i + 7]));
        }
      }
      const float mb = (SPEC && spec) ? INFINITY
                       : (MS ? fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * an.sinv2
                             : fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
      if (FLAG) {
        // rare: pairs possibly closer than e0.  Warp-aggregated append: one
        // atomicAdd per warp and tile, each lane writes at its prefix offset.
        if (__any_sync(0xffffffffu, mb + ic > thr)) {
          uint64_t msk = 0;
          const int64_t vb = (int64_t)tt * NP + half * SLICE;
          if (c < fo.ncands) {
#pragma unroll
            for (int i = 0; i < SW; ++i)
              if (S[i] + ic > thr && vb + i < fo.npoints) msk |= 1ull << i;
          }
          const int cnt = __popcll(msk);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          int base = 0;
          if (lane == 31 && incl > 0) base = atomicAdd(fo.count, incl);
          base = __shfl_sync(0xffffffffu, base, 31);
          int slot = base + incl - cnt;
          while (msk) {
            const int i = __ffsll((long long)msk) - 1;
            msk &= msk - 1;
            if (slot < fo.cap) fo.pairs[slot] = make_uint2((unsigned)(vb + i), (unsigned)c);
            ++slot;
          }
        }
      } else if (mb + icq > 0.f) {
        // upper bound only: gain/2 <= sum max(a + kq, 0) with a + kq = fl(b + icq);
        // fl(. + icq) is monotone, so a slice whose max gives <= 0 adds exactly 0.
        // Four independent fp32 partial sums per 32 columns (ILP); each partial
        // adds 8 terms, every fp64 fold covers <= 32 (the finalize bound).
        constexpr int GW = SW < 32 ? SW : 32;
        float tile_pos = 0.f;  // any positive term in this tile (SPEC)
#pragma unroll
        for (int h = 0; h < SW; h += GW) {
#if EBC200_EPI_FADD2
          float2 g2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          const float2 icq2 = make_float2(icq, icq);
#pragma unroll
          const float2 sv2 = make_float2(an.sinv2, an.sinv2);
          for (int i = h; i < h + GW; i += 2) {
            const float2 a = MS ? __ffma2_rn(make_float2(S[i], S[i + 1]), sv2, icq2)
                                : __fadd2_rn(make_float2(S[i], S[i + 1]), icq2);
            g2[(i >> 1) & 1] = __fadd2_rn(g2[(i >> 1) & 1], make_float2(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f)));
          }
          const float gt = (g2[0].x + g2[0].y) + (g2[1].x + g2[1].y);
          g64 += (double)gt;
          tile_pos += gt;
#else
          float g4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = h; i < h + GW; ++i) g4[i & 3] += fmaxf((MS ? S[i] * an.sinv2 : S[i]) + icq, 0.f);
          g64 += (double)((g4[0] + g4[1]) + (g4[2] + g4[3]));
          tile_pos += (g4[0] + g4[1]) + (g4[2] + g4[3]);
#endif
        }
        if (SPEC) spec = tile_pos > 0.f;
      } else if (SPEC) {
        spec = false;
      }
    }
    if (!FLAG && MB == 2) {  // each warpgroup owns its block's candidates outright
      part_g[blockIdx.y * part_stride + c] = g64;
      part_e[blockIdx.y * part_stride + c] = e;
    } else if (!FLAG) {
    // combine the slices of each candidate in slice order (named barrier over
    // the epilogue warps only)
    double* xg = reinterpret_cast<double*>(stage0);  // the ring is idle once every tile is consumed
    float* xe = reinterpret_cast<float*>(stage0 + (size_t)EPI_WARPGROUPS * M * sizeof(double));
    asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPGROUPS * 128));
    xg[half * M + cl] = g64;
    xe[half * M + cl] = e;
    asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPGROUPS * 128));
    if (half == 0) {
      double gs = 0.0;
      float es = 0.f;
#pragma unroll
      for (int w = 0; w < EPI_WARPGROUPS; ++w) {
        gs += xg[w * M + cl];
        es += xe[w * M + cl];
      }
      part_g[blockIdx.y * part_stride + c] = gs;
      part_e[blockIdx.y * part_stride + c] = es;
    }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}


// All-positive (block, tile) pairs of the tensor screen (tile_allpos): the
// block's upper-bound contribution from tile aggregates.  Same plan and grid as
// k_screen_tc, one thread per candidate; only where the screen used its kept-tile
// list (it then skipped exactly these tiles).  Per tile:
//   sum_v (a_v + kq) <= ipsum_a[t] + c'.vsum[t] + n_t (ic + kq_t) + (d + 2) u |c'| |vsum[t]|
// with the screen's own per-pair quantum kq_t (it bounds the fp32 seed, c' and
// ic roundings); the last term covers vsum's fp32 rounding and an
// fp32 dot.  The terms are linear in the tile, so the CTA first sums the
// block's all-positive tiles (fixed order, fp64): W = sum vsum[t], sum ipsum,
// sum n_t, sum n_t kpmax[t], sum n_t vmax[t], sum |vsum[t]| -- then each
// candidate needs ONE fp64 dot c'.W instead of one fp32 dot per tile (C4 step 0:
// every pair all-positive, 9.8 ms -> see DESIGN.md).  The fp64 sums and dot
// err by < (nl + d + 2) 2^-53 |c'| sum |vsum[t]|, far inside the kept (d + 2) u
// term; kq_t = fl32(kpmax + fl32(kxc vmax + kc)) (non-negative terms) is
// bounded by its exact value times (1 + 2^-21).
__global__ void __launch_bounds__(128) k_screen_agg(const float* __restrict__ V32, int pitch, int d, TcAnchors an,
                                                    int64_t cand0, int ntiles, int tiles_per_split, int np, int64_t n,
                                                    const double* __restrict__ ipsum, const float* __restrict__ vsum,
                                                    const float* __restrict__ vsn, double* __restrict__ part_a,
                                                    int64_t part_stride, const int* __restrict__ level_now,
                                                    int level, const int* __restrict__ anyflag) {
  if (level_now && *level_now != level) return;
  if (an.bflag && !an.bflag[blockIdx.x]) return;  // lazy step: block not re-screened
  if (*anyflag == 0) {  // no tile can be all-positive this step
    part_a[blockIdx.y * part_stride + cand0 + (int64_t)blockIdx.x * 128 + threadIdx.x] = 0.0;
    return;
  }
  extern __shared__ __align__(16) double agg_sm[];  // W[d], Wp[128], then the tile list
  double* W = agg_sm;
  double* Wp = agg_sm + d;
  uint16_t* tl = reinterpret_cast<uint16_t*>(agg_sm + d + 128);
  __shared__ int wsum[4];
  __shared__ double red[5][4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.y * tiles_per_split;
  const int t1 = min(ntiles, t0 + tiles_per_split);
  const int nt = t1 - t0;
  const int64_t crow = cand0 + (int64_t)blockIdx.x * 128;
  const int64_t c = crow + tid;
  double acc = 0.0;
  if (an.rho && an.rhomax && nt <= an.list_cap) {
    const int anc = an.tile_anchor[crow >> 7];
    const float rad = an.rad[crow >> 7];
    const float* rho = an.rho + (int64_t)anc * an.kpstride;
    const float* rhx = an.rhomax + (int64_t)anc * an.kpstride;
    // the block's all-positive tiles, classified once (same tests as the screen)
    int nl = 0;
    for (int i0 = 0; i0 < nt; i0 += 128) {
      const int i = i0 + tid;
      const bool on = i < nt && !tile_prunable(rho[t0 + i], rad, an.cmx[t0 + i]) &&
                      tile_allpos(rhx[t0 + i], rad, an.cmn[t0 + i]);
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (lane == 0) wsum[warp] = __popc(bal);
      __syncthreads();
      int off = nl;
      for (int w = 0; w < warp; ++w) off += wsum[w];
      if (on) tl[off + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)i;
      nl += wsum[0] + wsum[1] + wsum[2] + wsum[3];
      __syncthreads();
    }
    if (nl > 0) {
      const float* kpa = an.kpmax + (int64_t)anc * an.kpstride;
      const double* ips = ipsum + (int64_t)anc * an.kpstride;
      // the block's scalar sums: per-thread strided partials, butterfly, warps in order
      double sv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (int li = tid; li < nl; li += 128) {
        const int t = t0 + tl[li];
        const double nt_pts = (double)min((int64_t)np, n - (int64_t)t * np);
        sv[0] += ips[t];
        sv[1] += nt_pts;
        sv[2] += nt_pts * (double)kpa[t];
        sv[3] += nt_pts * (double)__ldg(an.vmax + t);
        sv[4] += (double)vsn[t];
      }
#pragma unroll
      for (int j = 0; j < 5; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sv[j] += __shfl_xor_sync(0xffffffffu, sv[j], o);
        if (lane == 0) red[j][warp] = sv[j];
      }
      // W = sum of the tiles' vsum rows: groups of d threads take every T-th tile
      if (d <= 128) {
        const int T = 128 / d, g = tid / d, k = tid - g * d;
        if (g < T) {
          double p = 0.0;
          for (int li = g; li < nl; li += T) p += (double)__ldg(vsum + (int64_t)(t0 + tl[li]) * pitch + k);
          Wp[g * d + k] = p;
        }
        __syncthreads();
        if (tid < d) {
          double w = 0.0;
          for (int q = 0; q < T; ++q) w += Wp[q * d + tid];
          W[tid] = w;
        }
      } else {
        for (int k = tid; k < d; k += 128) {
          double p = 0.0;
          for (int li = 0; li < nl; ++li) p += (double)__ldg(vsum + (int64_t)(t0 + tl[li]) * pitch + k);
          W[k] = p;
        }
      }
      __syncthreads();
      double S[5];
#pragma unroll
      for (int j = 0; j < 5; ++j) S[j] = ((red[j][0] + red[j][1]) + red[j][2]) + red[j][3];
      const float* mu = an.mu + (int64_t)anc * an.apitch;
      const float* row = V32 + c * pitch;
      float cn2 = 0.f, mc = 0.f, mn2 = 0.f;
      double dot = 0.0;
      for (int k = 0; k < d; ++k) {  // the screen's c' = fl(c - mu) and its sums, same order
        const float m = mu[k];
        const float x = row[k] - m;
        cn2 = fmaf(x, x, cn2);
        mc = fmaf(m, x, mc);
        mn2 = fmaf(m, m, mn2);
        dot = fma((double)x, W[k], dot);
      }
      const float cn = sqrtf(cn2) * (1.f + 1e-5f);
      const float ic = -(mc + 0.5f * cn2);
      const float kc = an.kc * (sqrtf(mn2) * (1.f + 1e-5f) * cn + cn2);
      const float kxc = an.kx * cn;
      const double edot = (double)(d + 2) * 5.960464477539063e-08 * 1.01 * (double)cn;
      const double kqs = (S[2] + (double)kxc * S[3] + (double)kc * S[1]) * (1.0 + 0x1p-21);
      acc = S[0] + dot + (double)ic * S[1] + kqs + edot * S[4];
    }
  }
  part_a[blockIdx.y * part_stride + c] = acc;
}

}  // namespace ebc
