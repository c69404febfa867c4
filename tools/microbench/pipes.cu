// Pipe-throughput microbenchmark for the EBC distance inner loop on sm_100a.
// Measures issue-limited throughput of the instruction mixes the screening
// kernels are built from (FADD2+FFMA2 direct form, scalar FFMA, half2, fp64),
// so the kernel design is chosen from measured numbers, not guesses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CHAINS 16
#define ITERS 4096

// diff = v + (-c); acc += diff*diff  — the direct-form pair loop, packed along d.
__global__ void k_f32x2(const float* in, float* out) {
  float2 v = make_float2(in[threadIdx.x], in[threadIdx.x + 1]);
  float2 acc[CHAINS], nc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { acc[i] = make_float2(0.f, 0.f); nc[i] = make_float2(-in[i], -in[i + 3]); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      float2 d = __fadd2_rn(v, nc[i]);
      acc[i] = __ffma2_rn(d, d, acc[i]);
    }
    v.x += 1e-7f;  // keep loop-carried dependence so nothing is hoisted
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Same math, scalar FADD + FFMA.
__global__ void k_f32(const float* in, float* out) {
  float v = in[threadIdx.x], v2 = in[threadIdx.x + 1];
  float acc[2 * CHAINS], nc[2 * CHAINS];
#pragma unroll
  for (int i = 0; i < 2 * CHAINS; ++i) { acc[i] = 0.f; nc[i] = -in[i]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 2 * CHAINS; ++i) {
      float d = ((i & 1) ? v2 : v) + nc[i];
      acc[i] = fmaf(d, d, acc[i]);
    }
    v += 1e-7f;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 2 * CHAINS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half2: HADD2 + HFMA2.
__global__ void k_h2(const float* in, float* out) {
  __half2 v = __floats2half2_rn(in[threadIdx.x], in[threadIdx.x + 1]);
  __half2 acc[CHAINS], nc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { acc[i] = __float2half2_rn(0.f); nc[i] = __floats2half2_rn(-in[i], -in[i + 3]); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      __half2 d = __hadd2(v, nc[i]);
      acc[i] = __hfma2(d, d, acc[i]);
    }
    v = __hadd2(v, __float2half2_rn(1e-3f));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += __low2float(acc[i]) + __high2float(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// fp64: DADD + DFMA.
__global__ void k_f64(const float* in, float* out) {
  double v = in[threadIdx.x];
  double acc[CHAINS], nc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { acc[i] = 0.0; nc[i] = -(double)in[i]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      double d = v + nc[i];
      acc[i] = fma(d, d, acc[i]);
    }
    v += 1e-9;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

// f32x2 pair loop plus the screening epilogue on every 2nd chain (FADD, FMNMX,
// FSETP/FSEL, FADD2) to see whether ALU-side work hides under the FMA pipe.
__global__ void k_f32x2_epi(const float* in, float* out) {
  float2 v = make_float2(in[threadIdx.x], in[threadIdx.x + 1]);
  float2 acc[CHAINS], nc[CHAINS];
  float cm = in[7], tau = in[8];
  float2 ge = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { acc[i] = make_float2(0.f, 0.f); nc[i] = make_float2(-in[i], -in[i + 3]); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      float2 d = __fadd2_rn(v, nc[i]);
      acc[i] = __ffma2_rn(d, d, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float t = cm - (acc[i].x + acc[i].y);
      float2 add = make_float2(fmaxf(t, 0.f), t > -tau ? tau : 0.f);
      ge = __fadd2_rn(ge, add);
    }
    v.x += 1e-7f;
  }
  float s = ge.x + ge.y;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d MHz\n", p.name, p.multiProcessorCount, clk_khz / 1000);
  float *in, *out;
  cudaMalloc(&in, 4096 * sizeof(float));
  cudaMemset(in, 0, 4096 * sizeof(float));
  const int threads = 256;
  for (int occ : {1, 2, 4}) {
    int blocks = p.multiProcessorCount * occ;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(float));
    struct { const char* name; void (*k)(const float*, float*); double ops_per_iter; } ks[] = {
        {"f32x2 fadd2+ffma2", k_f32x2, CHAINS * 4.0},
        {"f32 fadd+ffma", k_f32, 2 * CHAINS * 2.0},
        {"h2 hadd2+hfma2", k_h2, CHAINS * 4.0},
        {"f64 dadd+dfma", k_f64, CHAINS * 2.0},
        {"f32x2 + epilogue", k_f32x2_epi, CHAINS * 4.0},
    };
    for (auto& k : ks) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      k.k<<<blocks, threads>>>(in, out);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k.k<<<blocks, threads>>>(in, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      double ops = 5.0 * blocks * threads * (double)ITERS * k.ops_per_iter;
      double tops = ops / (ms * 1e-3) / 1e12;
      // ops per clock per SM at the nominal max clock
      double per_clk = ops / (ms * 1e-3) / (p.multiProcessorCount * 1965e6);
      printf("occ %d  %-20s %8.3f ms  %7.2f Tops/s  %6.1f ops/clk/SM(@1965)\n", occ, k.name, ms, tops, per_clk);
    }
    cudaFree(out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
