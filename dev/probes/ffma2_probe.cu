// Probe: FP32 throughput of scalar FFMA vs packed FFMA2 (sm_100a) per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
  return make_float2(a, b);
}

template <int MODE>  // 0: FFMA, 1: FFMA2, 2: FFMA + MUFU.EX2 mix (1:8)
__global__ void k(float* out, int iters, float s) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
  if (MODE == 1) {
    unsigned long long y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = pk(x[2 * j], x[2 * j + 1]);
    const unsigned long long m = pk(s, s), a = pk(1e-7f, 2e-7f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(m), "l"(a));
    }
    float acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { float2 t = upk(y[j]); acc += t.x + t.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], s, 1e-7f);
      if (MODE == 2) {
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x[0]));
        x[1] += e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x[2]));
        x[3] += e;
      }
    }
    float acc = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) acc += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  const int iters = 1 << 15;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<sms * 8, 256>>>(out, iters, 0.999f);
      if (mode == 1) k<1><<<sms * 8, 256>>>(out, iters, 0.999f);
      if (mode == 2) k<2><<<sms * 8, 256>>>(out, iters, 0.999f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double fma = (double)sms * 8 * 256 * iters * 16;
      if (rep) printf("mode %d: %.3f ms  %.1f TFMA/s  %.1f FMA/clk/SM (at %d MHz)\n", mode, ms, fma / ms / 1e9,
                      fma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
