// Probe: FP64 throughput on B200 (sm_100a): DFMA, DADD/DMUL, IEEE sqrt / div, exp().
// Sizing for the strict (fp64, reference operation order) mode.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: DFMA, 1: DADD+DMUL, 2: sqrt_rn + div_rn, 3: exp, 4: FFMA (fp32 ref)
__global__ void k(double* out, int iters, double s) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j + 1.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) x[j] = fma(x[j], s, 1e-7);
      if (MODE == 1) x[j] = __dadd_rn(__dmul_rn(x[j], s), 1e-7);
      if (MODE == 2) x[j] = __ddiv_rn(1.0, __dsqrt_rn(x[j])) + 1.0;
      if (MODE == 3) x[j] = exp(-x[j]) + 1.0;
    }
  }
  double acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"DFMA", "DMUL+DADD (ops)", "sqrt_rn+div_rn (pairs)", "exp"};
  for (int mode = 0; mode < 4; ++mode) {
    const int iters = mode >= 2 ? 1 << 10 : 1 << 13;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<sms * 8, 256>>>(out, iters, 0.999);
      if (mode == 1) k<1><<<sms * 8, 256>>>(out, iters, 0.999);
      if (mode == 2) k<2><<<sms * 8, 256>>>(out, iters, 0.999);
      if (mode == 3) k<3><<<sms * 8, 256>>>(out, iters, 0.999);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double ops = (double)sms * 8 * 256 * iters * 8 * (mode == 1 ? 2 : 1);
      if (rep)
        printf("%-24s %.3f ms  %.2f Gop/s  %.2f op/clk/SM (at %d MHz)\n", names[mode], ms,
               ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
