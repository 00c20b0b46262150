// FP64 peak microbenchmark (SURVEY 8d / BASELINE.md: "FP64 P64 measured by a DFMA
// microbenchmark"). The roofline denominator of the one compute-bound kernel class
// (the BiCGSTAB dense image, k_bi_image2: DFMA chains) and of the contract's
// mul-then-add kernels (no FMA contraction: one flop per instruction).
//
// Each thread runs 16 independent register chains; 148 SMs x 8 CTAs x 256 threads
// keep every FP64 pipe busy. Timed with CUDA events on the launching stream, best of
// `reps` after one warm-up launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "sylkrylov_b200.h"

namespace {

constexpr int kChains = 16;

template <bool FMA>
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) x[j] = (double)(threadIdx.x + j) * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
      if constexpr (FMA)
        x[j] = __fma_rn(x[j], a, b);
      else
        x[j] = __dadd_rn(__dmul_rn(x[j], a), b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += x[j];
  if (s == 123.456) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // never true: keeps the chains live
}

template <bool FMA>
double run(int sms, int iters, int reps, cudaStream_t st, double* sink) {
  const int ctas = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64_peak<FMA><<<ctas, 256, 0, st>>>(sink, iters, 0.999999, 1e-9);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, st);
    k_fp64_peak<FMA><<<ctas, 256, 0, st>>>(sink, iters, 0.999999, 1e-9);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = (double)ctas * 256.0 * kChains * (double)iters * 2.0;  // fma = mul + add = 2 flops
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace

extern "C" sk_status sk_measure_fp64_peak(int32_t device, double* dfma_tflops, double* dmul_dadd_tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return SK_ERR_CUDA;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SK_ERR_CUDA;
  double* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(double) * (size_t)prop.multiProcessorCount * 8 * 256) != cudaSuccess)
    return SK_ERR_OUT_OF_MEMORY;
  cudaStream_t st;
  cudaStreamCreate(&st);
  const double f = run<true>(prop.multiProcessorCount, 4096, 5, st, sink);
  const double m = run<false>(prop.multiProcessorCount, 4096, 5, st, sink);
  cudaStreamDestroy(st);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return SK_ERR_CUDA;
  if (dfma_tflops) *dfma_tflops = f;
  if (dmul_dadd_tflops) *dmul_dadd_tflops = m;
  return SK_OK;
}
