#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, long long* cyc, int iters, double a) {
  double x[CH];
  for (int j = 0; j < CH; ++j) x[j] = threadIdx.x * 1e-3 + j;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) x[j] = __dadd_rn(x[j], a);
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < CH; ++j) s += x[j];
  if (s == 1.2345) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
__global__ void km(double* out, long long* cyc, int iters, double a, double b) {
  double x[CH];
  for (int j = 0; j < CH; ++j) x[j] = threadIdx.x * 1e-3 + j;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) x[j] = __dadd_rn(__dmul_rn(x[j], a), b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < CH; ++j) s += x[j];
  if (s == 1.2345) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH> void run(int threads, const char* what, bool mul) {
  double* out; long long* cyc, h;
  cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8 * 16);
  const int iters = 4096;
  for (int r = 0; r < 2; ++r) {
    if (mul) km<CH><<<1, threads>>>(out, cyc, iters, 0.9999, 1e-9); else k<CH><<<1, threads>>>(out, cyc, iters, 1e-9);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)iters * CH * (mul ? 2 : 1);
  printf("%s threads %d chains %d: %.2f cycles per dependent op-step, %.2f warp-instr/clk/SM\n", what, threads, CH,
         (double)h / iters / (mul ? 2 : 1), ops * (threads / 32) / (double)h);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<1>(32, "DADD", false); run<2>(32, "DADD", false); run<4>(32, "DADD", false); run<8>(32, "DADD", false);
  run<1>(128, "DADD", false); run<2>(128, "DADD", false); run<4>(128, "DADD", false);
  run<1>(384, "DADD", false); run<2>(384, "DADD", false); run<4>(384, "DADD", false);
  run<1>(32, "DMUL+DADD", true); run<2>(384, "DMUL+DADD", true); run<4>(384, "DMUL+DADD", true);
  run<8>(512, "DMUL+DADD", true); run<4>(1024, "DMUL+DADD", true);
  return 0;
}
