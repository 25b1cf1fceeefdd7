// FP64 peak probes ("measure FP64 FMA and DMMA peaks on the box"):
// every warp of a full grid issues independent chains of mma.sync.m8n8k4.f64 (512 flop per
// warp instruction) or of DFMA (2 flop per thread instruction) from registers only.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dmma_probe_kernel(double *sink, int iters) {
  double c[kChains][2];
#pragma unroll
  for (int j = 0; j < kChains; ++j) c[j][0] = c[j][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - blockIdx.x * 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_probe_kernel(double *sink, int iters) {
  double c[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) c[j] = j * 1e-3;
  const double a = 1.0 - threadIdx.x * 1e-12, b = 1e-9 * blockIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) c[j] = fma(c[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += c[j];
  if (s == 12345.0) sink[threadIdx.x] = s;
}

}  // namespace

// mode 0: DMMA, mode 1: DFMA.  Returns the best of 5 launches in ms and the flop count.
extern "C" int lab_fp64_probe(int mode, int ctas_per_sm, int iters, double *d_sink, float *ms_out,
                              double *flops_out) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * ctas_per_sm, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    if (mode == 0) dmma_probe_kernel<<<grid, threads>>>(d_sink, iters);
    else dfma_probe_kernel<<<grid, threads>>>(d_sink, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double warps = (double)grid * threads / 32;
  *flops_out = mode == 0 ? warps * iters * kChains * 512.0
                         : (double)grid * threads * iters * kChains * 2.0;
  *ms_out = best;
  return (int)cudaGetLastError();
}
