// Gram building blocks on the fp64 tensor cores (mma.m8n8k4), shared by the factor Gram
// (dense.cu) and the STS tree's leaf Grams (samplers.cu).  For a 4-row step of
// Z = diag(s) U, thread t of a warp holds Z[r0 + t%4][8 tile + t/4] for every 8-column
// tile: at once the A fragment (Z^T, row-major 8x4) and the B fragment (Z, col-major 4x8),
// so every upper tile pair (a <= b) of G = Z^T Z accumulates from registers.  Thread t's
// accumulator of pair (a, b) holds G[8a + t/4][8b + 2(t%4) + {0, 1}].
#pragma once
#include "common.cuh"

namespace rcp {

__device__ __forceinline__ void gram_dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int T>
__device__ __forceinline__ void gram_load(const double *__restrict__ U,
                                          const double *__restrict__ scale, int64_t r,
                                          int64_t rend, int R, int col, double (&f)[T]) {
  const bool ok = r < rend;
  const double sc = ok ? (scale ? scale[r] : 1.0) : 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int c = 8 * t + col;
    f[t] = (ok && c < R) ? U[r * R + c] * sc : 0.0;
  }
}

template <int T>
__device__ __forceinline__ void gram_accum(const double (&f)[T], double (&acc)[T * (T + 1) / 2][2]) {
  int p = 0;
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int b = a; b < T; ++b) {
      gram_dmma(acc[p][0], acc[p][1], f[a], f[b]);
      ++p;
    }
}


// The pairs of group g of G (a compile-time range of the T(T+1)/2 upper tile pairs): R > 64,
// where one warp cannot hold every pair's accumulators.
template <int T, int G, int g>
__device__ __forceinline__ void gram_accum_group(const double (&f)[T],
                                                 double (&acc)[(T * (T + 1) / 2 + G - 1) / G][2]) {
  constexpr int PPG = (T * (T + 1) / 2 + G - 1) / G;
  int p = 0;
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int b = a; b < T; ++b) {
      if (p >= g * PPG && p < (g + 1) * PPG) gram_dmma(acc[p - g * PPG][0], acc[p - g * PPG][1], f[a], f[b]);
      ++p;
    }
}

}  // namespace rcp
