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

// ---- shared-memory staged slabs (64 < R <= 128): 32 rows per slab, row stride 8T + 4
// doubles (4 or 12 mod 16: the fragment reads of a half-warp hit 16 distinct double-banks);
// warp g of 8 owns the tile pairs of group g (gram_accum_group<T, 8, g>).
constexpr int kGsRows = 32;
constexpr int kGsStages = 3;

template <int T>
__host__ __device__ constexpr int gs_stride() { return 8 * T + 4; }

template <int T, int g>
__device__ __forceinline__ void gram_staged_body(const double *ring, const double *sc, bool scaled,
                                                 int lane, double (&acc)[(T * (T + 1) / 2 + 7) / 8][2]) {
  constexpr int ST = gs_stride<T>();
  const int kk = lane & 3, col = lane >> 2;
#pragma unroll 2
  for (int j = 0; j < kGsRows / 4; ++j) {
    const double *row = ring + (4 * j + kk) * ST + col;
    const double w = scaled ? sc[4 * j + kk] : 1.0;
    double f[T];
#pragma unroll
    for (int t = 0; t < T; ++t) f[t] = row[8 * t] * w;
    gram_accum_group<T, 8, g>(f, acc);
  }
}

}  // namespace rcp
