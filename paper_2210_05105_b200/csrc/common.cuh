// Shared device helpers for the randcp B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/randcp_b200.h"

namespace rcp {

void set_error(const char *msg);
int check_launch(const char *what);

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void raise_status(int *st, int flag) {
  if (st) atomicOr(st, flag);
}

// ----------------------------------------------------------------------------------------
// Philox4x64-10 (Random123 constants; numpy's bit generator).  Block b of a stream is the
// permutation of counter (b+1, 0, 0, 0) under the 2x64 key; draw m is word m%4 of block m/4.
// ----------------------------------------------------------------------------------------
struct U64x4 {
  uint64_t v[4];
};

__host__ __device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t &lo,
                                                   uint64_t &hi) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

__host__ __device__ __forceinline__ U64x4 philox4x64_10(U64x4 c, uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    uint64_t lo0, hi0, lo1, hi1;
    mulhilo64(0xD2E7470EE14C6C93ull, c.v[0], lo0, hi0);
    mulhilo64(0xCA5A826395121157ull, c.v[2], lo1, hi1);
    U64x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

// 64-bit word m of the stream (counter = m/4 + 1, 128-bit carry never reached here).
__host__ __device__ __forceinline__ uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t m) {
  U64x4 c;
  c.v[0] = (m >> 2) + 1;
  c.v[1] = 0;
  c.v[2] = 0;
  c.v[3] = 0;
  U64x4 o = philox4x64_10(c, k0, k1);
  return o.v[m & 3];
}

__host__ __device__ __forceinline__ double u64_to_unit(uint64_t x) {
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

// Largest double below 1 (ref samplers.py:31 _ONE_BELOW).
__host__ __device__ __forceinline__ double one_below() { return 0x1.fffffffffffffp-1; }

// Per-mode strides passed by value to kernels (N <= 8 modes).
struct Strides8 {
  int64_t s[8];
};

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

// Node stride of packed R x R Gram blocks: R(R+1)/2 rounded up to even (16-byte aligned
// nodes for vector loads; the pad element is zero).
__host__ __device__ __forceinline__ int tri_stride(int R) {
  const int t = R * (R + 1) / 2;
  return (t + 1) & ~1;
}

// Packed upper-triangular index of (a, b), a <= b, row-major.
__host__ __device__ __forceinline__ int tri_index(int a, int b, int R) {
  return a * R - (a * (a - 1)) / 2 + (b - a);
}

// ---- asynchronous staging of 8-row tiles (cp.async), shared by the tall-skinny mma kernels
__device__ __forceinline__ void cpa8_zfill(double *smem, const double *gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;   // src-size 0: the 8 destination bytes are zero-filled
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// wait until at most nbuf - 1 groups are pending (nbuf in 1..4)
__device__ __forceinline__ void cpa_wait_stages(int nbuf) {
  if (nbuf >= 4) cpa_wait<3>();
  else if (nbuf == 3) cpa_wait<2>();
  else if (nbuf == 2) cpa_wait<1>();
  else cpa_wait<0>();
}
// Rows r0 .. r0+7 of a row-major (n x R) matrix into a warp's tile with row stride zs:
// rows >= nb are zero-filled, columns >= R are left untouched (zero them once).
__device__ __forceinline__ void stage_tile8(double *tile, const double *__restrict__ src,
                                            int64_t r0, int nb, int R, int zs, int lane) {
  for (int c = lane; c < 8 * R; c += 32) {
    const int j = c / R, col = c - j * R;
    const bool ok = j < nb;
    cpa8_zfill(tile + j * zs + col, ok ? src + (r0 + j) * R + col : src, ok);
  }
}

}  // namespace rcp

#define RCP_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) {                                 \
      rcp::set_error(cudaGetErrorString(_e));                \
      return RCP_ERR_CUDA;                                   \
    }                                                        \
  } while (0)

#define RCP_LAUNCH_CHECK(name)                               \
  do {                                                       \
    int _r = rcp::check_launch(name);                        \
    if (_r) return _r;                                       \
  } while (0)

#define RCP_STREAM(s) (reinterpret_cast<cudaStream_t>(s))
