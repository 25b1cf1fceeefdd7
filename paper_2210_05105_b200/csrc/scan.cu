// Deterministic tiled prefix scans (fixed 2048-element tiles, ordered carries), used for
// the CP-ARLS-LEV cdf (numpy cumsum analogue) and for sampled-fiber/row offsets.
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "scan.cuh"

namespace rcp {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;

template <typename T>
__device__ T block_inclusive(T v, T *warp_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_tot[wid] = v;
  __syncthreads();
  if (wid == 0) {
    T w = lane < (kScanThreads / 32) ? warp_tot[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (kScanThreads / 32)) warp_tot[lane] = w;
  }
  __syncthreads();
  if (wid > 0) v += warp_tot[wid - 1];
  return v;
}

template <typename T>
__device__ __forceinline__ int64_t dev_n(int64_t n_max, const int64_t *d_n) {
  if (!d_n) return n_max;
  int64_t n = *d_n;
  return n < n_max ? n : n_max;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
tile_sum_kernel(const T *__restrict__ in, int64_t n_max, const int64_t *d_n, T *__restrict__ sums) {
  __shared__ T wt[32];
  const int64_t n = dev_n<T>(n_max, d_n);
  const int64_t base = (int64_t)blockIdx.x * kTile;
  T s = 0;
  if (base < n) {
    const int64_t i0 = base + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (i0 + k < n) s += in[i0 + k];
  }
  T tot = block_inclusive<T>(s, wt);
  if (threadIdx.x == kScanThreads - 1) sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(1024) carry_kernel(T *__restrict__ sums, int64_t ntiles) {
  // exclusive scan of the tile sums in place, sequential over chunks of 1024
  __shared__ T wt[32];
  __shared__ T carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t c = 0; c < ntiles; c += 1024) {
    int64_t i = c + threadIdx.x;
    T v = i < ntiles ? sums[i] : T(0);
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wt[wid] = x;
    __syncthreads();
    if (wid == 0) {
      T w = wt[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wt[lane] = w;
    }
    __syncthreads();
    T incl = x + (wid > 0 ? wt[wid - 1] : T(0));
    T c0 = carry;
    if (i < ntiles) sums[i] = c0 + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + incl;
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
tile_scan_kernel(const T *__restrict__ in, int64_t n_max, const int64_t *d_n,
                 const T *__restrict__ offs, T *__restrict__ out, int exclusive) {
  __shared__ T wt[32];
  const int64_t n = dev_n<T>(n_max, d_n);
  const int64_t base = (int64_t)blockIdx.x * kTile;
  if (base >= n) {
    if (exclusive && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
    return;
  }
  const int64_t i0 = base + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (i0 + k < n) ? in[i0 + k] : T(0);
    s += v[k];
  }
  T incl = block_inclusive<T>(s, wt);
  T run = offs[blockIdx.x] + incl - s;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    run += v[k];
    if (i0 + k < n) {
      if (exclusive) out[i0 + k + 1] = run; else out[i0 + k] = run;
    }
  }
  if (exclusive && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

template <typename T>
int scan_impl(const T *in, T *out, int64_t n_max, const int64_t *d_n, void *ws, int exclusive,
              cudaStream_t st) {
  if (n_max <= 0) {
    if (exclusive) RCP_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(T), st));
    return RCP_OK;
  }
  const int64_t ntiles = ceil_div(n_max, kTile);
  T *sums = reinterpret_cast<T *>(ws);
  tile_sum_kernel<T><<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n_max, d_n, sums);
  RCP_LAUNCH_CHECK("scan_tiles");
  carry_kernel<T><<<1, 1024, 0, st>>>(sums, ntiles);
  RCP_LAUNCH_CHECK("scan_carry");
  tile_scan_kernel<T><<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n_max, d_n, sums, out,
                                                                 exclusive);
  RCP_LAUNCH_CHECK("scan_apply");
  return RCP_OK;
}

}  // namespace

static size_t cub_scan_bytes(int64_t n_items) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t *)nullptr, (int64_t *)nullptr,
                                (int)(n_items > 0 ? n_items : 1));
  return b;
}

size_t scan_ws_bytes(int64_t n_max) {
  const size_t tiles = (size_t)(ceil_div(n_max > 0 ? n_max : 1, kTile) + 1) * 8;
  const size_t cb = cub_scan_bytes(n_max + 1) + 256;
  return tiles > cb ? tiles : cb;
}

int scan_f64_inclusive(const double *in, double *out, int64_t n, void *ws, cudaStream_t st) {
  return scan_impl<double>(in, out, n, nullptr, ws, 0, st);
}

// Integer offsets: one CUB decoupled-look-back pass over n_max + 1 items (exact in any
// order).  out[i] for i <= n depends only on in[0, n), so the device count d_n needs no
// host round trip; in[] must have n_max + 1 readable items.
int scan_i64_exclusive(const int64_t *in, int64_t *out, int64_t n_max, const int64_t *d_n,
                       void *ws, cudaStream_t st) {
  (void)d_n;
  if (n_max < 0) return RCP_ERR_ARG;
  size_t bytes = cub_scan_bytes(n_max + 1);
  RCP_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws, bytes, in, out, (int)(n_max + 1), st));
  RCP_LAUNCH_CHECK("scan_i64");
  return RCP_OK;
}

}  // namespace rcp
