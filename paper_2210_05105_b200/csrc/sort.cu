// Stable device orderings for the one-time store build and the drop-in CSR gather
// (ref matricization.py:56-77 lexsort((rows, keys)); ref mttkrp.py:131-155 counting-sort
// transpose): LSD radix sorts of non-negative int64 keys carrying positions, so equal keys
// keep their input order exactly like numpy's stable sorts.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

extern "C" int rcp_device_sms();

namespace rcp {
namespace {

__global__ void iota_kernel(int64_t *__restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

__global__ void gather_keys_kernel(const int64_t *__restrict__ key, const int64_t *__restrict__ pos,
                                   int64_t n, uint64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint64_t)key[pos[i]];
}

int bit_length(int64_t v) {
  int b = 1;
  while (b < 63 && ((int64_t)1 << b) <= v) ++b;
  return b;
}

size_t cub_sort_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const int64_t *)nullptr, (int64_t *)nullptr, n > 0 ? n : 1, 0,
                                  64);
  return b;
}

int sm_count() {
  static int s = 0;
  if (!s) {
    s = rcp_device_sms();
    if (!s) s = 148;
  }
  return s;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

unsigned grid_for(int64_t n) {
  int64_t b = ceil_div(n, 256);
  const int64_t cap = 32LL * sm_count();
  return (unsigned)(b > cap ? cap : b);
}

}  // namespace
}  // namespace rcp

using namespace rcp;

extern "C" {

// two key buffers + one position buffer + the radix sort's own scratch
size_t rcp_sort_ws_bytes(int64_t n) {
  const size_t a = align256(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  return 3 * a + align256(cub_sort_bytes(n)) + 256;
}

int rcp_order_by_key_row(const int64_t *d_key, const int64_t *d_row, int64_t n, int64_t key_max,
                         int64_t row_max, int64_t *d_order, void *d_ws, size_t ws_bytes,
                         void *stream) {
  if (n < 0 || key_max < 0 || row_max < 0) return RCP_ERR_ARG;
  if (n == 0) return RCP_OK;
  if (!d_row || !d_order || !d_ws || ws_bytes < rcp_sort_ws_bytes(n)) return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  const size_t a = align256(sizeof(int64_t) * (size_t)n);
  char *w = (char *)d_ws;
  uint64_t *kA = (uint64_t *)w, *kB = (uint64_t *)(w + a);
  int64_t *vB = (int64_t *)(w + 2 * a);
  void *tmp = w + 3 * a;
  size_t tb = cub_sort_bytes(n);
  const unsigned g = grid_for(n);
  if (!d_key) {   // argsort of d_row alone
    iota_kernel<<<g, 256, 0, st>>>(vB, n);
    RCP_LAUNCH_CHECK("sort_iota");
    RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, (const uint64_t *)d_row, kB, vB, d_order, n,
                                                 0, bit_length(row_max), st));
    return RCP_OK;
  }
  // minor key first: rows, carrying the input positions
  int64_t *o1 = vB;
  iota_kernel<<<g, 256, 0, st>>>(d_order, n);
  RCP_LAUNCH_CHECK("sort_iota");
  RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, (const uint64_t *)d_row, kB, d_order, o1, n,
                                               0, bit_length(row_max), st));
  // major key: the column key at those positions, stable
  gather_keys_kernel<<<g, 256, 0, st>>>(d_key, o1, n, kA);
  RCP_LAUNCH_CHECK("sort_gather");
  RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, kA, kB, o1, d_order, n, 0,
                                               bit_length(key_max), st));
  return RCP_OK;
}

}  // extern "C"
