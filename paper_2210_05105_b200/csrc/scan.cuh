#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rcp {
// Scratch bytes for a scan of up to n_max elements.
size_t scan_ws_bytes(int64_t n_max);
// out[i] = in[0] + ... + in[i] (fixed tiling => deterministic rounding).
int scan_f64_inclusive(const double *in, double *out, int64_t n, void *ws, cudaStream_t st);
// out[0] = 0, out[i+1] = in[0] + ... + in[i] for i < n, with n = *d_n (device, clamped to
// n_max) when d_n != nullptr, else n_max.
int scan_i64_exclusive(const int64_t *in, int64_t *out, int64_t n_max, const int64_t *d_n,
                       void *ws, cudaStream_t st);
}  // namespace rcp
