// Experiment harness (not product code): bandwidth probes behind the sampled-MTTKRP design
// (L2 reduction and gather rates).  Built by tools/lab/run_lab.py into
// tools/lab/libspmm_lab.so together with the product sources.  The SpMM variants measured
// with it earlier (cache hints on the Hs gather, a fused row-ordering + SpMM kernel) are
// recorded in DESIGN.md section 4.
#include "../../paper_2210_05105_b200/csrc/mttkrp.cu"

// ---------------------------------------------------------------- L2 red / gather probes
namespace {
__global__ void red_probe_kernel(double *out, int64_t n_rows, int R, int64_t nflush, int mode) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t f = w0; f < nflush; f += nw) {
    const int64_t row = (int64_t)(mix64((uint64_t)f) % (uint64_t)n_rows);
    const int c = 2 * lane;
    if (c < R) {
      double *o = out + row * R + c;
      if (mode == 0) {
        atomicAdd(o, 1.0);
        atomicAdd(o + 1, 1.0);
      } else if (mode == 1) {
        atomicAdd(o, 1.0);
      } else {
        const double2 h = *reinterpret_cast<const double2 *>(out + row * 64 + c);
        acc += h.x + h.y;
      }
    }
  }
  if (mode == 2 && acc == 12345.0) out[0] = acc;
}
}  // namespace

extern "C" int lab_red_probe(double *d_out, int64_t n_rows, int R, int64_t nflush, int mode,
                             float *ms_out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    red_probe_kernel<<<8 * sm_count(), 256>>>(d_out, n_rows, R, nflush, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  *ms_out = best;
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- L2 gather peak probe
// Random 400-B row gathers (25 lanes x double2 of 512-B-strided rows, the SpMM's Hs access)
// with 8 independent loads in flight per lane: the L2 -> SM gather bandwidth the segmented
// SpMM is bound by.
namespace {
__global__ void __launch_bounds__(256)
gather_probe_kernel(const double2 *__restrict__ tab, int64_t rows, int64_t n, double *sink) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double2 acc = make_double2(0.0, 0.0);
  const int32_t *idx = reinterpret_cast<const int32_t *>(sink + 8);
  for (int64_t g = w0 * 32; g < n; g += nw * 32) {
   const int32_t mine = idx[g + lane];
   for (int q = 0; q < 32; q += 8) {
    double2 h[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = __shfl_sync(0xffffffffu, mine, q + u);
      h[u] = lane < 25 ? tab[r * 32 + lane] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc.x += h[u].x;
      acc.y += h[u].y;
    }
   }
  }
  if (acc.x == 1234.5) sink[0] = acc.y;
}
}  // namespace

extern "C" int lab_gather_probe(const double *d_tab, int64_t rows, int64_t n, double *d_sink,
                                float *ms_out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    gather_probe_kernel<<<8 * sm_count(), 256>>>((const double2 *)d_tab, rows, n, d_sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  *ms_out = best;
  return (int)cudaGetLastError();
}
