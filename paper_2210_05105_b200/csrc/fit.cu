// Exact fit and exact MTTKRP from the device-resident mode store (row F1 of SURVEY.md 8(f)).
// Ref: compute_fit linalg.py:130-151 and mttkrp_exact mttkrp.py:65-108.
//
// The fit needs three scalars:
//   ||T||^2            = sum_e v_e^2                              (rcp_sum_squares)
//   <T, T_hat>         = sum_e v_e sum_r sigma_r prod_m U_m[i_m(e), r]   (rcp_fit_cross)
//   ||T_hat||^2        = sigma^T (Hadamard of the Grams) sigma     (rcp_model_norm)
// The cross term walks a mode-k store fiber by fiber: a fiber's off-mode indices come
// from its column key (mixed radix, earlier modes fastest, ref matricization.py:21-64), so
// g = sigma (.) prod_{m != k} U_m[i_m] is formed once per fiber and every entry adds
// v * <U_k[row], g>.  One pass over the store: 12 B per entry plus one factor-row gather,
// no atomics.  Partial sums land in per-chunk slots and are added in a fixed order, so the
// result is bit-reproducible run to run.
//
// The exact MTTKRP (drop-in `mttkrp_exact`) uses the same traversal with h = prod_{m != k}
// U_m[i_m] and adds v * h into out[row] with fp64 red.global (off the sampled hot path).
#include "common.cuh"

using namespace rcp;

namespace {

constexpr int kMaxModes = 8;
constexpr int kFitChunk = 256;   // entries per warp work item
constexpr int kReduceThreads = 1024;

struct Factors {
  const double *U[kMaxModes];   // full (or gathered) factor of each mode, row-major n_m x R
  int64_t lo[kMaxModes];        // global index of U[m]'s first row
  int64_t dims[kMaxModes];
  int64_t stride[kMaxModes];    // key strides of the store's off-mode key (0 for mode k)
};

// largest c in [0, n) with a[c] <= x
__device__ __forceinline__ int64_t floor_idx(const int64_t *__restrict__ a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// Lane's columns (c = lane + 32 j) of prod_{m != k} U_m[i_m(key)] (times sigma if given).
template <int NP>
__device__ __forceinline__ void fiber_row(const Factors &F, int N, int k, int64_t key, int R,
                                          const double *__restrict__ sigma, int lane,
                                          double (&g)[NP]) {
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int c = lane + 32 * j;
    g[j] = (sigma && c < R) ? sigma[c] : 1.0;
  }
  for (int m = 0; m < N; ++m) {
    if (m == k) continue;
    const int64_t i = (key / F.stride[m]) % F.dims[m];
    const double *u = F.U[m] + (i - F.lo[m]) * R;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int c = lane + 32 * j;
      if (c < R) g[j] *= u[c];
    }
  }
}

// MODE 0: cross-term partials (one per chunk); MODE 1: exact MTTKRP scatter-add.
template <int NP, int MODE>
__global__ void __launch_bounds__(256)
store_pass_kernel(const int64_t *__restrict__ keys, const int64_t *__restrict__ colptr,
                  int64_t n_cols, const int32_t *__restrict__ rows, const double *__restrict__ vals,
                  int64_t nnz, Factors F, int N, int k, const double *__restrict__ Uk, int R,
                  const double *__restrict__ sigma, double *__restrict__ partials,
                  double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = ceil_div(nnz, kFitChunk);
  for (int64_t ch = warp0; ch < nchunks; ch += nwarps) {
    const int64_t c0 = ch * kFitChunk, c1 = min(c0 + kFitChunk, nnz);
    int64_t col = floor_idx(colptr, n_cols + 1, c0);
    double acc = 0.0;
    double g[NP];
    int64_t e = c0;
    int64_t ce = -1;   // end of the current fiber's entries (g valid for [.., ce))
    for (int64_t base = c0; base < c1; base += 32) {
      const int nb = (int)min((int64_t)32, c1 - base);
      int32_t mr = 0;
      double mv = 0.0;
      if (lane < nb) {
        mr = rows[base + lane];
        mv = vals[base + lane];
      }
      for (int q = 0; q < nb; ++q) {
        e = base + q;
        while (e >= ce) {   // next fiber (warp-uniform)
          if (ce >= 0) ++col;
          ce = colptr[col + 1];
          if (e < ce) fiber_row<NP>(F, N, k, keys[col], R, MODE == 0 ? sigma : nullptr, lane, g);
        }
        const int32_t row = __shfl_sync(0xffffffffu, mr, q);
        const double v = __shfl_sync(0xffffffffu, mv, q);
        const double *u = Uk + (int64_t)row * R;
        if (MODE == 0) {
          double d = 0.0;
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            const int c = lane + 32 * j;
            if (c < R) d = fma(u[c], g[j], d);
          }
          acc = fma(v, d, acc);
        } else {
          double *o = out + (int64_t)row * R;
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            const int c = lane + 32 * j;
            if (c < R) atomicAdd(o + c, v * g[j]);
          }
        }
      }
    }
    if (MODE == 0) {
      acc = warp_sum(acc);
      if (lane == 0) partials[ch] = acc;
    }
  }
}

__global__ void square_partials_kernel(const double *__restrict__ v, int64_t n,
                                       double *__restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = ceil_div(n, kFitChunk);
  for (int64_t ch = warp0; ch < nchunks; ch += nwarps) {
    const int64_t c0 = ch * kFitChunk, c1 = min(c0 + kFitChunk, n);
    double acc = 0.0;
    for (int64_t e = c0 + lane; e < c1; e += 32) acc = fma(v[e], v[e], acc);
    acc = warp_sum(acc);
    if (lane == 0) partials[ch] = acc;
  }
}

// Fixed-order sum of n partials (one CTA): deterministic for a given n.
__global__ void __launch_bounds__(kReduceThreads)
reduce_fixed_kernel(const double *__restrict__ p, int64_t n, double *__restrict__ out) {
  __shared__ double s[kReduceThreads];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kReduceThreads) a += p[i];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int w = kReduceThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = s[0];
}

// sigma^T (G_0 (.) G_1 (.) ... ) sigma, Hadamard folded left to right in mode order
// (ref hadamard_gram_chain linalg.py:73-82 then sigma @ chain @ sigma, linalg.py:146).
__global__ void model_norm_kernel(const double *__restrict__ grams, int N, int R,
                                  const double *__restrict__ sigma, double *__restrict__ out) {
  __shared__ double s[1024];
  double a = 0.0;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double h = grams[e];
    for (int m = 1; m < N; ++m) h *= grams[(int64_t)m * R * R + e];
    a = fma(sigma[e / R] * h, sigma[e % R], a);
  }
  s[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = s[0];
}

int sm_count() {
  static int s = 0;
  if (!s) {
    s = rcp_device_sms();
    if (!s) s = 148;
  }
  return s;
}

int fill_factors(Factors &F, int N, int k, const int64_t *h_dims, const int64_t *h_strides,
                 const double *const *h_U, const int64_t *h_lo) {
  for (int m = 0; m < kMaxModes; ++m) {
    F.U[m] = nullptr;
    F.lo[m] = 0;
    F.dims[m] = 1;
    F.stride[m] = 1;
  }
  for (int m = 0; m < N; ++m) {
    F.dims[m] = h_dims[m];
    if (m == k) continue;
    if (!h_U[m] || h_strides[m] < 1 || h_dims[m] < 1) return RCP_ERR_ARG;
    F.U[m] = h_U[m];
    F.lo[m] = h_lo ? h_lo[m] : 0;
    F.stride[m] = h_strides[m];
  }
  return RCP_OK;
}

template <int MODE>
int launch_store_pass(const int64_t *keys, const int64_t *colptr, int64_t n_cols,
                      const int32_t *rows, const double *vals, int64_t nnz, const Factors &F,
                      int N, int k, const double *Uk, int R, const double *sigma,
                      double *partials, double *out, cudaStream_t st) {
  int64_t blocks = ceil_div(ceil_div(nnz, kFitChunk), 8);
  if (blocks > 8LL * sm_count()) blocks = 8LL * sm_count();
  if (blocks < 1) blocks = 1;
  const unsigned b = (unsigned)blocks;
  switch ((R + 31) / 32) {
    case 1: store_pass_kernel<1, MODE><<<b, 256, 0, st>>>(keys, colptr, n_cols, rows, vals, nnz, F, N, k, Uk, R, sigma, partials, out); break;
    case 2: store_pass_kernel<2, MODE><<<b, 256, 0, st>>>(keys, colptr, n_cols, rows, vals, nnz, F, N, k, Uk, R, sigma, partials, out); break;
    case 3: store_pass_kernel<3, MODE><<<b, 256, 0, st>>>(keys, colptr, n_cols, rows, vals, nnz, F, N, k, Uk, R, sigma, partials, out); break;
    default: store_pass_kernel<4, MODE><<<b, 256, 0, st>>>(keys, colptr, n_cols, rows, vals, nnz, F, N, k, Uk, R, sigma, partials, out); break;
  }
  RCP_LAUNCH_CHECK(MODE == 0 ? "fit_cross" : "exact_mttkrp");
  return RCP_OK;
}

}  // namespace

extern "C" {

size_t rcp_fit_ws_bytes(int64_t nnz) {
  return sizeof(double) * (size_t)(ceil_div(nnz > 0 ? nnz : 1, kFitChunk) + 1);
}

int rcp_fit_cross(const int64_t *d_keys, const int64_t *d_colptr, int64_t n_cols,
                  const int32_t *d_rows, const double *d_vals, int64_t nnz, int N, int k,
                  const int64_t *h_dims, const int64_t *h_strides, const double *const *h_U,
                  const int64_t *h_lo, const double *d_Uk, int R, const double *d_sigma,
                  double *d_out, void *d_ws, size_t ws_bytes, void *stream) {
  if (N < 2 || N > kMaxModes || k < 0 || k >= N || R < 1 || R > RCP_MAX_RANK || nnz < 0 ||
      n_cols < 0 || !h_dims || !h_strides || !h_U || !d_out)
    return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (nnz == 0) {
    RCP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    return RCP_OK;
  }
  if (!d_keys || !d_colptr || !d_rows || !d_vals || !d_Uk || !d_sigma || !d_ws ||
      ws_bytes < rcp_fit_ws_bytes(nnz))
    return RCP_ERR_ARG;
  Factors F;
  if (fill_factors(F, N, k, h_dims, h_strides, h_U, h_lo)) return RCP_ERR_ARG;
  double *partials = (double *)d_ws;
  int rc = launch_store_pass<0>(d_keys, d_colptr, n_cols, d_rows, d_vals, nnz, F, N, k, d_Uk, R,
                                d_sigma, partials, nullptr, st);
  if (rc) return rc;
  reduce_fixed_kernel<<<1, kReduceThreads, 0, st>>>(partials, ceil_div(nnz, kFitChunk), d_out);
  RCP_LAUNCH_CHECK("fit_reduce");
  return RCP_OK;
}

int rcp_sum_squares(const double *d_v, int64_t n, double *d_out, void *d_ws, size_t ws_bytes,
                    void *stream) {
  if (n < 0 || !d_out) return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (n == 0) {
    RCP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    return RCP_OK;
  }
  if (!d_v || !d_ws || ws_bytes < rcp_fit_ws_bytes(n)) return RCP_ERR_ARG;
  double *partials = (double *)d_ws;
  int64_t blocks = ceil_div(ceil_div(n, kFitChunk), 8);
  if (blocks > 8LL * sm_count()) blocks = 8LL * sm_count();
  square_partials_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_v, n, partials);
  RCP_LAUNCH_CHECK("sum_squares");
  reduce_fixed_kernel<<<1, kReduceThreads, 0, st>>>(partials, ceil_div(n, kFitChunk), d_out);
  RCP_LAUNCH_CHECK("sum_squares_reduce");
  return RCP_OK;
}

int rcp_model_norm(const double *d_grams, int N, int R, const double *d_sigma, double *d_out,
                   void *stream) {
  if (N < 1 || R < 1 || R > RCP_MAX_RANK || !d_grams || !d_sigma || !d_out) return RCP_ERR_ARG;
  model_norm_kernel<<<1, 1024, 0, RCP_STREAM(stream)>>>(d_grams, N, R, d_sigma, d_out);
  RCP_LAUNCH_CHECK("model_norm");
  return RCP_OK;
}

int rcp_exact_mttkrp(const int64_t *d_keys, const int64_t *d_colptr, int64_t n_cols,
                     const int32_t *d_rows, const double *d_vals, int64_t nnz, int64_t n_rows,
                     int N, int k, const int64_t *h_dims, const int64_t *h_strides,
                     const double *const *h_U, const int64_t *h_lo, int R, double *d_out,
                     void *stream) {
  if (N < 2 || N > kMaxModes || k < 0 || k >= N || R < 1 || R > RCP_MAX_RANK || nnz < 0 ||
      n_rows < 0 || n_cols < 0 || !h_dims || !h_strides || !h_U)
    return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (n_rows == 0) return RCP_OK;
  if (!d_out) return RCP_ERR_ARG;
  RCP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double) * n_rows * R, st));
  if (nnz == 0) return RCP_OK;
  if (!d_keys || !d_colptr || !d_rows || !d_vals) return RCP_ERR_ARG;
  Factors F;
  if (fill_factors(F, N, k, h_dims, h_strides, h_U, h_lo)) return RCP_ERR_ARG;
  return launch_store_pass<1>(d_keys, d_colptr, n_cols, d_rows, d_vals, nnz, F, N, k, nullptr, R,
                              nullptr, nullptr, d_out, st);
}

}  // extern "C"
