// On-device ingest for the tensors too large to build on the host (row F2 of SURVEY.md
// 8(f): C4 1.7B nonzeros, C5 4.7B).  Ref: sum_duplicates tensor.py:72-83, permute_modes
// tensor.py:182-210 (the synthetic draws stand in for load_frostt tensor.py:86-149).
//
// Draws are counter-based (a splitmix64 hash of (seed, chunk, index, salt)), so any range
// of the draw sequence can be regenerated independently: the generator makes one pass per
// hash partition of the cell space and keeps only that partition's draws, which bounds
// the working set to draws / parts cells.  The stream is the one synth.zipf_tensor uses
// (torch), so both produce the same coordinates for the same chunking.
//
// Zipf indices are inverse-CDF draws (first i with cdf[i] > u, numpy/torch searchsorted
// side='right') started from a guide table and corrected in both directions, so the
// result equals the binary search exactly.
#include <math.h>

#include "common.cuh"

using namespace rcp;

namespace {

constexpr int kMaxModes = 8;
constexpr int kPoisK = 40;

struct ZipfTables {
  const double *cdf[kMaxModes];
  const int32_t *guide[kMaxModes];
  int64_t n[kMaxModes];
  int64_t G[kMaxModes];
  uint64_t stride[kMaxModes];   // row-major cell id strides (mode 0 slowest)
};

struct PoissonTable {
  double cdf[kPoisK];
};

struct PermPtrs {
  const int32_t *p[kMaxModes];   // device permutation of each mode (NULL: identity)
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// synth._splitmix_uniform: z = (i + base*phi + salt*2^40) * phi, splitmix finaliser.
__device__ __forceinline__ double splitmix_uniform(uint64_t base, uint64_t i, uint64_t salt) {
  const uint64_t phi = 0x9E3779B97F4A7C15ull;
  uint64_t z = (i + base * phi + (salt << 40)) * phi;
  z = mix64(z);
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ int64_t zipf_index(const ZipfTables &T, int m, double u) {
  const double *cdf = T.cdf[m];
  const int64_t n = T.n[m];
  int64_t b = (int64_t)(u * (double)T.G[m]);
  if (b >= T.G[m]) b = T.G[m] - 1;
  int64_t i = T.guide[m][b];
  while (i > 0 && cdf[i - 1] > u) --i;
  while (i < n && cdf[i] <= u) ++i;
  return i < n ? i : n - 1;
}

__global__ void guide_kernel(const double *__restrict__ cdf, int64_t n, int64_t G,
                             int32_t *__restrict__ guide) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= G) return;
  const double x = (double)b / (double)G;
  int64_t lo = 0, hi = n;   // first i with cdf[i] > x
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > x) hi = mid; else lo = mid + 1;
  }
  guide[b] = (int32_t)(lo < n ? lo : n - 1);
}

// value kinds: 0 lognormal(0, sigma), 1 Poisson(3) counts (log1p applied after summing)
__global__ void __launch_bounds__(256)
zipf_draws_kernel(ZipfTables T, int N, uint64_t seed, int chunk_bits, int64_t d0, int64_t d1,
                  int vkind, double sigma, PoissonTable pois, int part_bits, uint64_t part,
                  int64_t *__restrict__ out_key, double *__restrict__ out_val,
                  unsigned long long *__restrict__ count, int64_t cap, int *status) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t mask = (1ull << chunk_bits) - 1ull;
  for (int64_t base_d = d0 + blockIdx.x * (int64_t)blockDim.x; base_d < d1;
       base_d += stride) {   // warp-uniform trip count
    const int64_t d = base_d + threadIdx.x;
    bool keep = d < d1;
    uint64_t lin = 0;
    double v = 0.0;
    if (keep) {
      const uint64_t rnd = (uint64_t)d >> chunk_bits, i = (uint64_t)d & mask;
      const uint64_t b = seed * 1000ull + rnd;
      for (int m = 0; m < N; ++m) {
        const double u = splitmix_uniform(b, i, (uint64_t)(m + 1));
        lin += (uint64_t)zipf_index(T, m, u) * T.stride[m];
      }
      if (part_bits > 0) keep = (mix64(lin) >> (64 - part_bits)) == part;
      if (keep) {
        const double u1 = splitmix_uniform(b, i, 101);
        if (vkind == 0) {
          const double u2 = splitmix_uniform(b, i, 102);
          const double z = sqrt(-2.0 * log1p(-u1)) * cos(2.0 * M_PI * u2);
          v = exp(sigma * z);
        } else {
          int k = 0;
          while (k < kPoisK && pois.cdf[k] <= u1) ++k;
          v = (double)k;
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (!bal) continue;
    unsigned long long basep = 0;
    if (lane == 0) basep = atomicAdd(count, (unsigned long long)__popc(bal));
    basep = __shfl_sync(0xffffffffu, basep, 0);
    if (keep) {
      const int64_t o = (int64_t)basep + __popc(bal & ((1u << lane) - 1u));
      if (o < cap) {
        out_key[o] = (int64_t)lin;
        out_val[o] = v;
      } else {
        raise_status(status, RCP_ST_CAPACITY);
      }
    }
  }
}

// Sorted keys (equal cells adjacent): segment starts of the distinct cells.
__global__ void run_flags_kernel(const int64_t *__restrict__ k, int64_t n, int32_t *__restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// Per distinct cell: sum of its draws' values in draw order (the sort is stable), decoded
// coordinates (row-major cell id), optionally permuted (idx'[m] = perm_m[idx[m]]), and for
// Poisson counts ln(1 + count) (ref tensor.py:145-148 dedup-then-log1p).
__global__ void cells_kernel(const int64_t *__restrict__ skey, const double *__restrict__ sval,
                             const int64_t *__restrict__ starts, int64_t n_cells, int64_t n,
                             ZipfTables T, int N, PermPtrs perm, int log1p_vals,
                             int32_t *__restrict__ idx_out, double *__restrict__ val_out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  const int64_t a = starts[c], b = c + 1 < n_cells ? starts[c + 1] : n;
  double s = 0.0;
  for (int64_t e = a; e < b; ++e) s += sval[e];
  val_out[c] = log1p_vals ? log1p(s) : s;
  uint64_t lin = (uint64_t)skey[a];
  for (int m = 0; m < N; ++m) {
    const uint64_t q = lin / T.stride[m];
    lin -= q * T.stride[m];
    const int32_t i = (int32_t)q;
    idx_out[c * N + m] = perm.p[m] ? perm.p[m][i] : i;
  }
}

int sm_count() {
  static int s = 0;
  if (!s) {
    s = rcp_device_sms();
    if (!s) s = 148;
  }
  return s;
}

int fill_tables(ZipfTables &T, int N, const int64_t *h_dims, const double *const *h_cdf,
                const int32_t *const *h_guide, const int64_t *h_G) {
  if (N < 1 || N > kMaxModes) return RCP_ERR_ARG;
  uint64_t s = 1;
  for (int m = N - 1; m >= 0; --m) {
    if (h_dims[m] < 1 || h_dims[m] >= (1LL << 31)) return RCP_ERR_ARG;
    T.stride[m] = s;
    const unsigned __int128 nxt = (unsigned __int128)s * (uint64_t)h_dims[m];
    if (nxt > (unsigned __int128)UINT64_MAX) return RCP_ERR_ARG;   // cell ids must fit u64
    s = (uint64_t)nxt;
  }
  for (int m = 0; m < kMaxModes; ++m) {
    T.cdf[m] = m < N ? h_cdf[m] : nullptr;
    T.guide[m] = m < N && h_guide ? h_guide[m] : nullptr;
    T.n[m] = m < N ? h_dims[m] : 1;
    T.G[m] = m < N && h_G ? h_G[m] : 1;
  }
  return RCP_OK;
}

}  // namespace

extern "C" {

int rcp_zipf_guide(const double *d_cdf, int64_t n, int64_t G, int32_t *d_guide, void *stream) {
  if (n < 1 || G < 1 || n >= (1LL << 31) || !d_cdf || !d_guide) return RCP_ERR_ARG;
  guide_kernel<<<(unsigned)ceil_div(G, 256), 256, 0, RCP_STREAM(stream)>>>(d_cdf, n, G, d_guide);
  RCP_LAUNCH_CHECK("zipf_guide");
  return RCP_OK;
}

int rcp_zipf_draws(int N, const int64_t *h_dims, const double *const *h_cdf,
                   const int32_t *const *h_guide, const int64_t *h_G, uint64_t seed,
                   int chunk_bits, int64_t d0, int64_t d1, int value_kind, double sigma,
                   int part_bits, int64_t part, int64_t *d_key, double *d_val, int64_t *d_count,
                   int64_t cap, int *d_status, void *stream) {
  if (!h_dims || !h_cdf || !h_guide || !h_G || chunk_bits < 1 || chunk_bits > 62 || d0 < 0 ||
      d1 < d0 || value_kind < 0 || value_kind > 1 || part_bits < 0 || part_bits > 16 ||
      part < 0 || part >= (1LL << part_bits) || !d_count || cap < 0)
    return RCP_ERR_ARG;
  ZipfTables T;
  if (fill_tables(T, N, h_dims, h_cdf, h_guide, h_G)) return RCP_ERR_ARG;
  for (int m = 0; m < N; ++m)
    if (!T.cdf[m] || !T.guide[m]) return RCP_ERR_ARG;
  if (d1 == d0) return RCP_OK;
  if (!d_key || !d_val) return RCP_ERR_ARG;
  PoissonTable P;
  {   // synth._poisson3: the same IEEE operations in the same order
    const double lam = 3.0;
    double p = exp(-lam);
    P.cdf[0] = p;
    for (int k = 1; k < kPoisK; ++k) {
      p = p * lam / k;
      P.cdf[k] = P.cdf[k - 1] + p;
    }
  }
  int64_t blocks = ceil_div(d1 - d0, 256);
  if (blocks > 32LL * sm_count()) blocks = 32LL * sm_count();
  zipf_draws_kernel<<<(unsigned)blocks, 256, 0, RCP_STREAM(stream)>>>(
      T, N, seed, chunk_bits, d0, d1, value_kind, sigma, P, part_bits, (uint64_t)part, d_key,
      d_val, (unsigned long long *)d_count, cap, d_status);
  RCP_LAUNCH_CHECK("zipf_draws");
  return RCP_OK;
}

// d_flag[i] = 1 where a new cell starts in the sorted key array.
int rcp_run_flags(const int64_t *d_sorted, int64_t n, int32_t *d_flag, void *stream) {
  if (n < 0 || (n > 0 && (!d_sorted || !d_flag))) return RCP_ERR_ARG;
  if (n == 0) return RCP_OK;
  run_flags_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, RCP_STREAM(stream)>>>(d_sorted, n, d_flag);
  RCP_LAUNCH_CHECK("run_flags");
  return RCP_OK;
}

int rcp_cells(const int64_t *d_sorted, const double *d_sval, const int64_t *d_starts,
              int64_t n_cells, int64_t n, int N, const int64_t *h_dims,
              const int32_t *const *h_perm, int log1p_vals, int32_t *d_idx, double *d_val,
              void *stream) {
  if (n_cells < 0 || n < n_cells || !h_dims) return RCP_ERR_ARG;
  if (n_cells == 0) return RCP_OK;
  if (!d_sorted || !d_sval || !d_starts || !d_idx || !d_val) return RCP_ERR_ARG;
  ZipfTables T;
  const double *nocdf[kMaxModes] = {};
  if (fill_tables(T, N, h_dims, nocdf, nullptr, nullptr)) return RCP_ERR_ARG;
  PermPtrs pp;
  for (int m = 0; m < kMaxModes; ++m) pp.p[m] = (h_perm && m < N) ? h_perm[m] : nullptr;
  cells_kernel<<<(unsigned)ceil_div(n_cells, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_sorted, d_sval, d_starts, n_cells, n, T, N, pp, log1p_vals, d_idx, d_val);
  RCP_LAUNCH_CHECK("cells");
  return RCP_OK;
}

}  // extern "C"
