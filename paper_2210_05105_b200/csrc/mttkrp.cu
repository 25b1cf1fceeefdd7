// Sampled (downsampled) MTTKRP for one mode solve, device-resident and free of host
// synchronisation (all sizes stay on the device, so a whole ALS round can be captured in
// a CUDA graph).  Ref: gather_sampled_nonzeros_to_csr mttkrp.py:131-155 and
// downsampled_mttkrp mttkrp.py:158-189 (with _row_blocks/_accumulate_rows :31-62).
//
// Pipeline (per solve, per rank):
//  1. column key of every sample; hash-dedup -> distinct fibers d with multiplicity c_d
//     and representative sample (smallest id);                       [dedup]
//  2. binary search of each distinct key in the mode's sorted store -> [lo_d, lo_d+len_d);
//     scaled KRP row Hs_d = c_d w^2 H[rep_d,:];                      [lookup]
//  3. exclusive scan of len_d -> gathered-entry offsets;            [scan]
//  4. row histogram of the gathered entries (CTA-private in shared memory when the
//     block's row count fits, one global atomic per (CTA,row));   [row count + scan]
//  5. scatter entries (fiber id, value) into row order (the "sparse transpose" the
//     paper uses instead of atomics);            [scatter]
//  6. warp-per-chunk segmented reduction out[i,:] = sum val * Hs_d, plain stores for rows
//     owned by one warp, fp64 red.add only for rows split across chunks.   [spmm]
#include <limits.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "scan.cuh"

using namespace rcp;

namespace {

int g_mttkrp_mode = -1;   // rcp_set_mttkrp_mode; -1: not yet read from the environment
int mttkrp_mode() {
  if (g_mttkrp_mode < 0) {
    const char *e = getenv("RCP_MTTKRP_PATH");
    g_mttkrp_mode = e && !strcmp(e, "tiles") ? 1 : 0;
  }
  return g_mttkrp_mode;
}

int sm_count() {
  static int s = 0;
  if (!s) {
    s = rcp_device_sms();
    if (!s) s = 148;
  }
  return s;
}

constexpr int kMaxModes = 8;
constexpr int kPrivRows = 49152;   // CTA-private row histogram limit (int32 in smem)
// (overridable at compile time for parameter sweeps: tools/lab/sweep_spmm.py)
#ifndef RCP_SPMM_CHUNK
#define RCP_SPMM_CHUNK 256
#endif
#ifndef RCP_SPMM_U
#define RCP_SPMM_U 4
#endif
#ifndef RCP_SPMM_GROUP
#define RCP_SPMM_GROUP 1   // 0: spmm_packed_kernel (entries broadcast by shuffles)
#endif
#ifndef RCP_SPMM_GU
#define RCP_SPMM_GU 2   // spmm_group_kernel, R in 33..64: batch steps with Hs loads in flight
#endif
#ifndef RCP_SPMM_GU5
#define RCP_SPMM_GU5 2   // spmm_group_kernel, R > 64
#endif
#ifndef RCP_SPMM_BLOCKS_PER_SM
#define RCP_SPMM_BLOCKS_PER_SM 8
#endif
constexpr int kSpmmChunk = RCP_SPMM_CHUNK;   // entries per warp in the segmented reduction
constexpr int64_t kItemE = 512;    // entries per traversal item (a fiber chunk)
[[maybe_unused]] constexpr int kSpmmU = RCP_SPMM_U;           // Hs-row loads in flight per lane

// Row stride of the scaled KRP rows Hs: a multiple of 16 doubles, so every row starts on a
// 128-byte line and a warp's double2 row load touches ceil(R/16) lines, not one more.
__host__ __device__ __forceinline__ int hs_stride(int R) { return (R + 15) & ~15; }

struct Strides {
  int64_t s[kMaxModes];
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t sample_key(const int64_t *__restrict__ X, int N, int64_t J,
                                              int k, const Strides &st, int64_t s) {
  int64_t key = 0;
  for (int m = 0; m < N; ++m)
    if (m != k) key += X[(int64_t)m * J + s] * st.s[m];
  return key;
}

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t *__restrict__ a, int64_t n,
                                                   int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// First i in [0, n) with a[i] >= x (n if none), found by a whole warp: 32 probes per step
// (about log_32 n dependent loads instead of log_2 n).  Every lane returns the answer.
__device__ __forceinline__ int64_t warp_lower_bound(const int64_t *__restrict__ a, int64_t n,
                                                    int64_t x, int lane) {
  int64_t lo = 0, hi = n;   // answer in [lo, hi]
  while (hi - lo >= 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t pos = lo + lane * step;
    const bool ge = pos < hi ? a[pos] >= x : true;
    const unsigned m = __ballot_sync(0xffffffffu, ge);
    if (m == 0u) {
      lo = lo + 31 * step + 1;
    } else {
      const int f = __ffs(m) - 1;
      if (f == 0) return lo;   // a[lo] >= x
      const int64_t nlo = lo + (f - 1) * step + 1;
      hi = min(hi, lo + f * step);
      lo = nlo;
    }
  }
  const int64_t pos = lo + lane;
  const bool ge = pos < hi ? a[pos] >= x : true;
  const unsigned m = __ballot_sync(0xffffffffu, ge);
  return lo + (__ffs(m) - 1);   // hi - lo <= 31: lane hi - lo always reports true
}

// largest i in [0, n) with a[i] <= x  (a nondecreasing, a[0] <= x)
__device__ __forceinline__ int64_t floor_index(const int64_t *__restrict__ a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// One launch for every per-call initialisation: the output rows and the hash table.
__global__ void mttkrp_init_kernel(double *__restrict__ out, int64_t n_out, int64_t T,
                                   unsigned long long *__restrict__ tkey, int32_t *__restrict__ tcnt,
                                   int32_t *__restrict__ trep, unsigned long long *__restrict__ twmin,
                                   unsigned long long *__restrict__ twmax, double *__restrict__ twsum) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_out; i += stride)
    out[i] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T; i += stride) {
    tkey[i] = ~0ull;
    tcnt[i] = 0;
    trep[i] = INT_MAX;
    twmin[i] = ~0ull;
    twmax[i] = 0ull;
    twsum[i] = 0.0;
  }
}

// ------------------------------------------------------------------------- dedup
// Samples with equal column keys are merged.  Their KRP rows are equal (H is a function
// of the index tuple); their weights are equal for sampler output (w depends on the
// tuple's probability only), in which case the merged weight is count * w^2 exactly.
// Unequal weights (e.g. an injected batch) fall back to the sum of w^2.
__global__ void hash_insert_kernel(const int64_t *__restrict__ X, int N, int64_t J, int k,
                                   Strides st, int64_t tmask, const double *__restrict__ w,
                                   unsigned long long *tkey, int32_t *tcnt, int32_t *trep,
                                   unsigned long long *twmin, unsigned long long *twmax,
                                   double *twsum) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  const int64_t key = sample_key(X, N, J, k, st, s);
  const double w2 = w[s] * w[s];
  const unsigned long long wb = (unsigned long long)__double_as_longlong(w2);  // w2 >= 0
  uint64_t h = mix64((uint64_t)key) & (uint64_t)tmask;
  while (true) {
    unsigned long long prev = atomicCAS(&tkey[h], ~0ull, (unsigned long long)key);
    if (prev == ~0ull || prev == (unsigned long long)key) {
      atomicAdd(&tcnt[h], 1);
      atomicMin(&trep[h], (int32_t)s);
      atomicMin(&twmin[h], wb);
      atomicMax(&twmax[h], wb);
      atomicAdd(&twsum[h], w2);
      return;
    }
    h = (h + 1) & (uint64_t)tmask;
  }
}

// ------------------------------------------------------------------------ lookup
__global__ void lookup_kernel(const int64_t *__restrict__ keys, int64_t n_cols,
                              const int64_t *__restrict__ colptr, const int64_t *dkey,
                              const int32_t *__restrict__ dcnt, const int32_t *__restrict__ drep,
                              const int64_t *__restrict__ S, const double *__restrict__ H,
                              const double *__restrict__ dsc, int R, int Rp,
                              int64_t *__restrict__ dlo,
                              int64_t *__restrict__ dlen, double *__restrict__ Hs,
                              int64_t *icnt /* aliases dkey */, int64_t *__restrict__ stats) {
  // persistent warps over the distinct fibers; the stats counters take one atomic per CTA
  __shared__ unsigned long long cnt_ne[8], cnt_m[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nS = S[0];
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long ne = 0, nm = 0;
  for (int64_t d = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; d < nS; d += nwarps) {
    int64_t lo = 0, len = 0;
    const int64_t key = dkey[d];
    const int64_t c = warp_lower_bound(keys, n_cols, key, lane);
    if (lane == 0) {
      if (c < n_cols && keys[c] == key) {
        lo = colptr[c];
        len = colptr[c + 1] - lo;
      }
      dlo[d] = lo;
      dlen[d] = len;
      icnt[d] = ceil_div(len, kItemE);   // traversal items of this fiber (aliases dkey[d])
      if (len > 0) {
        ne += 1;
        nm += (unsigned long long)(len * (int64_t)dcnt[d]);
      }
    }
    const int32_t rep = drep[d];
    const double sc = dsc[d];
    for (int q = lane; q < Rp; q += 32) Hs[d * Rp + q] = q < R ? sc * H[(int64_t)rep * R + q] : 0.0;
  }
  if (lane == 0) {
    cnt_ne[wid] = ne;
    cnt_m[wid] = nm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += cnt_ne[w];
      b += cnt_m[w];
    }
    if (a) atomicAdd((unsigned long long *)&stats[1], a);
    if (b) atomicAdd((unsigned long long *)&stats[3], b);
  }
}

// nnz[0] = gathered entries to process, nnz[1] = entries required.  A call whose entries
// exceed the workspace capacity processes nothing (S = 0 downstream, output stays zero)
// and raises RCP_ST_CAPACITY; the caller re-runs it with a larger workspace.
__global__ void finalize_counts_kernel(int64_t *__restrict__ S, const int64_t *__restrict__ doff,
                                       int64_t *__restrict__ nnz, int64_t *__restrict__ stats,
                                       int64_t cap, int *status) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t s = S[0];
    const int64_t t = doff[s];
    nnz[1] = t;
    if (t > cap) {
      nnz[0] = 0;
      S[0] = 0;
      raise_status(status, RCP_ST_CAPACITY);
      return;
    }
    nnz[0] = t;
    stats[0] += s;
    stats[2] += t;
  }
}

__global__ void rows_hit_kernel(const int64_t *__restrict__ rcnt, int64_t n_rows,
                                int64_t *__restrict__ stats) {
  int64_t c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x)
    c += rcnt[i] > 0 ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long *)&stats[4], (unsigned long long)c);
}

// ------------------------------------------------------------ entry traversal
// Work items: chunks of at most kItemE consecutive entries of one fiber.  A fiber's entries
// are contiguous in the store, so a warp reads an item's rows/values fully coalesced.
constexpr int kTraverseThreads = 1024;
constexpr int kInFlight = 8;   // entries per lane with loads in flight (latency hiding)

// item -> fiber table: fiber d owns items [ioff[d], ioff[d+1])
__global__ void item_fill_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                                 int32_t *__restrict__ ifib) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= Sp[0]) return;
  for (int64_t it = ioff[d]; it < ioff[d + 1]; ++it) ifib[it] = (int32_t)d;
}

struct ItemSpan {
  int64_t d, a, b;   // fiber, store range [a, b)
};

__device__ __forceinline__ ItemSpan item_span(int64_t it, const int64_t *__restrict__ ioff,
                                              const int32_t *__restrict__ ifib,
                                              const int64_t *__restrict__ dlo,
                                              const int64_t *__restrict__ dlen) {
  ItemSpan sp;
  sp.d = ifib[it];   // fiber of the item (table filled by item_fill_kernel)
  const int64_t c = it - ioff[sp.d];
  const int64_t base = dlo[sp.d];
  sp.a = base + c * kItemE;
  sp.b = min(base + dlen[sp.d], sp.a + kItemE);
  return sp;
}

__device__ __forceinline__ void cta_items(int64_t n_items, int64_t &i0, int64_t &i1) {
  const int64_t per = ceil_div(n_items, (int64_t)gridDim.x);
  i0 = (int64_t)blockIdx.x * per;
  i1 = min(i0 + per, n_items);
}

__global__ void __launch_bounds__(kTraverseThreads)
row_count_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                 const int32_t *__restrict__ ifib,
                 const int64_t *__restrict__ dlo, const int64_t *__restrict__ dlen,
                 const int32_t *__restrict__ rows, int64_t n_rows, int priv,
                 int64_t *__restrict__ rcnt) {
  extern __shared__ int32_t hist[];
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  if (i0 >= i1) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (priv) {
    for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  for (int64_t it = i0 + wid; it < i1; it += nw) {
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    for (int64_t pos = sp.a + lane; pos < sp.b; pos += 32) {
      const int32_t row = rows[pos];
      if (priv) atomicAdd(&hist[row], 1);
      else atomicAdd((unsigned long long *)&rcnt[row], 1ull);
    }
  }
  if (priv) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x)
      if (hist[i]) atomicAdd((unsigned long long *)&rcnt[i], (unsigned long long)hist[i]);
  }
}

__global__ void __launch_bounds__(kTraverseThreads)
scatter_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                 const int32_t *__restrict__ ifib,
               const int64_t *__restrict__ dlo, const int64_t *__restrict__ dlen,
               const int32_t *__restrict__ rows, const double *__restrict__ vals, int64_t n_rows,
               int priv, const int64_t *__restrict__ rptr, int64_t *__restrict__ rcur,
               double2 *__restrict__ ent, int64_t cap, int *status) {
  extern __shared__ int32_t hist[];
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  if (i0 >= i1) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (priv) {
    // pass A: CTA-local counts; reserve one contiguous run per (CTA, row)
    for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t it = i0 + wid; it < i1; it += nw) {
      const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
      for (int64_t pos = sp.a + lane; pos < sp.b; pos += 32) atomicAdd(&hist[rows[pos]], 1);
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) {
      const int32_t c = hist[i];
      if (c) hist[i] = (int32_t)atomicAdd((unsigned long long *)&rcur[i], (unsigned long long)c);
    }
    __syncthreads();
  }
  for (int64_t it = i0 + wid; it < i1; it += nw) {
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    for (int64_t pos = sp.a + lane; pos < sp.b; pos += 32) {
      const int32_t row = rows[pos];
      const double v = vals[pos];
      int64_t slot;
      if (priv) slot = atomicAdd(&hist[row], 1);
      else slot = (int64_t)atomicAdd((unsigned long long *)&rcur[row], 1ull);
      const int64_t o = rptr[row] + slot;
      if (o >= cap) {
        raise_status(status, RCP_ST_CAPACITY);
        continue;
      }
      ent[o] = make_double2(__longlong_as_double((long long)sp.d), v);
    }
  }
}

// Blocks with CTA-private histograms (rows fit in shared memory): no global atomics.
//  1. every CTA histograms the rows of its items into cmat[cta][row];
//  2. per row, an exclusive prefix over CTAs (in place) and the row totals;
//  3. after the row scan, CTA c writes its entries of row r at rptr[r] + cmat[c][r] + k.
__global__ void __launch_bounds__(kTraverseThreads)
cta_hist_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                 const int32_t *__restrict__ ifib,
                const int64_t *__restrict__ dlo, const int64_t *__restrict__ dlen,
                const int32_t *__restrict__ rows, int64_t n_rows, int32_t *__restrict__ cmat) {
  extern __shared__ int32_t hist[];
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  __shared__ int claim;
  for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) claim = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  while (true) {   // the CTA's items, claimed one at a time by its warps
    int c = 0;
    if (lane == 0) c = atomicAdd(&claim, 1);
    const int64_t it = i0 + __shfl_sync(0xffffffffu, c, 0);
    if (it >= i1) break;
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    for (int64_t pos = sp.a + lane; pos < sp.b; pos += 32 * kInFlight) {
      int32_t rw[kInFlight];
#pragma unroll
      for (int q = 0; q < kInFlight; ++q) rw[q] = pos + 32 * q < sp.b ? rows[pos + 32 * q] : -1;
#pragma unroll
      for (int q = 0; q < kInFlight; ++q)
        if (rw[q] >= 0) atomicAdd(&hist[rw[q]], 1);
    }
  }
  __syncthreads();
  int32_t *mine = cmat + (int64_t)blockIdx.x * n_rows;
  for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) mine[i] = hist[i];
}

// Per row, exclusive prefix over the G CTA counts (in place) and the row total.  Four
// threads per row each own a quarter of the CTAs (independent loads in flight), then the
// quarters are offset by their predecessors' sums.
constexpr int kPrefixSeg = 4;
constexpr int kPrefixRows = 64;    // rows per 256-thread block
constexpr int kPrefixMaxPer = 80;  // CTA counts one thread keeps in registers (G <= 320)
constexpr int kPrefixMaxPerFast = 48;   // the row-transpose path's grid (one CTA per SM)

template <int MP>
__global__ void __launch_bounds__(kPrefixRows * kPrefixSeg)
cta_prefix_kernel(int32_t *__restrict__ cmat, int G, int64_t n_rows, int64_t *__restrict__ rcnt) {
  __shared__ int32_t seg_sum[kPrefixSeg][kPrefixRows];
  const int rl = threadIdx.x % kPrefixRows, sg = threadIdx.x / kPrefixRows;
  const int64_t r = blockIdx.x * (int64_t)kPrefixRows + rl;
  const int per = (G + kPrefixSeg - 1) / kPrefixSeg;
  const int c0 = sg * per, c1 = min(G, c0 + per);
  int32_t v[MP];
  int32_t sum = 0;
#pragma unroll
  for (int q = 0; q < MP; ++q) {
    const int c = c0 + q;
    v[q] = (r < n_rows && c < c1) ? cmat[(int64_t)c * n_rows + r] : 0;
    sum += v[q];
  }
  seg_sum[sg][rl] = sum;
  __syncthreads();
  int32_t run = 0;
  for (int q = 0; q < sg; ++q) run += seg_sum[q][rl];
  if (r < n_rows) {
#pragma unroll
    for (int q = 0; q < MP; ++q) {
      const int c = c0 + q;
      if (c < c1) {
        cmat[(int64_t)c * n_rows + r] = run;
        run += v[q];
      }
    }
    if (sg == kPrefixSeg - 1) rcnt[r] = run;
  }
}

__device__ __forceinline__ void put_entry(double2 *__restrict__ ent, int64_t o, int64_t d, double v) {
  ent[o] = make_double2(__longlong_as_double((long long)d), v);
}

__global__ void __launch_bounds__(kTraverseThreads)
cta_scatter_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                   const int32_t *__restrict__ ifib,
                   const int64_t *__restrict__ dlo, const int64_t *__restrict__ dlen,
                   const int32_t *__restrict__ rows, const double *__restrict__ vals,
                   int64_t n_rows, const int64_t *__restrict__ rptr,
                   const int32_t *__restrict__ cmat, double2 *__restrict__ ent, int64_t cap,
                   int *status) {
  extern __shared__ int32_t cur[];   // absolute next slot per row (< 2^31)
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  const int32_t *mine = cmat + (int64_t)blockIdx.x * n_rows;
  __shared__ int claim;
  for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) cur[i] = (int32_t)(rptr[i] + mine[i]);
  if (threadIdx.x == 0) claim = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  while (true) {   // the CTA's items, claimed one at a time by its warps
    int c = 0;
    if (lane == 0) c = atomicAdd(&claim, 1);
    const int64_t it = i0 + __shfl_sync(0xffffffffu, c, 0);
    if (it >= i1) break;
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    for (int64_t pos = sp.a + lane; pos < sp.b; pos += 32 * kInFlight) {
      // issue every load of the batch before the dependent cursor atomics and stores
      int32_t rw[kInFlight];
      double v[kInFlight];
#pragma unroll
      for (int q = 0; q < kInFlight; ++q) {
        const bool ok = pos + 32 * q < sp.b;
        rw[q] = ok ? rows[pos + 32 * q] : -1;
        v[q] = ok ? vals[pos + 32 * q] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kInFlight; ++q) {
        if (rw[q] < 0) continue;
        const int64_t o = atomicAdd(&cur[rw[q]], 1);
        if (o < cap) put_entry(ent, o, sp.d, v[q]);
        else raise_status(status, RCP_ST_CAPACITY);
      }
    }
  }
}

// ------------------------------------------------------------ bucketed transpose
// The single-pass scatter above writes every entry to a random 16-B slot (each write fills
// a 32-B sector: half the DRAM traffic is wasted).  The bucketed variant moves the same
// entries in two near-sequential passes:
//  A. per CTA, entries of row bucket b (rows [b 2^sh, (b+1) 2^sh), <= 256 buckets) go to the
//     CTA's contiguous slice of the bucket's final range — ~256 write streams per CTA
//     instead of one per row — as {row, fiber, value};
//  B. one CTA per bucket orders its range by row in place of the final array (the range,
//     ~1/256 of the entries, stays L2-resident while its rows' cursors advance).
#ifndef RCP_BUCKET_MAX
#define RCP_BUCKET_MAX 512   // <= kBigBucketMax (bucket_scatter's shared cursors, bofs)
#endif
constexpr int kBucketMax = RCP_BUCKET_MAX;   // buckets of the small-row (CTA-histogram) path
constexpr int kBigBucketMax = 2048;    // buckets of the large-row path (<= 2^14 rows each)
constexpr int kBigMaxShift = 14;
#ifndef RCP_BUCKET_MIN_ROWS
#define RCP_BUCKET_MIN_ROWS 4096
#endif
constexpr int64_t kBucketMinRows = RCP_BUCKET_MIN_ROWS;   // below: the single-pass scatter is faster

// bofs[cta][b] = start of the CTA's slice of bucket b = rptr[b << sh] + sum over the
// bucket's rows of the CTA-exclusive prefix cmat[cta][row]
__global__ void bucket_offsets_kernel(const int32_t *__restrict__ cmat, int G, int64_t n_rows,
                                      int sh, int nb, const int64_t *__restrict__ rptr,
                                      int64_t *__restrict__ bofs) {
  // one warp per (CTA, bucket): lanes read the bucket's rows coalesced
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= (int64_t)G * nb) return;
  const int c = (int)(i / nb), b = (int)(i - (int64_t)c * nb);
  const int64_t r0 = (int64_t)b << sh, r1 = min(n_rows, r0 + ((int64_t)1 << sh));
  const int32_t *row = cmat + (int64_t)c * n_rows;
  long long acc = 0;
  for (int64_t r = r0 + lane; r < r1; r += 32) acc += row[r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) bofs[i] = rptr[r0] + acc;
}

__global__ void __launch_bounds__(kTraverseThreads)
bucket_scatter_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                      const int32_t *__restrict__ ifib, const int64_t *__restrict__ dlo,
                      const int64_t *__restrict__ dlen, const int32_t *__restrict__ rows,
                      const double *__restrict__ vals, int sh, int nb,
                      const int64_t *__restrict__ bofs, double2 *__restrict__ tmp, int64_t cap,
                      int *status) {
  __shared__ int bcur[kBigBucketMax];   // offsets relative to the CTA's slice base (< 2^31)
  __shared__ int64_t bbase[kBigBucketMax];
  __shared__ int claim;
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    bcur[b] = 0;
    bbase[b] = bofs[(int64_t)blockIdx.x * nb + b];
  }
  if (threadIdx.x == 0) claim = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  while (true) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&claim, 1);
    const int64_t it = i0 + __shfl_sync(0xffffffffu, c, 0);
    if (it >= i1) break;
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    for (int64_t pos0 = sp.a; pos0 < sp.b; pos0 += 32 * kInFlight) {
      int32_t rw[kInFlight];
      double v[kInFlight];
#pragma unroll
      for (int q = 0; q < kInFlight; ++q) {
        const int64_t pos = pos0 + 32 * q + lane;
        const bool ok = pos < sp.b;
        rw[q] = ok ? rows[pos] : -1;
        v[q] = ok ? vals[pos] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kInFlight; ++q) {
        if (pos0 + 32 * q >= sp.b) break;   // warp-uniform
        const bool ok = rw[q] >= 0;
        if (ok) {
          const int b = rw[q] >> sh;
          const int64_t o = bbase[b] + atomicAdd(&bcur[b], 1);
          if (o < cap)
            tmp[o] = make_double2(
                __longlong_as_double((long long)(((uint64_t)(uint32_t)rw[q] << 32) | (uint32_t)sp.d)),
                v[q]);
          else
            raise_status(status, RCP_ST_CAPACITY);
        }
      }
    }
  }
}

// One CTA per bucket: entries of [rptr[b << sh], rptr[(b+1) << sh]) ordered by row.
__global__ void __launch_bounds__(256)
bucket_rows_kernel(const double2 *__restrict__ tmp, int64_t n_rows, int sh,
                   const int64_t *__restrict__ rptr, double2 *__restrict__ ent) {
  extern __shared__ int64_t rbase[];   // per row of the bucket: row start, then int32 cursors
  const int b = blockIdx.x;
  const int64_t r0 = (int64_t)b << sh, r1 = min(n_rows, r0 + ((int64_t)1 << sh));
  const int nr = (int)(r1 - r0);
  int *rcur = reinterpret_cast<int *>(rbase + ((int64_t)1 << sh));
  for (int q = threadIdx.x; q < nr; q += blockDim.x) {
    rbase[q] = rptr[r0 + q];
    rcur[q] = 0;
  }
  __syncthreads();
  const int64_t e0 = rptr[r0], e1 = rptr[r1];
  constexpr int U = 8;   // entries in flight per thread
  for (int64_t base = e0; base < e1; base += (int64_t)blockDim.x * U) {
    double2 t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * blockDim.x + threadIdx.x;
      t[u] = e < e1 ? tmp[e] : make_double2(__longlong_as_double(-1LL), 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t key = (uint64_t)__double_as_longlong(t[u].x);
      if (key == ~0ull) continue;
      const int row = (int)(key >> 32);
      const int64_t o = rbase[row - r0] + atomicAdd(&rcur[row - r0], 1);
      ent[o] = make_double2(__longlong_as_double((long long)(uint32_t)(key & 0xffffffffu)), t[u].y);
    }
  }
}

// ------------------------------------------------------------ large-row transpose
// Row counts above the CTA-histogram limit (C4/C5 factor modes: 10^6..10^7 rows): no
// per-row global atomics.  Entries are bucketed by row >> sh (<= 2048 buckets of
// <= 2^14 rows): per-CTA bucket counts, per-bucket prefix over CTAs, pass A (the shared
// bucket_scatter_kernel) writes each CTA's entries to its slice of the bucket, and pass B
// counting-sorts each bucket by row in shared memory, emitting the row pointers.

__global__ void __launch_bounds__(kTraverseThreads)
big_hist_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                const int32_t *__restrict__ ifib, const int64_t *__restrict__ dlo,
                const int64_t *__restrict__ dlen, const int32_t *__restrict__ rows, int sh, int nb,
                int32_t *__restrict__ bmat) {
  __shared__ int cnt[kBigBucketMax];
  __shared__ int claim;
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
  if (threadIdx.x == 0) claim = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  while (true) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&claim, 1);
    const int64_t it = i0 + __shfl_sync(0xffffffffu, c, 0);
    if (it >= i1) break;
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    for (int64_t pos = sp.a + lane; pos < sp.b; pos += 32 * kInFlight) {
      int32_t rw[kInFlight];
#pragma unroll
      for (int q = 0; q < kInFlight; ++q) rw[q] = pos + 32 * q < sp.b ? rows[pos + 32 * q] : -1;
#pragma unroll
      for (int q = 0; q < kInFlight; ++q)
        if (rw[q] >= 0) atomicAdd(&cnt[rw[q] >> sh], 1);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) bmat[(int64_t)blockIdx.x * nb + b] = cnt[b];
}

// per bucket: exclusive prefix over the CTAs (in place) and the bucket total
__global__ void big_colprefix_kernel(int32_t *__restrict__ bmat, int G, int nb,
                                     int64_t *__restrict__ btot) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) {   // the scan below reads one element past the buckets
    btot[nb] = 0;
    return;
  }
  int64_t run = 0;
  for (int c = 0; c < G; ++c) {
    const int32_t v = bmat[(int64_t)c * nb + b];
    bmat[(int64_t)c * nb + b] = (int32_t)run;
    run += v;
  }
  btot[b] = run;
}

__global__ void big_offsets_kernel(const int32_t *__restrict__ bmat, const int64_t *__restrict__ bstart,
                                   int G, int nb, int64_t *__restrict__ bofs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)G * nb) return;
  bofs[i] = bstart[i % nb] + bmat[i];
}

constexpr int kBigRowsThreads = 1024;

// One CTA per bucket: row counts -> row pointers (and rows hit) -> entries in row order.
__global__ void __launch_bounds__(kBigRowsThreads)
big_rows_kernel(const double2 *__restrict__ tmp, int64_t n_rows, int sh,
                const int64_t *__restrict__ bstart, int64_t *__restrict__ rptr,
                double2 *__restrict__ ent, int64_t *__restrict__ stats) {
  extern __shared__ int cnt[];   // per row of the bucket
  __shared__ int wsum[32];
  __shared__ int hit_s;
  const int b = blockIdx.x;
  const int64_t r0 = (int64_t)b << sh;
  const int nr = (int)min((int64_t)1 << sh, n_rows - r0);
  const int64_t e0 = bstart[b], e1 = bstart[b + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < nr; q += blockDim.x) cnt[q] = 0;
  if (threadIdx.x == 0) hit_s = 0;
  __syncthreads();
  constexpr int U = 8;
  for (int64_t base = e0; base < e1; base += (int64_t)blockDim.x * U) {
    int rr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * blockDim.x + threadIdx.x;
      rr[u] = e < e1 ? (int)((uint64_t)__double_as_longlong(tmp[e].x) >> 32) - (int)r0 : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (rr[u] >= 0) atomicAdd(&cnt[rr[u]], 1);
  }
  __syncthreads();
  // exclusive scan of cnt[0, nr): each thread owns a contiguous run of rows
  const int per = (nr + blockDim.x - 1) / blockDim.x;
  const int q0 = min(nr, (int)threadIdx.x * per), q1 = min(nr, q0 + per);
  int mine = 0, hits = 0;
  for (int q = q0; q < q1; ++q) {
    mine += cnt[q];
    hits += cnt[q] > 0;
  }
  int x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
  if (lane == 0 && hits) atomicAdd(&hit_s, hits);
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int v = lane < nw ? wsum[lane] : 0;
    int z = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nw) wsum[lane] = z - v;
  }
  __syncthreads();
  int run = wsum[wid] + x - mine;
  for (int q = q0; q < q1; ++q) {
    const int c = cnt[q];
    cnt[q] = run;
    rptr[r0 + q] = e0 + run;
    run += c;
  }
  if (threadIdx.x == 0) {
    if (hit_s) atomicAdd((unsigned long long *)&stats[4], (unsigned long long)hit_s);
    if (r0 + nr == n_rows) rptr[n_rows] = e1;
  }
  __syncthreads();
  for (int64_t base = e0; base < e1; base += (int64_t)blockDim.x * U) {
    double2 t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * blockDim.x + threadIdx.x;
      t[u] = e < e1 ? tmp[e] : make_double2(__longlong_as_double(-1LL), 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t key = (uint64_t)__double_as_longlong(t[u].x);
      if (key == ~0ull) continue;
      const int row = (int)(key >> 32) - (int)r0;
      const int64_t o = e0 + atomicAdd(&cnt[row], 1);
      ent[o] = make_double2(__longlong_as_double((long long)(uint32_t)(key & 0xffffffffu)), t[u].y);
    }
  }
}

int big_shift(int64_t n_rows) {
  int sh = 0;
  while (ceil_div(n_rows, (int64_t)1 << sh) > kBigBucketMax) ++sh;
  return sh;
}

// ------------------------------------------------------------ segmented SpMM
// One warp per chunk of kSpmmChunk row-sorted entries; lanes own output columns.
// Entries come as separate column/value arrays (reference-shaped CSR, drop-in path); the
// fused path uses spmm_packed_kernel below.
struct CsrEntries {
  const int64_t *col;
  const double *val;
  const double *scale;
  __device__ __forceinline__ void get(int64_t x, int64_t &d, double &v) const {
    d = col[x];
    v = val[x];
    if (scale) v *= scale[d];
  }
};

template <int RPL, typename Acc>
__global__ void __launch_bounds__(256)
spmm_kernel(const int64_t *__restrict__ rptr, int64_t n_rows, const int64_t *__restrict__ nnzp,
            int64_t nnz_host, Acc acc_in, const double *__restrict__ Hs, int R,
            double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nnz = nnzp ? nnzp[0] : nnz_host;
  const int64_t nchunks = ceil_div(nnz, kSpmmChunk);
  for (int64_t ch = warp0; ch < nchunks; ch += nwarps) {
    const int64_t c0 = ch * kSpmmChunk;
    const int64_t c1 = min(c0 + kSpmmChunk, nnz);
    int64_t row = floor_index(rptr, n_rows + 1, c0);
    int64_t e = c0;
    while (e < c1) {
      const int64_t rs = rptr[row], re = rptr[row + 1];
      const int64_t stop = min(re, c1);
      if (stop > e) {
        double acc[RPL];
#pragma unroll
        for (int j = 0; j < RPL; ++j) acc[j] = 0.0;
        int64_t x = e;
        for (; x + 4 <= stop; x += 4) {
          int64_t d0, d1, d2, d3;
          double v0, v1, v2, v3;
          acc_in.get(x, d0, v0);
          acc_in.get(x + 1, d1, v1);
          acc_in.get(x + 2, d2, v2);
          acc_in.get(x + 3, d3, v3);
#pragma unroll
          for (int j = 0; j < RPL; ++j) {
            const int c = lane + 32 * j;
            if (c < R) {
              const double h0 = Hs[d0 * R + c], h1 = Hs[d1 * R + c];
              const double h2 = Hs[d2 * R + c], h3 = Hs[d3 * R + c];
              acc[j] = fma(v0, h0, acc[j]);
              acc[j] = fma(v1, h1, acc[j]);
              acc[j] = fma(v2, h2, acc[j]);
              acc[j] = fma(v3, h3, acc[j]);
            }
          }
        }
        for (; x < stop; ++x) {
          int64_t d0;
          double v0;
          acc_in.get(x, d0, v0);
#pragma unroll
          for (int j = 0; j < RPL; ++j) {
            const int c = lane + 32 * j;
            if (c < R) acc[j] = fma(v0, Hs[d0 * R + c], acc[j]);
          }
        }
        const bool whole = (rs >= c0) && (re <= c1);
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int c = lane + 32 * j;
          if (c < R) {
            if (whole) out[row * R + c] = acc[j];
            else atomicAdd(&out[row * R + c], acc[j]);
          }
        }
        e = stop;
      }
      ++row;
    }
  }
}

// Fused-path variant: packed entries, Hs rows at the padded stride, each lane owns a
// column pair loaded as one double2 (one load instruction per entry for R <= 64).  The
// warp loads 32 entries at once (one per lane) and broadcasts them with shuffles: a
// broadcast load would cost the L1 as many register-writeback cycles as an Hs row
// (measured: writeback was the limiter at ~75% busy).
template <int NP, bool DET = false>
__global__ void __launch_bounds__(256)
spmm_packed_kernel(const int64_t *__restrict__ rptr, int64_t n_rows, const int64_t *__restrict__ nnzp,
                   const double2 *__restrict__ ent, const double *__restrict__ Hs, int R,
                   double *__restrict__ out, double2 *__restrict__ slotF = nullptr,
                   double2 *__restrict__ slotL = nullptr) {
  const int lane = threadIdx.x & 31;
  const int Rp = hs_stride(R);
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nnz = nnzp[0];
  const int64_t nchunks = ceil_div(nnz, kSpmmChunk);
  const double2 *H2 = reinterpret_cast<const double2 *>(Hs);
  const int Rp2 = Rp >> 1;
  for (int64_t ch = warp0; ch < nchunks; ch += nwarps) {
    const int64_t c0 = ch * kSpmmChunk;
    const int64_t c1 = min(c0 + kSpmmChunk, nnz);
    int64_t row = floor_index(rptr, n_rows + 1, c0);   // (top levels stay in L1)
    int64_t rs = rptr[row], re = rptr[row + 1];
    double2 acc[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[j] = make_double2(0.0, 0.0);
    auto flush = [&]() {
      if (re > rs) {
        const bool whole = (rs >= c0) && (re <= c1);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const int c = 2 * (lane + 32 * j);
          if (c < R) {
            double *o = out + row * R + c;
            if (whole) {
              o[0] = acc[j].x;
              if (c + 1 < R) o[1] = acc[j].y;
            } else if (DET) {   // a split row: this chunk's partial, combined in chunk order
              (rs < c0 ? slotF : slotL)[ch * (32 * NP) + lane + 32 * j] = acc[j];
            } else {
              atomicAdd(o, acc[j].x);
              if (c + 1 < R) atomicAdd(o + 1, acc[j].y);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[j] = make_double2(0.0, 0.0);
    };
    for (int64_t base = c0; base < c1; base += 32) {
      const int nb = (int)min((int64_t)32, c1 - base);
      double2 mine = make_double2(0.0, 0.0);
      if (lane < nb) mine = ent[base + lane];
      const int md = (int)(int32_t)__double_as_longlong(mine.x);
      const double mv = mine.y;
      int q = 0;
      while (q < nb) {
        while (base + q >= re) {   // next non-finished row (warp-uniform)
          flush();
          ++row;
          rs = re;
          re = rptr[row + 1];
        }
        const int run = (int)min((int64_t)(nb - q), re - (base + q));   // entries of this row here
        int t = 0;
        for (; t + kSpmmU <= run; t += kSpmmU) {
          int dq[kSpmmU];
          double vq[kSpmmU];
#pragma unroll
          for (int u = 0; u < kSpmmU; ++u) {
            dq[u] = __shfl_sync(0xffffffffu, md, q + t + u);
            vq[u] = __shfl_sync(0xffffffffu, mv, q + t + u);
          }
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            const int c2 = lane + 32 * j;
            if (2 * c2 < R) {
              double2 h[kSpmmU];
#pragma unroll
              for (int u = 0; u < kSpmmU; ++u) h[u] = H2[(int64_t)dq[u] * Rp2 + c2];
#pragma unroll
              for (int u = 0; u < kSpmmU; ++u) {
                acc[j].x = fma(vq[u], h[u].x, acc[j].x);
                acc[j].y = fma(vq[u], h[u].y, acc[j].y);
              }
            }
          }
        }
        for (; t < run; ++t) {
          const int d = __shfl_sync(0xffffffffu, md, q + t);
          const double v = __shfl_sync(0xffffffffu, mv, q + t);
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            const int c2 = lane + 32 * j;
            if (2 * c2 < R) {
              const double2 h = H2[(int64_t)d * Rp2 + c2];
              acc[j].x = fma(v, h.x, acc[j].x);
              acc[j].y = fma(v, h.y, acc[j].y);
            }
          }
        }
        q += run;
      }
    }
    // the row holding the chunk's last entry
    flush();
  }
}

// Grouped variant (the product path): the warp's lanes form 4 groups of 8; group g takes
// the entries e = g (mod 4) of a row and its 8 lanes split each Hs row (column pairs
// li + 8k, k < NL).  A row's entries are loaded 32 at a time (lane 8g + t holds entry
// 4t + g of the batch, the next batch prefetched) and one shuffle per word hands each
// group its own entry, so a shuffle serves 4 entries: the L1's register writeback, which
// limits spmm_packed_kernel (3 shuffles = 384 B per entry beside the 400-byte Hs row at
// R = 50), carries ~112 B per entry here.  The 4 groups' partial row sums are combined by
// a 2-step butterfly when the row (or the chunk's part of it) ends; outputs and the
// deterministic mode's split-row slots keep spmm_packed_kernel's layout (column pair c2
// of chunk ch at ch * 32 NP + c2).
#ifndef RCP_SPMM_GMIN
#define RCP_SPMM_GMIN 4   // spmm_group_kernel: minimum resident CTAs per SM (64 registers; swept 1/3/4/5)
#endif
template <int NL, bool DET = false>
__global__ void __launch_bounds__(256, NL <= 4 ? RCP_SPMM_GMIN : 2)
spmm_group_kernel(const int64_t *__restrict__ rptr, int64_t n_rows, const int64_t *__restrict__ nnzp,
                  const double2 *__restrict__ ent, const double *__restrict__ Hs, int R,
                  double *__restrict__ out, double2 *__restrict__ slotF = nullptr,
                  double2 *__restrict__ slotL = nullptr) {
  constexpr int NP = NL <= 4 ? 1 : 2;   // slot stride of the deterministic mode (32 NP pairs)
  constexpr int U = NL <= 2 ? 4 : (NL <= 4 ? RCP_SPMM_GU : RCP_SPMM_GU5);   // steps in flight
  const int lane = threadIdx.x & 31, g = lane >> 3, li = lane & 7;
  const int R2 = (R + 1) >> 1;
  const int Rp2 = hs_stride(R) >> 1;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nnz = nnzp[0];
  const int64_t nchunks = ceil_div(nnz, kSpmmChunk);
  const double2 *H2 = reinterpret_cast<const double2 *>(Hs);
  const int mine_off = g + 4 * li;   // this lane's entry within a batch of 32
  for (int64_t ch = warp0; ch < nchunks; ch += nwarps) {
    const int64_t c0 = ch * kSpmmChunk;
    const int64_t c1 = min(c0 + kSpmmChunk, nnz);
    int64_t row = floor_index(rptr, n_rows + 1, c0);
    int64_t rs = rptr[row], re = rptr[row + 1];
    while (true) {
      const int64_t e0 = max(rs, c0), e1 = min(re, c1);
      if (e1 > e0) {
        double2 acc[NL];
#pragma unroll
        for (int k = 0; k < NL; ++k) acc[k] = make_double2(0.0, 0.0);
        double2 nxt = e0 + mine_off < e1 ? ent[e0 + mine_off] : make_double2(0.0, 0.0);
        for (int64_t base = e0; base < e1; base += 32) {
          const double2 cur = nxt;
          if (base + 32 < e1)
            nxt = base + 32 + mine_off < e1 ? ent[base + 32 + mine_off] : make_double2(0.0, 0.0);
          const int md = (int)(int32_t)__double_as_longlong(cur.x);
          const double mv = cur.y;
          const int nsteps = (int)min((int64_t)8, (e1 - base + 3) >> 2);   // warp-uniform
          for (int t0 = 0; t0 < nsteps; t0 += U) {
            int64_t d[U];
            double v[U];
            bool ok[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int src = (lane & 24) | (t0 + u);
              d[u] = __shfl_sync(0xffffffffu, md, src);
              v[u] = __shfl_sync(0xffffffffu, mv, src);
              ok[u] = base + g + 4 * (t0 + u) < e1;
            }
            double2 h[U][NL];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int k = 0; k < NL; ++k) {
                const int c2 = li + 8 * k;
                h[u][k] = (ok[u] && c2 < R2) ? H2[d[u] * Rp2 + c2] : make_double2(0.0, 0.0);
              }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int k = 0; k < NL; ++k) {
                acc[k].x = fma(v[u], h[u][k].x, acc[k].x);
                acc[k].y = fma(v[u], h[u][k].y, acc[k].y);
              }
          }
        }
#pragma unroll
        for (int k = 0; k < NL; ++k) {
          acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 8);
          acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 8);
          acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 16);
          acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 16);
        }
        const bool whole = (rs >= c0) && (re <= c1);
#pragma unroll
        for (int k = 0; k < NL; ++k) {
          const int c2 = li + 8 * k;
          if ((k & 3) != g || c2 >= R2) continue;   // the 4 groups share the stores
          if (whole) {
            double *o = out + row * R + 2 * c2;
            o[0] = acc[k].x;
            if (2 * c2 + 1 < R) o[1] = acc[k].y;
          } else if (DET) {
            (rs < c0 ? slotF : slotL)[ch * (32 * NP) + c2] = acc[k];
          } else {
            double *o = out + row * R + 2 * c2;
            atomicAdd(o, acc[k].x);
            if (2 * c2 + 1 < R) atomicAdd(o + 1, acc[k].y);
          }
        }
      }
      if (re >= c1) break;
      ++row;
      rs = re;
      re = rptr[row + 1];
    }
  }
}

// Segmented reduction of the packed row-sorted entries (rptr over n_rows, entry count at
// nnzp on the device); slotF/slotL: the deterministic mode's split-row partials.
template <bool DET>
void launch_spmm_packed(unsigned blocks, const int64_t *rptr, int64_t n_rows, const int64_t *nnzp,
                        const double2 *ent, const double *Hs, int R, double *out, double2 *slotF,
                        double2 *slotL, cudaStream_t st) {
#if RCP_SPMM_GROUP
  switch ((R + 15) / 16) {
#define RCP_SG(K)                                                                            \
  case K:                                                                                    \
    spmm_group_kernel<K, DET><<<blocks, 256, 0, st>>>(rptr, n_rows, nnzp, ent, Hs, R, out,   \
                                                      slotF, slotL);                         \
    break;
    RCP_SG(1) RCP_SG(2) RCP_SG(3) RCP_SG(4) RCP_SG(5) RCP_SG(6) RCP_SG(7)
    default: RCP_SG(8)
#undef RCP_SG
  }
#else
  if (R <= 64)
    spmm_packed_kernel<1, DET><<<blocks, 256, 0, st>>>(rptr, n_rows, nnzp, ent, Hs, R, out, slotF, slotL);
  else
    spmm_packed_kernel<2, DET><<<blocks, 256, 0, st>>>(rptr, n_rows, nnzp, ent, Hs, R, out, slotF, slotL);
#endif
}

template <typename Acc>
int launch_spmm(const int64_t *rptr, int64_t n_rows, const int64_t *nnzp, int64_t nnz_host,
                Acc acc, const double *Hs, int R, double *out, cudaStream_t st) {
  int64_t chunks_host = nnzp ? -1 : ceil_div(nnz_host, kSpmmChunk);
  int64_t blocks = 8LL * sm_count();
  if (chunks_host >= 0) {
    int64_t need = ceil_div(chunks_host, 8);
    if (need < blocks) blocks = need;
    if (blocks < 1) return RCP_OK;
  }
  switch ((R + 31) / 32) {
    case 1: spmm_kernel<1, Acc><<<(unsigned)blocks, 256, 0, st>>>(rptr, n_rows, nnzp, nnz_host, acc, Hs, R, out); break;
    case 2: spmm_kernel<2, Acc><<<(unsigned)blocks, 256, 0, st>>>(rptr, n_rows, nnzp, nnz_host, acc, Hs, R, out); break;
    case 3: spmm_kernel<3, Acc><<<(unsigned)blocks, 256, 0, st>>>(rptr, n_rows, nnzp, nnz_host, acc, Hs, R, out); break;
    default: spmm_kernel<4, Acc><<<(unsigned)blocks, 256, 0, st>>>(rptr, n_rows, nnzp, nnz_host, acc, Hs, R, out); break;
  }
  RCP_LAUNCH_CHECK("spmm");
  return RCP_OK;
}

// ------------------------------------------------------------ drop-in CSR helpers
__global__ void fiber_lookup_kernel(const int64_t *__restrict__ keys, int64_t n_cols,
                                    const int64_t *__restrict__ colptr,
                                    const int64_t *__restrict__ X, int N, int64_t J, int k,
                                    Strides st, int64_t *__restrict__ lo,
                                    int64_t *__restrict__ cnt) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  const int64_t key = sample_key(X, N, J, k, st, s);
  const int64_t c = lower_bound_i64(keys, n_cols, key);
  int64_t a = 0, b = 0;
  if (c < n_cols && keys[c] == key) {
    a = colptr[c];
    b = colptr[c + 1];
  }
  lo[s] = a;
  cnt[s] = b - a;
}

__global__ void fiber_expand_kernel(const int64_t *__restrict__ lo, const int64_t *__restrict__ off,
                                    int64_t J, const int32_t *__restrict__ rows,
                                    const double *__restrict__ vals, int64_t *__restrict__ ro,
                                    int64_t *__restrict__ co, double *__restrict__ vo) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= J) return;
  const int64_t a = lo[s], o = off[s], len = off[s + 1] - off[s];
  for (int64_t t = lane; t < len; t += 32) {
    ro[o + t] = rows[a + t];
    co[o + t] = s;
    vo[o + t] = vals[a + t];
  }
}

#include "mttkrp_tiles.cuh"

// radix sort temporary storage (double-buffer mode) for up to n pairs keyed by tile
size_t sort_tmp_bytes(int64_t n) {
  size_t b = 0;
  const int nn = (int)(n < (1LL << 31) - 1 ? n : (1LL << 31) - 1);
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint64_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, b, k, v, nn > 0 ? nn : 1);
  return b + 256;
}

size_t wsort_tmp_bytes(int64_t J) {
  size_t b = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr), v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, b, k, v, (int)(J > 0 ? J : 1));
  return b + 256;
}

// ------------------------------------------------------------ workspace layout
struct Ws {
  size_t off[64];
  int n = 0;
  size_t total = 0;
  size_t add(size_t bytes) {
    size_t o = (total + 255) & ~(size_t)255;
    total = o + bytes;
    off[n++] = o;
    return o;
  }
};

struct MttkrpLayout {
  int64_t T;
  size_t o_tkey, o_tcnt, o_trep, o_twmin, o_twmax, o_twsum, o_dsc, o_bcnt, o_dkey, o_dcnt,
      o_drep, o_dlo, o_dlen, o_doff, o_ioff, o_ifib, o_Hs, o_scan, o_rcnt, o_rptr, o_cmat,
      o_ent, o_tmp, o_bofs, o_S,
      o_nnz, o_flag, o_fpos, o_sslot, o_icnt, o_ipos,
      o_t64, o_sort, o_np, o_wk, o_wv, o_wk2, o_wv2, o_wst, o_wsort, o_slots, o_slots2;
  size_t total;
  MttkrpLayout(int64_t J, int64_t cap, int64_t n_rows, int R) {
    T = 1024;
    while (T < 2 * J) T <<= 1;
    Ws w;
    o_tkey = w.add(sizeof(int64_t) * T);
    o_tcnt = w.add(sizeof(int32_t) * T);
    o_trep = w.add(sizeof(int32_t) * T);
    o_twmin = w.add(sizeof(int64_t) * T);
    o_twmax = w.add(sizeof(int64_t) * T);
    o_twsum = w.add(sizeof(double) * T);
    o_dsc = w.add(sizeof(double) * (J + 1));
    o_bcnt = w.add(sizeof(int64_t) * (T / 1024));
    o_dkey = w.add(sizeof(int64_t) * (J + 1));
    o_dcnt = w.add(sizeof(int32_t) * (J + 1));
    o_drep = w.add(sizeof(int32_t) * (J + 1));
    o_dlo = w.add(sizeof(int64_t) * (J + 1));
    o_dlen = w.add(sizeof(int64_t) * (J + 1));
    o_doff = w.add(sizeof(int64_t) * (J + 2));
    o_ioff = w.add(sizeof(int64_t) * (J + 2));
    o_ifib = w.add(sizeof(int32_t) * (J + cap / kItemE + 2));     // items <= S + nnz / kItemE
    o_Hs = w.add(sizeof(double) * (size_t)(J + 1) * hs_stride(R));
    int64_t sc = J + 1 > n_rows + 1 ? J + 1 : n_rows + 1;
    if (J + cap / kItemE + 2 > sc) sc = J + cap / kItemE + 2;   // per-item pair offsets
    o_scan = w.add(scan_ws_bytes(sc));
    o_rcnt = w.add(sizeof(int64_t) * (n_rows + 1));
    o_rptr = w.add(sizeof(int64_t) * (n_rows + 2));
    o_cmat = w.add(sizeof(int32_t) * (size_t)sm_count() *
                   (size_t)(n_rows < kPrivRows ? n_rows : kPrivRows));
    o_ent = w.add(sizeof(double2) * (cap + 1));
    o_tmp = w.add(sizeof(double2) * (cap + 1));
    o_bofs = w.add(sizeof(int64_t) * ((size_t)sm_count() + 1) * (kBigBucketMax + 1));
    o_S = w.add(sizeof(int64_t) * 4);
    o_nnz = w.add(sizeof(int64_t) * 4);
    o_flag = w.add(sizeof(int64_t) * (J + 1));
    o_fpos = w.add(sizeof(int64_t) * (J + 2));
    o_sslot = w.add(sizeof(int32_t) * (J + 1));
    // deterministic mode: per-item pair counts and offsets (many row tiles), per-tile int64
    // arrays (tile pointers, entry counts and offsets, chunk counts and offsets), the radix
    // sort's temporary storage and the pair count
    const int64_t nitems = J + cap / kItemE + 2;
    o_icnt = w.add(sizeof(int64_t) * nitems);
    o_ipos = w.add(sizeof(int64_t) * (nitems + 1));
    const int64_t nt = n_rows / 8 + 4;
    o_t64 = w.add(sizeof(int64_t) * 5 * nt);
    o_sort = w.add(sort_tmp_bytes(cap));
    o_np = w.add(sizeof(int64_t) * 2);
    // deterministic mode: samples sorted by distinct fiber for ordered weight sums
    o_wk = w.add(sizeof(uint32_t) * (J + 1));
    o_wv = w.add(sizeof(uint32_t) * (J + 1));
    o_wk2 = w.add(sizeof(uint32_t) * (J + 1));
    o_wv2 = w.add(sizeof(uint32_t) * (J + 1));
    o_wst = w.add(sizeof(int32_t) * (J + 1));
    o_wsort = w.add(wsort_tmp_bytes(J));
    // deterministic mode: the SpMM's per-chunk partials of rows split across chunks
    o_slots2 = w.add(sizeof(double2) * 2 * (size_t)(cap / kSpmmChunk + 2) * 32 * (R <= 64 ? 1 : 2));
    // per (32-pair chunk, tile row) entry counts, then slots: chunks <= cap / 32 + tiles
    o_slots = w.add(sizeof(int64_t) * (size_t)(cap / 32 + n_rows / 8 + 2) * 16);
    total = w.total + 256;
  }
};

}  // namespace

extern "C" {

int rcp_set_mttkrp_mode(int mode) {
  const int prev = mttkrp_mode();
  if (mode >= 0) g_mttkrp_mode = mode ? 1 : 0;
  return prev;
}

size_t rcp_mttkrp_ws_bytes(int64_t J, int64_t store_nnz, int64_t n_rows, int R) {
  MttkrpLayout L(J, store_nnz, n_rows, R);
  return L.total;
}

// Entry capacity implied by a workspace size (the layout is monotone in it).
static int64_t mttkrp_cap(int64_t J, int64_t n_rows, int R, size_t ws_bytes) {
  MttkrpLayout base(J, 0, n_rows, R);
  if (ws_bytes < base.total) return -1;
  // largest cap whose layout fits (alignment padding makes the size a step function)
  int64_t lo = 0, hi = (int64_t)((ws_bytes - base.total) / sizeof(double2)) + 64;
  while (hi - lo > 1) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (MttkrpLayout(J, mid, n_rows, R).total <= ws_bytes) lo = mid; else hi = mid;
  }
  return lo;
}

int rcp_mttkrp_layout(int64_t J, int64_t n_rows, int R, size_t ws_bytes, int64_t *h_out) {
  if (!h_out) return RCP_ERR_ARG;
  int64_t cap = mttkrp_cap(J, n_rows, R, ws_bytes);
  if (cap < 0) return RCP_ERR_ARG;
  MttkrpLayout L(J, cap, n_rows, R);
  const size_t o[] = {L.o_dkey, L.o_dcnt, L.o_drep, L.o_dlo, L.o_dlen, L.o_doff, L.o_Hs,
                      L.o_rcnt, L.o_rptr, L.o_ent, L.o_cmat, L.o_S, L.o_nnz};
  for (int i = 0; i < 13; ++i) h_out[i] = (int64_t)o[i];
  h_out[13] = cap;
  return RCP_OK;
}

int rcp_sampled_mttkrp(const int64_t *d_keys, const int64_t *d_colptr, int64_t n_cols,
                       const int32_t *d_rows, const double *d_vals, int64_t n_rows,
                       const int64_t *d_X, int N, int64_t J, int k, const int64_t *h_strides,
                       const double *d_H, const double *d_w, int R, double *d_out,
                       int64_t *d_stats, void *d_ws, size_t ws_bytes, int *d_status,
                       void *stream) {
  if (N < 2 || N > kMaxModes || k < 0 || k >= N || R < 1 || R > RCP_MAX_RANK || J < 0 ||
      J >= (1LL << 26) || n_rows < 0 || n_rows >= (1LL << 31) || n_cols < 0 || !h_strides ||
      !d_stats)
    return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (J == 0 || n_rows == 0 || n_cols == 0) {
    if (n_rows > 0) RCP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double) * n_rows * R, st));
    return RCP_OK;
  }
  if (!d_keys || !d_colptr || !d_rows || !d_vals || !d_X || !d_H || !d_w || !d_out || !d_ws)
    return RCP_ERR_ARG;
  // the capacity of the entry arrays is implied by ws_bytes
  const int64_t cap = mttkrp_cap(J, n_rows, R, ws_bytes);
  if (cap < 0) return RCP_ERR_ARG;
  MttkrpLayout L(J, cap, n_rows, R);
  char *w = (char *)d_ws;
  auto P = [&](size_t o) { return (void *)(w + o); };
  unsigned long long *tkey = (unsigned long long *)P(L.o_tkey);
  int32_t *tcnt = (int32_t *)P(L.o_tcnt), *trep = (int32_t *)P(L.o_trep);
  int64_t *bcnt = (int64_t *)P(L.o_bcnt);
  int64_t *dkey = (int64_t *)P(L.o_dkey);
  int32_t *dcnt = (int32_t *)P(L.o_dcnt), *drep = (int32_t *)P(L.o_drep);
  int64_t *dlo = (int64_t *)P(L.o_dlo), *dlen = (int64_t *)P(L.o_dlen), *doff = (int64_t *)P(L.o_doff);
  double *Hs = (double *)P(L.o_Hs);
  void *scan_ws = P(L.o_scan);
  int64_t *rcnt = (int64_t *)P(L.o_rcnt), *rptr = (int64_t *)P(L.o_rptr);
  double2 *ent = (double2 *)P(L.o_ent);
  int64_t *S = (int64_t *)P(L.o_S), *nnz = (int64_t *)P(L.o_nnz);

  Strides sd;
  for (int m = 0; m < kMaxModes; ++m) sd.s[m] = m < N ? h_strides[m] : 0;

  // 1. dedup
  // The row-tile path (row tiles fit one scan, < 2^22 samples) writes every output row
  // itself; the row-transpose path (large row counts, or RCP_MTTKRP_PATH=rows) zeroes first.
  const int force_rows = mttkrp_mode() == 1 ? 0 : 1;
  const int tile_np = R <= 64 ? 1 : 2;
  const int tile_ts = tile_np == 1 ? 4 : 3;
  const int64_t n_tiles = ceil_div(n_rows, (int64_t)1 << tile_ts);
  bool tiles = !force_rows && n_tiles <= kTileMaxTiles && J < (1LL << 22) &&
               cap < (1LL << 31) && 2 * sm_count() <= kPrefixSeg * kPrefixMaxPer;
  // many row tiles: sorted pairs (reads the pair count on the host, so not inside a graph)
  bool tiles_big = false;
  if (!force_rows && !tiles && J < (1LL << 22) && cap < (1LL << 31)) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    RCP_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
    tiles_big = cs == cudaStreamCaptureStatusNone;
  }
  if (tiles_big) tiles = false;

  unsigned long long *twmin = (unsigned long long *)P(L.o_twmin);
  unsigned long long *twmax = (unsigned long long *)P(L.o_twmax);
  double *twsum = (double *)P(L.o_twsum), *dsc = (double *)P(L.o_dsc);
  mttkrp_init_kernel<<<4 * sm_count(), 256, 0, st>>>(d_out, n_rows * (int64_t)R, L.T, tkey,
                                                      tcnt, trep, twmin, twmax, twsum);
  RCP_LAUNCH_CHECK("mttkrp_init");
  hash_insert_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(
      d_X, N, J, k, sd, L.T - 1, d_w, tkey, tcnt, trep, twmin, twmax, twsum);
  RCP_LAUNCH_CHECK("hash_insert");
  {   // distinct fibers numbered in representative-sample order (deterministic)
    int64_t *flag = (int64_t *)P(L.o_flag), *fpos = (int64_t *)P(L.o_fpos);
    int32_t *sslot = (int32_t *)P(L.o_sslot);
    rep_flag_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(d_X, N, J, k, sd, L.T - 1, tkey, trep,
                                                                flag, sslot);
    RCP_LAUNCH_CHECK("rep_flag");
    int rc0 = scan_i64_exclusive(flag, fpos, J, nullptr, P(L.o_scan), st);
    if (rc0) return rc0;
    rep_compact_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(flag, fpos, J, sslot, tkey, tcnt, twmin,
                                                                   twmax, twsum, dkey, dcnt, drep, dsc, S);
    RCP_LAUNCH_CHECK("rep_compact");
    if (tiles || tiles_big) {   // unequal weights of one fiber: their w^2 summed in sample order
      uint32_t *wk = (uint32_t *)P(L.o_wk), *wv = (uint32_t *)P(L.o_wv);
      uint32_t *wk2 = (uint32_t *)P(L.o_wk2), *wv2 = (uint32_t *)P(L.o_wv2);
      int32_t *wst = (int32_t *)P(L.o_wst);
      sample_fiber_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(sslot, trep, fpos, J, wk, wv);
      RCP_LAUNCH_CHECK("sample_fiber");
      cub::DoubleBuffer<uint32_t> kb(wk, wk2), vb(wv, wv2);
      int bits = 1;
      while (bits < 31 && ((int64_t)1 << bits) < J) ++bits;
      size_t tb = wsort_tmp_bytes(J);
      RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(P(L.o_wsort), tb, kb, vb, (int)J, 0, bits, st));
      fiber_start_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(kb.Current(), J, wst);
      RCP_LAUNCH_CHECK("fiber_start");
      ordered_w2_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(S, wst, dcnt, vb.Current(), d_w, drep,
                                                                    sslot, twmin, twmax, dsc);
      RCP_LAUNCH_CHECK("ordered_w2");
    }
  }
  // 2. lookup + scaled KRP rows
  lookup_kernel<<<(unsigned)std::min<int64_t>(ceil_div(J * 32, 256), 8LL * sm_count()), 256, 0, st>>>(
      d_keys, n_cols, d_colptr, dkey, dcnt, drep, S, d_H, dsc, R, hs_stride(R), dlo, dlen, Hs,
      dkey, d_stats);
  RCP_LAUNCH_CHECK("lookup");
  // 3. fiber offsets
  int rc = scan_i64_exclusive(dlen, doff, J, S, scan_ws, st);
  if (rc) return rc;
  finalize_counts_kernel<<<1, 32, 0, st>>>(S, doff, nnz, d_stats, cap, d_status);
  RCP_LAUNCH_CHECK("finalize_counts");
  // 3b. work items: fiber chunks of <= kItemE entries (dkey reused for the counts)
  int64_t *icnt = dkey;
  int64_t *ioff = (int64_t *)P(L.o_ioff);
  rc = scan_i64_exclusive(icnt, ioff, J, S, scan_ws, st);
  if (rc) return rc;
  int32_t *ifib = (int32_t *)P(L.o_ifib);
  item_fill_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, st>>>(ioff, S, ifib);
  RCP_LAUNCH_CHECK("item_fill");
  // deterministic mode, after the pairs: row-sorted entries per tile (stable), then the
  // segmented SpMM with split rows combined in chunk order
  auto det_csr = [&](const uint64_t *pairs_, const int64_t *tptr_, int64_t nt_, double2 *ent_) -> int {
    int64_t *t64_ = (int64_t *)P(L.o_t64);
    int64_t *te = t64_ + (nt_ + 2), *eoff = t64_ + 2 * (nt_ + 2);
    const unsigned gw = (unsigned)(8 * sm_count());
    tile_entries_kernel<<<gw, 256, 0, st>>>(tptr_, nt_, pairs_, te);
    RCP_LAUNCH_CHECK("tile_entries");
    int rcx = scan_i64_exclusive(te, eoff, nt_, nullptr, scan_ws, st);
    if (rcx) return rcx;
    // 32-pair chunks per tile: per-chunk row counts -> stable slots -> entries
    int64_t *nchk = t64_ + 3 * (nt_ + 2), *choff = nchk + (nt_ + 2);
    tile_chunks_kernel<<<(unsigned)ceil_div(nt_, 256), 256, 0, st>>>(tptr_, nt_, nchk);
    RCP_LAUNCH_CHECK("tile_chunks");
    rcx = scan_i64_exclusive(nchk, choff, nt_, nullptr, scan_ws, st);
    if (rcx) return rcx;
    int64_t *cc = (int64_t *)P(L.o_slots);   // <= pairs / 32 + n_tiles chunks x TR rows
    if (tile_ts == 4) {
      chunk_rows_kernel<4><<<gw, 256, 0, st>>>(tptr_, choff, nt_, pairs_, d_rows, cc);
      tile_rowscan_kernel<4><<<gw, 256, 0, st>>>(choff, nt_, n_rows, eoff, cc, rptr, d_stats);
      chunk_write_kernel<4><<<gw, 256, 0, st>>>(tptr_, choff, nt_, pairs_, d_rows, d_vals, cc, ent_);
    } else {
      chunk_rows_kernel<3><<<gw, 256, 0, st>>>(tptr_, choff, nt_, pairs_, d_rows, cc);
      tile_rowscan_kernel<3><<<gw, 256, 0, st>>>(choff, nt_, n_rows, eoff, cc, rptr, d_stats);
      chunk_write_kernel<3><<<gw, 256, 0, st>>>(tptr_, choff, nt_, pairs_, d_rows, d_vals, cc, ent_);
    }
    RCP_LAUNCH_CHECK("tile_expand");
    double2 *slotF = (double2 *)P(L.o_slots2);
    double2 *slotL = slotF + (size_t)(cap / kSpmmChunk + 2) * 32 * tile_np;
    const unsigned sb2 = (unsigned)(RCP_SPMM_BLOCKS_PER_SM * sm_count());
    const int64_t *nnzp = eoff + nt_;
    launch_spmm_packed<true>(sb2, rptr, n_rows, nnzp, ent_, Hs, R, d_out, slotF, slotL, st);
    RCP_LAUNCH_CHECK("spmm_det");
    if (tile_np == 1) spmm_fix_kernel<1><<<gw, 256, 0, st>>>(rptr, n_rows, slotF, slotL, R, d_out);
    else spmm_fix_kernel<2><<<gw, 256, 0, st>>>(rptr, n_rows, slotF, slotL, R, d_out);
    RCP_LAUNCH_CHECK("spmm_fix");
    return RCP_OK;
  };
  if (tiles) {
    const int grid = 2 * sm_count();                    // pair passes: 2 CTAs per SM
    const int nt = (int)n_tiles;
    int32_t *cmat = (int32_t *)P(L.o_cmat);            // grid x n_tiles
    int64_t *tcntp = rcnt;                              // pairs per tile
    int64_t *tptr = (int64_t *)P(L.o_t64);              // tile pointers (n_tiles + 1)
    uint64_t *pairs = (uint64_t *)P(L.o_tmp);           // <= entries <= cap pairs
    static bool tattr = false;
    if (!tattr) {
      const int scat = (int)pair_scatter_smem(kTileMaxTiles);
      RCP_CUDA_TRY(cudaFuncSetAttribute(pair_scatter_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, scat));
      RCP_CUDA_TRY(cudaFuncSetAttribute(pair_scatter_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, scat));
      tattr = true;
    }
    const size_t hsm = sizeof(int32_t) * nt;
    if (tile_ts == 4) tile_hist_kernel<4><<<grid, kPairThreads, hsm, st>>>(ioff, S, ifib, dlo, dlen, d_rows, nt, cmat);
    else tile_hist_kernel<3><<<grid, kPairThreads, hsm, st>>>(ioff, S, ifib, dlo, dlen, d_rows, nt, cmat);
    RCP_LAUNCH_CHECK("tile_hist");
    cta_prefix_kernel<kPrefixMaxPer><<<(unsigned)ceil_div(nt, kPrefixRows), kPrefixRows * kPrefixSeg, 0, st>>>(
        cmat, grid, nt, tcntp);
    RCP_LAUNCH_CHECK("cta_prefix");
    rc = scan_i64_exclusive(tcntp, tptr, nt, nullptr, scan_ws, st);
    if (rc) return rc;
    const size_t ssm = pair_scatter_smem(nt);
    if (tile_ts == 4) pair_scatter_kernel<4><<<grid, kPairThreads, ssm, st>>>(ioff, S, ifib, dlo, dlen, d_rows, nt, tptr, cmat, pairs);
    else pair_scatter_kernel<3><<<grid, kPairThreads, ssm, st>>>(ioff, S, ifib, dlo, dlen, d_rows, nt, tptr, cmat, pairs);
    RCP_LAUNCH_CHECK("pair_scatter");
    rc = det_csr(pairs, tptr, nt, ent);
    if (rc) return rc;
    return RCP_OK;
  }
  if (tiles_big) {
    const int64_t nt = n_tiles;
    uint32_t *kA = (uint32_t *)((char *)P(L.o_ent) + sizeof(uint64_t) * (size_t)cap);
    uint64_t *vA = (uint64_t *)P(L.o_ent);
    uint32_t *kB = (uint32_t *)((char *)P(L.o_tmp) + sizeof(uint64_t) * (size_t)cap);
    uint64_t *vB = (uint64_t *)P(L.o_tmp);
    int64_t *icnt2 = (int64_t *)P(L.o_icnt), *ipos = (int64_t *)P(L.o_ipos);
    int64_t *np = (int64_t *)P(L.o_np);
    int64_t *tptr = (int64_t *)P(L.o_t64);   // tile pointers (n_tiles + 1)
    const int ts = tile_ts;
    const unsigned gw = (unsigned)(8 * sm_count());
    if (ts == 4) pair_count_kernel<4><<<gw, 256, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, icnt2, np + 1);
    else pair_count_kernel<3><<<gw, 256, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, icnt2, np + 1);
    RCP_LAUNCH_CHECK("pair_count");
    rc = scan_i64_exclusive(icnt2, ipos, J + cap / kItemE + 1, np + 1, scan_ws, st);
    if (rc) return rc;
    if (ts == 4) pair_emit_kernel<4><<<gw, 256, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, ipos, kA, vA);
    else pair_emit_kernel<3><<<gw, 256, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, ipos, kA, vA);
    RCP_LAUNCH_CHECK("pair_emit");
    // the pair count: ipos[n_items]
    int64_t h_nit = 0, h_np = 0;
    RCP_CUDA_TRY(cudaMemcpyAsync(&h_nit, np + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RCP_CUDA_TRY(cudaStreamSynchronize(st));
    RCP_CUDA_TRY(cudaMemcpyAsync(&h_np, ipos + h_nit, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RCP_CUDA_TRY(cudaStreamSynchronize(st));
    RCP_CUDA_TRY(cudaMemcpyAsync(np, &h_np, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    cub::DoubleBuffer<uint32_t> kb(kA, kB);
    cub::DoubleBuffer<uint64_t> vb(vA, vB);
    int bits = 1;
    while (bits < 32 && ((int64_t)1 << bits) < nt) ++bits;
    size_t tb = sort_tmp_bytes(cap);
    if (h_np > 0)
      RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(P(L.o_sort), tb, kb, vb, (int)h_np, 0, bits, st));
    const uint32_t *tk = kb.Current();
    const uint64_t *pairs = vb.Current();
    double2 *entries = (double2 *)(vb.Current() == vA ? (void *)vB : (void *)vA);
    tile_bounds_kernel<<<(unsigned)ceil_div(nt + 1, 256), 256, 0, st>>>(tk, np, nt, tptr);
    RCP_LAUNCH_CHECK("tile_bounds");
    rc = det_csr(pairs, tptr, nt, entries);
    if (rc) return rc;
    return RCP_OK;
  }
  // 4. row histogram -> row pointers; 5. scatter into row order (packed entries)
  const int priv =
      (n_rows <= kPrivRows && cap < (1LL << 31) && sm_count() <= kPrefixSeg * kPrefixMaxPerFast) ? 1 : 0;
  static bool attr = false;
  if (!attr) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(cta_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RCP_CUDA_TRY(cudaFuncSetAttribute(cta_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const int grid = sm_count();
  if (priv) {
    int32_t *cmat = (int32_t *)P(L.o_cmat);
    const size_t smem = sizeof(int32_t) * n_rows;
    cta_hist_kernel<<<grid, kTraverseThreads, smem, st>>>(ioff, S, ifib, dlo, dlen, d_rows, n_rows, cmat);
    RCP_LAUNCH_CHECK("cta_hist");
    cta_prefix_kernel<kPrefixMaxPerFast><<<(unsigned)ceil_div(n_rows, kPrefixRows), kPrefixRows * kPrefixSeg, 0, st>>>(
        cmat, grid, n_rows, rcnt);
    RCP_LAUNCH_CHECK("cta_prefix");
    rc = scan_i64_exclusive(rcnt, rptr, n_rows, nullptr, scan_ws, st);
    if (rc) return rc;
    if (n_rows < kBucketMinRows) {   // few rows: their segments are long, scatter directly
      cta_scatter_kernel<<<grid, kTraverseThreads, smem, st>>>(ioff, S, ifib, dlo, dlen, d_rows,
                                                               d_vals, n_rows, rptr, cmat, ent, cap,
                                                               d_status);
      RCP_LAUNCH_CHECK("cta_scatter");
    } else {
    // bucketed transpose (two near-sequential passes)
    int sh = 0;
    while ((ceil_div(n_rows, (int64_t)1 << sh)) > kBucketMax) ++sh;
    const int nb = (int)ceil_div(n_rows, (int64_t)1 << sh);
    int64_t *bofs = (int64_t *)P(L.o_bofs);
    double2 *tmp = (double2 *)P(L.o_tmp);
    bucket_offsets_kernel<<<(unsigned)ceil_div((int64_t)grid * nb * 32, 256), 256, 0, st>>>(
        cmat, grid, n_rows, sh, nb, rptr, bofs);
    RCP_LAUNCH_CHECK("bucket_offsets");
    bucket_scatter_kernel<<<grid, kTraverseThreads, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, d_vals,
                                                             sh, nb, bofs, tmp, cap, d_status);
    RCP_LAUNCH_CHECK("bucket_scatter");
    bucket_rows_kernel<<<nb, 256, (sizeof(int64_t) + sizeof(int)) * ((size_t)1 << sh), st>>>(
        tmp, n_rows, sh, rptr, ent);
    RCP_LAUNCH_CHECK("bucket_rows");
    }
  } else if (big_shift(n_rows) <= kBigMaxShift && cap < (1LL << 40)) {
    // large-row bucketed transpose (no per-row global atomics)
    const int sh = big_shift(n_rows);
    const int nb = (int)ceil_div(n_rows, (int64_t)1 << sh);
    int32_t *bmat = (int32_t *)P(L.o_cmat);            // grid x nb <= grid x kPrivRows
    int64_t *bofs = (int64_t *)P(L.o_bofs);            // grid x nb, then btot, bstart
    int64_t *btot = bofs + (int64_t)grid * nb;
    int64_t *bstart = btot + (nb + 1);
    double2 *tmp = (double2 *)P(L.o_tmp);
    big_hist_kernel<<<grid, kTraverseThreads, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, sh, nb, bmat);
    RCP_LAUNCH_CHECK("big_hist");
    big_colprefix_kernel<<<(unsigned)ceil_div(nb + 1, 256), 256, 0, st>>>(bmat, grid, nb, btot);
    RCP_LAUNCH_CHECK("big_colprefix");
    rc = scan_i64_exclusive(btot, bstart, nb, nullptr, scan_ws, st);
    if (rc) return rc;
    big_offsets_kernel<<<(unsigned)ceil_div((int64_t)grid * nb, 256), 256, 0, st>>>(bmat, bstart, grid,
                                                                                    nb, bofs);
    RCP_LAUNCH_CHECK("big_offsets");
    bucket_scatter_kernel<<<grid, kTraverseThreads, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, d_vals,
                                                             sh, nb, bofs, tmp, cap, d_status);
    RCP_LAUNCH_CHECK("bucket_scatter");
    static bool battr = false;
    if (!battr) {
      RCP_CUDA_TRY(cudaFuncSetAttribute(big_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(sizeof(int) << kBigMaxShift)));
      battr = true;
    }
    big_rows_kernel<<<nb, kBigRowsThreads, sizeof(int) << sh, st>>>(tmp, n_rows, sh, bstart, rptr, ent,
                                                                   d_stats);
    RCP_LAUNCH_CHECK("big_rows");
  } else {
    RCP_CUDA_TRY(cudaMemsetAsync(rcnt, 0, sizeof(int64_t) * (n_rows + 1), st));
    row_count_kernel<<<grid, kTraverseThreads, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, n_rows, 0, rcnt);
    RCP_LAUNCH_CHECK("row_count");
    rc = scan_i64_exclusive(rcnt, rptr, n_rows, nullptr, scan_ws, st);
    if (rc) return rc;
    {
      int64_t b = ceil_div(n_rows, 256);
      if (b > 4LL * sm_count()) b = 4LL * sm_count();
      rows_hit_kernel<<<(unsigned)b, 256, 0, st>>>(rcnt, n_rows, d_stats);
      RCP_LAUNCH_CHECK("rows_hit");
    }
    RCP_CUDA_TRY(cudaMemsetAsync(rcnt, 0, sizeof(int64_t) * (n_rows + 1), st));
    scatter_kernel<<<grid, kTraverseThreads, 0, st>>>(ioff, S, ifib, dlo, dlen, d_rows, d_vals, n_rows, 0,
                                                      rptr, rcnt, ent, cap, d_status);
    RCP_LAUNCH_CHECK("scatter");
  }
  if (priv) {
    int64_t b = ceil_div(n_rows, 256);
    if (b > 4LL * sm_count()) b = 4LL * sm_count();
    rows_hit_kernel<<<(unsigned)b, 256, 0, st>>>(rcnt, n_rows, d_stats);
    RCP_LAUNCH_CHECK("rows_hit");
  }
  // 6. segmented reduction
  const unsigned sb = (unsigned)(RCP_SPMM_BLOCKS_PER_SM * sm_count());
  launch_spmm_packed<false>(sb, rptr, n_rows, nnz, ent, Hs, R, d_out, nullptr, nullptr, st);
  RCP_LAUNCH_CHECK("spmm_packed");
  return RCP_OK;
}

int rcp_fiber_lookup(const int64_t *d_keys, int64_t n_cols, const int64_t *d_colptr,
                     const int64_t *d_X, int N, int64_t J, int k, const int64_t *h_strides,
                     int64_t *d_lo, int64_t *d_counts, void *stream) {
  if (N < 2 || N > kMaxModes || k < 0 || k >= N || J < 0 || !h_strides) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (!d_X || !d_lo || !d_counts || (n_cols > 0 && (!d_keys || !d_colptr))) return RCP_ERR_ARG;
  Strides sd;
  for (int m = 0; m < kMaxModes; ++m) sd.s[m] = m < N ? h_strides[m] : 0;
  fiber_lookup_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_keys, n_cols, d_colptr, d_X, N, J, k, sd, d_lo, d_counts);
  RCP_LAUNCH_CHECK("fiber_lookup");
  return RCP_OK;
}

int rcp_fiber_expand(const int64_t *d_lo, const int64_t *d_off, int64_t J, const int32_t *d_rows,
                     const double *d_vals, int64_t *d_row_out, int64_t *d_col_out,
                     double *d_val_out, void *stream) {
  if (J < 0) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (!d_lo || !d_off || !d_row_out || !d_col_out || !d_val_out) return RCP_ERR_ARG;
  fiber_expand_kernel<<<(unsigned)ceil_div(J * 32, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_lo, d_off, J, d_rows, d_vals, d_row_out, d_col_out, d_val_out);
  RCP_LAUNCH_CHECK("fiber_expand");
  return RCP_OK;
}

int rcp_csr_spmm(const int64_t *d_row_ptr, int64_t n_rows, const int64_t *d_col,
                 const double *d_val, const double *d_H, const double *d_scale, int R,
                 double *d_out, void *stream) {
  if (n_rows < 0 || R < 1 || R > RCP_MAX_RANK || !d_row_ptr) return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (n_rows == 0) return RCP_OK;
  RCP_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double) * n_rows * R, st));
  int64_t nnz = 0;
  RCP_CUDA_TRY(cudaMemcpyAsync(&nnz, d_row_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RCP_CUDA_TRY(cudaStreamSynchronize(st));
  if (nnz == 0) return RCP_OK;
  CsrEntries acc{d_col, d_val, d_scale};
  return launch_spmm<CsrEntries>(d_row_ptr, n_rows, nullptr, nnz, acc, d_H, R, d_out, st);
}

}  // extern "C"
