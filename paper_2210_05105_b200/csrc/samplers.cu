// Leverage-score samplers on the device.
//  * CP-ARLS-LEV (ref samplers.py:104-191): per-row leverage u G+ u^T, ordered mass,
//    normalised cdf, inverse-CDF draws on Philox LOCAL_DRAW streams, SHUFFLE fold.
//  * STS-CP (ref samplers.py:194-468): a complete binary tree of packed node Grams over
//    leaf blocks of consecutive rows; one warp walks one sample, evaluating the two child
//    masses h^T (G (.) M) h per level as a dot product of the node Gram with the
//    sample's precomputed packed P = (h h^T) (.) M, then an inverse-CDF over the leaf's
//    rows.  In exact arithmetic this is the reference's inverse CDF of r over rows in
//    global order (the reference itself is leaf-size and rank-count invariant).
#include <float.h>

#include <stdlib.h>

#include "common.cuh"
#include "gram_mma.cuh"
#include "scan.cuh"

using namespace rcp;

namespace {

int sm_count() {
  static int s = 0;
  if (!s) {
    s = rcp_device_sms();
    if (!s) s = 148;
  }
  return s;
}

// ------------------------------------------------------------------ ARLS leverage
// Row leverages on the fp64 tensor cores (every R <= RCP_MAX_RANK).  A warp takes 8-row tiles Z of U
// (staged in shared memory), forms Y = Z G+ with mma.m8n8k4 (G+ zero-padded to Rn x Rn in
// shared memory) and d_q = <Y_q, Z_q>.  Tiles are assigned to warps in a fixed order, so
// the per-CTA partial masses (and the ordered total) are reproducible.
constexpr int kLevMmaMaxR = 128;
static_assert(kLevMmaMaxR >= RCP_MAX_RANK, "leverage scores run on the tensor cores for every rank");
__host__ __device__ __forceinline__ int lev_rn(int R) { return (R + 7) & ~7; }
// Row stride of the staged U tile and of G+ in shared memory: Rn + 4 (4 or 12 mod 16
// doubles) makes the mma fragment reads conflict-free.
__host__ __device__ __forceinline__ int lev_zs(int R) { return lev_rn(R) + 4; }

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

#ifndef RCP_LEV_MINB
#define RCP_LEV_MINB 1   // __launch_bounds__ min blocks of leverage_mma_kernel
#endif
template <int KS>   // k-steps = Rn / 4
__global__ void __launch_bounds__(256, RCP_LEV_MINB)
leverage_mma_kernel(const double *__restrict__ U, int64_t n, int R, const double *__restrict__ Gp,
                    double *__restrict__ lev, double *__restrict__ part, int nbuf) {
  extern __shared__ double sh[];
  constexpr int Rn = KS * 4;
  const int Zs = lev_zs(R);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *G = sh;                                          // Rn x Zs
  double *zbase = sh + Rn * Zs + (size_t)wid * nbuf * 8 * Zs;   // this warp's nbuf tiles
  for (int e = threadIdx.x; e < Rn * Zs; e += blockDim.x) {
    const int a = e / Zs, b = e - a * Zs;
    // u'Gu over the 8x8 blocks at or above the diagonal only: the blocks above it carry 2 G
    // (G symmetric: a pseudo-inverse or the walk's conditioning matrix), the ones below are
    // never read
    G[e] = (a < R && b < R) ? ((a >> 3) < (b >> 3) ? 2.0 * Gp[a * R + b] : Gp[a * R + b]) : 0.0;
  }
  for (int c = lane; c < nbuf * 8 * Zs; c += 32) zbase[c] = 0.0;   // padding columns stay 0
  __syncthreads();
  const int row = lane >> 2, quad = lane & 3;
  double local = 0.0;
  const int64_t tiles = (n + 7) >> 3;
  const int64_t stride = (int64_t)gridDim.x * nw, t0 = (int64_t)blockIdx.x * nw + wid;
  // nbuf-stage cp.async pipeline: the tiles nbuf - 1 ahead load while this one computes
  auto stage = [&](int64_t tl, int slot) {
    if (tl < tiles)
      stage_tile8(zbase + slot * 8 * Zs, U, tl << 3, (int)min((int64_t)8, n - (tl << 3)), R, Zs,
                  lane);
    cpa_commit();
  };
  for (int s = 0; s < nbuf - 1; ++s) stage(t0 + s * stride, s);
  int slot = 0;
  for (int64_t tl = t0; tl < tiles; tl += stride) {
    stage(tl + (nbuf - 1) * stride, slot == 0 ? nbuf - 1 : slot - 1);
    cpa_wait_stages(nbuf);
    __syncwarp();
    const int64_t r0 = tl << 3;
    const int nb = (int)min((int64_t)8, n - r0);
    const double *zr = zbase + slot * 8 * Zs + row * Zs;
    double a[KS];   // A fragments of the tile, reused by every n-tile
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[ks] = zr[ks * 4 + quad];
    double msum = 0.0;
    // two n-tiles at a time: two independent accumulator chains per warp (the mma of one
    // chain issues while the other's result is in flight)
#pragma unroll
    for (int nt = 0; nt < Rn; nt += 16) {
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {   // (conditions resolved at compile time: unrolled)
        if (ks * 4 < nt + 8) dmma_8x8x4(c0, c1, a[ks], G[(ks * 4 + quad) * Zs + nt + row]);
        if (nt + 8 < Rn && ks * 4 < nt + 16)
          dmma_8x8x4(d0, d1, a[ks], G[(ks * 4 + quad) * Zs + nt + 8 + row]);
      }
      msum = fma(c0, zr[nt + 2 * quad], msum);
      msum = fma(c1, zr[nt + 2 * quad + 1], msum);
      if (nt + 8 < Rn) {
        msum = fma(d0, zr[nt + 8 + 2 * quad], msum);
        msum = fma(d1, zr[nt + 8 + 2 * quad + 1], msum);
      }
    }
    msum += __shfl_xor_sync(0xffffffffu, msum, 1);
    msum += __shfl_xor_sync(0xffffffffu, msum, 2);
    const double d = msum > 0.0 ? msum : 0.0;
    if (quad == 0 && row < nb) lev[r0 + row] = d;
    // fixed-order warp partial: rows of the tile in order
    double t = (quad == 0 && row < nb) ? d : 0.0;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    local += t;
    __syncwarp();   // every lane is done with this slot before it is refilled
    slot = slot + 1 == nbuf ? 0 : slot + 1;
  }
  cpa_wait<0>();
  __syncthreads();
  if (lane == 0) sh[wid] = local;   // reuse (G no longer needed)
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += sh[w];
    part[blockIdx.x] = s;
  }
}

// Ordered (deterministic) sum of the per-CTA partial masses; one block of 256 threads.
__global__ void mass_kernel(const double *__restrict__ part, int nparts, double *mass) {
  __shared__ double red[256];
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) s += part[p];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) mass[0] = red[0];
}

__global__ void normalize_kernel(double *__restrict__ dist, int64_t n, const double *mass) {
  const double C = mass[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (C > 0.0) dist[i] = dist[i] / C;
}

__global__ void cdf_div_kernel(double *__restrict__ cdf, int64_t n) {
  const double last = cdf[n - 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cdf[i] = cdf[i] / last;
}

__global__ void arls_draw_kernel(const double *__restrict__ cdf, const double *__restrict__ dist,
                                 int64_t n, int64_t row_lo, double ratio, const double *tmass,
                                 uint64_t k0, uint64_t k1, const uint64_t *__restrict__ dkey,
                                 int64_t q, int64_t offset,
                                 int64_t *__restrict__ rows, double *__restrict__ prob,
                                 const double *__restrict__ U, int R, double *__restrict__ urow,
                                 int *status, int zero_flag) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= q) return;
  if (dkey) {   // stream key resident on the device (graph-replayed rounds)
    k0 = dkey[0];
    k1 = dkey[1];
  }
  if (tmass && !(tmass[0] > 0.0)) {
    if (t == 0) raise_status(status, zero_flag);
    rows[offset + t] = row_lo;
    prob[offset + t] = 0.0;
    return;
  }
  const double u = u64_to_unit(philox_word(k0, k1, (uint64_t)t));
  // searchsorted(cdf, u, side='right'): number of entries <= u
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
  }
  if (lo > n - 1) lo = n - 1;
  rows[offset + t] = row_lo + lo;
  prob[offset + t] = ratio * dist[lo];
  if (urow)
    for (int c = 0; c < R; ++c) urow[(offset + t) * R + c] = U[lo * R + c];
}

__global__ void batch_fold_kernel(const int64_t *__restrict__ perm, const int64_t *__restrict__ rows,
                                  const double *__restrict__ prob, int64_t J,
                                  const double *__restrict__ U, int64_t u_lo,
                                  const double *__restrict__ urows, int R, int first,
                                  int64_t *__restrict__ Xi, double *__restrict__ pmp,
                                  double *__restrict__ H) {
  // one warp per sample: coalesced H row update
  const int lane = threadIdx.x & 31;
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= J) return;
  const int64_t t = perm ? perm[s] : s;
  const int64_t x = rows[t];
  if (lane == 0) {
    Xi[s] = x;
    pmp[s] = prob[t];
  }
  const double *src = urows ? urows + t * R : U + (x - u_lo) * R;
  for (int c = lane; c < R; c += 32) H[s * R + c] = first ? src[c] : H[s * R + c] * src[c];
}

// --------------------------------------------------------------------- STS build
int getenv_leaf_ffma() {   // RCP_LEAF_FFMA=1: the FFMA leaf Grams for every R > 64 (A/B)
  const char *e = getenv("RCP_LEAF_FFMA");
  return e && e[0] == '1' ? 1 : 0;
}

int getenv_leaf_split() {   // RCP_LEAF_SPLIT=1: not the staged leaf Grams (A/B)
  const char *e = getenv("RCP_LEAF_SPLIT");
  return e && e[0] == '1' ? 1 : 0;
}

__global__ void sts_leaf_kernel(const double *__restrict__ U, int64_t n, int R, int leaf,
                                int64_t nleaves, double *__restrict__ level) {
  extern __shared__ double rows[];  // leaf x R, then the packed (a, b) table
  const int Rt = R * (R + 1) / 2;
  const int Rs = tri_stride(R);
  uint16_t *ab = reinterpret_cast<uint16_t *>(rows + (size_t)leaf * R);
  for (int a = threadIdx.x; a < R; a += blockDim.x) {   // row a of the packed triangle
    const int e0 = a * R - (a * (a - 1)) / 2;
    for (int b = a; b < R; ++b) ab[e0 + b - a] = (uint16_t)(a | (b << 8));
  }
  for (int64_t v = blockIdx.x; v < nleaves; v += gridDim.x) {
    const int64_t r0 = v * leaf;
    const int nr = (int)min((int64_t)leaf, n - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * R; e += blockDim.x) rows[e] = U[r0 * R + e];
    __syncthreads();
    double *out = level + v * Rs;
    if (Rs > Rt && threadIdx.x == 0) out[Rt] = 0.0;
    for (int e = threadIdx.x; e < Rt; e += blockDim.x) {
      const int a = ab[e] & 0xff, b = ab[e] >> 8;
      double s = 0.0;
      for (int q = 0; q < nr; ++q) s = fma(rows[q * R + a], rows[q * R + b], s);
      out[e] = s;
    }
  }
}

// R <= 64: leaf Grams on the fp64 tensor cores, one warp per leaf (gram_mma.cuh), written
// as the packed upper triangle.
// CTAs per SM (register cap): swept 1/2/3 with tools/lab/dense_lab.py at 4.8M rows —
// R = 50 (T = 7): 3.35 / 2.62 / 4.04 ms per tree build; R = 25 (T = 4): 0.82 / 0.74 / 0.60.
template <int T>
__global__ void __launch_bounds__(256, (T <= 4 ? 3 : 2))
sts_leaf_mma_kernel(const double *__restrict__ U, int64_t n, int R, int leaf, int64_t nleaves,
                    double *__restrict__ level) {
  extern __shared__ double sh[];   // one packed node per warp
  constexpr int NP = T * (T + 1) / 2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int Rt = R * (R + 1) / 2, Rs = tri_stride(R);
  const int kk = lane & 3, col = lane >> 2;
  for (int64_t v = (int64_t)blockIdx.x * nw + wid; v < nleaves; v += (int64_t)gridDim.x * nw) {
    const int64_t r0 = v * leaf, rend = min(r0 + leaf, n);
    double acc[NP][2];
#pragma unroll
    for (int p = 0; p < NP; ++p) acc[p][0] = acc[p][1] = 0.0;
    for (int k0 = 0; k0 < leaf; k0 += 16) {   // 4 row steps' loads in flight at once
      double f[4][T];
#pragma unroll
      for (int g = 0; g < 4; ++g) gram_load<T>(U, nullptr, r0 + k0 + 4 * g + kk, rend, R, col, f[g]);
#pragma unroll
      for (int g = 0; g < 4; ++g)
        if (k0 + 4 * g < leaf) gram_accum<T>(f[g], acc);
    }
    // packed triangle staged in shared memory, then written with coalesced stores
    double *stage = sh + (size_t)wid * Rs;
    int p = 0;
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
      for (int b = a; b < T; ++b) {
        const int ga = 8 * a + col;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int gb = 8 * b + 2 * kk + u;
          if (ga <= gb && gb < R) stage[tri_index(ga, gb, R)] = acc[p][u];
        }
        ++p;
      }
    if (Rs > Rt && lane == 0) stage[Rt] = 0.0;
    __syncwarp();
    double *out = level + v * Rs;
    for (int e = lane; e < Rs; e += 32) out[e] = stage[e];
    __syncwarp();
  }
}

// 64 < R <= 128: leaf Grams on the fp64 tensor cores with the tile pairs split over G warps
// per leaf (gram_accum_group); the CTA's 8 warps serve 8 / G leaves at a time, each leaf's
// warps meeting at their own named barrier before the packed triangle is written.
template <int T, int G, int g>
__device__ __forceinline__ void leaf_split_body(const double *__restrict__ U, int64_t r0, int64_t rend,
                                                int R, int leaf, double *stage) {
  constexpr int NP = T * (T + 1) / 2;
  constexpr int PPG = (NP + G - 1) / G;
  const int lane = threadIdx.x & 31, kk = lane & 3, col = lane >> 2;
  double acc[PPG][2];
#pragma unroll
  for (int p = 0; p < PPG; ++p) acc[p][0] = acc[p][1] = 0.0;
  for (int k0 = 0; k0 < leaf; k0 += 8) {   // two row steps' loads in flight
    double f0[T], f1[T];
    gram_load<T>(U, nullptr, r0 + k0 + kk, rend, R, col, f0);
    gram_load<T>(U, nullptr, r0 + k0 + 4 + kk, rend, R, col, f1);
    gram_accum_group<T, G, g>(f0, acc);
    if (k0 + 4 < leaf) gram_accum_group<T, G, g>(f1, acc);
  }
  int p = 0;
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int b = a; b < T; ++b) {
      if (p >= g * PPG && p < (g + 1) * PPG) {
        const int ga = 8 * a + col;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int gb = 8 * b + 2 * kk + u;
          if (ga <= gb && gb < R) stage[tri_index(ga, gb, R)] = acc[p - g * PPG][u];
        }
      }
      ++p;
    }
}

template <int T, int G>
__global__ void __launch_bounds__(256, 1)
sts_leaf_split_kernel(const double *__restrict__ U, int64_t n, int R, int leaf, int64_t nleaves,
                      double *__restrict__ level) {
  extern __shared__ double sh[];   // one packed node per leaf slot
  constexpr int SLOTS = 8 / G;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int grp = wid % G, slot = wid / G;
  const int Rt = R * (R + 1) / 2, Rs = tri_stride(R);
  double *stage = sh + (size_t)slot * Rs;
  for (int64_t v = (int64_t)blockIdx.x * SLOTS + slot; v < nleaves; v += (int64_t)gridDim.x * SLOTS) {
    const int64_t r0 = v * leaf, rend = min(r0 + leaf, n);
    switch (grp) {
      case 0: leaf_split_body<T, G, 0>(U, r0, rend, R, leaf, stage); break;
      case 1: leaf_split_body<T, G, (G > 1 ? 1 : 0)>(U, r0, rend, R, leaf, stage); break;
      case 2: leaf_split_body<T, G, (G > 2 ? 2 : 0)>(U, r0, rend, R, leaf, stage); break;
      case 3: leaf_split_body<T, G, (G > 3 ? 3 : 0)>(U, r0, rend, R, leaf, stage); break;
      case 4: leaf_split_body<T, G, (G > 4 ? 4 : 0)>(U, r0, rend, R, leaf, stage); break;
      case 5: leaf_split_body<T, G, (G > 5 ? 5 : 0)>(U, r0, rend, R, leaf, stage); break;
      case 6: leaf_split_body<T, G, (G > 6 ? 6 : 0)>(U, r0, rend, R, leaf, stage); break;
      default: leaf_split_body<T, G, (G > 7 ? 7 : 0)>(U, r0, rend, R, leaf, stage); break;
    }
    if (Rs > Rt && grp == 0 && lane == 0) stage[Rt] = 0.0;
    // the leaf's G warps (named barrier 1 + slot), then its packed triangle out
    asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * G) : "memory");
    double *out = level + v * Rs;
    for (int e = grp * 32 + lane; e < Rs; e += 32 * G) out[e] = stage[e];
    asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * G) : "memory");
  }
}

// 64 < R <= 128, leaves of 32 or 64 rows: the staged form of the factor Gram (dense.cu).
// A CTA takes whole leaves; their 32-row slabs go through a 3-stage cp.async ring, warp w of
// the 8 owns the tile pairs of group w in registers and, after a leaf's last slab, writes
// them into the leaf's packed node.  Same products in the same order as the register-split
// and FFMA kernels: identical trees.
template <int T, int g>
__device__ __forceinline__ void leaf_staged_flush(double (&acc)[(T * (T + 1) / 2 + 7) / 8][2], int R,
                                                  int lane, double *__restrict__ out) {
  constexpr int NP = T * (T + 1) / 2;
  constexpr int PPW = (NP + 7) / 8;
  const int kk = lane & 3, col = lane >> 2;
  int p = 0;
#pragma unroll
  for (int a = 0; a < T; ++a)
#pragma unroll
    for (int b = a; b < T; ++b) {
      if (p >= g * PPW && p < (g + 1) * PPW) {
        const int ga = 8 * a + col;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int gb = 8 * b + 2 * kk + u;
          if (ga <= gb && gb < R) out[tri_index(ga, gb, R)] = acc[p - g * PPW][u];
          acc[p - g * PPW][u] = 0.0;
        }
      }
      ++p;
    }
}

template <int T>
__global__ void __launch_bounds__(256, 2)
sts_leaf_staged_kernel(const double *__restrict__ U, int64_t n, int R, int leaf, int64_t nleaves,
                       double *__restrict__ level) {
  constexpr int NP = T * (T + 1) / 2;
  constexpr int PPW = (NP + 7) / 8;
  constexpr int ST = gs_stride<T>();
  constexpr int SLAB = kGsRows * ST;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int Rt = R * (R + 1) / 2, Rs = tri_stride(R);
  const int spl = leaf / kGsRows;   // slabs per leaf (1 or 2)
  double acc[PPW][2];
#pragma unroll
  for (int p = 0; p < PPW; ++p) acc[p][0] = acc[p][1] = 0.0;
  for (int e = threadIdx.x; e < kGsStages * kGsRows * (ST - R); e += blockDim.x) {
    const int st = e / (kGsRows * (ST - R)), q = e - st * (kGsRows * (ST - R));
    const int r = q / (ST - R), c = R + (q - r * (ST - R));
    sm[st * SLAB + r * ST + c] = 0.0;
  }
  // this CTA's slabs, in order: leaf blockIdx.x + (q / spl) gridDim.x, part q % spl
  const int64_t my_leaves = blockIdx.x < nleaves ? (nleaves - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t my_slabs = my_leaves * spl;
  const int crow = threadIdx.x >> 3, c0 = threadIdx.x & 7;
  auto issue = [&](int64_t q, int st) {
    if (q < my_slabs) {
      const int64_t v = blockIdx.x + (q / spl) * gridDim.x;
      const int64_t r = v * leaf + (q % spl) * kGsRows + crow;
      const bool ok = r < n;
      const double *src = U + (ok ? r : 0) * (int64_t)R;
      double *dst = sm + st * SLAB + crow * ST;
      for (int c = c0; c < R; c += 8) cpa8_zfill(dst + c, src + c, ok);
    }
    cpa_commit();
  };
  issue(0, 0);
  issue(1, 1);
  int st = 0;
  for (int64_t q = 0; q < my_slabs; ++q) {
    cpa_wait<1>();
    __syncthreads();
    issue(q + 2, st == 0 ? 2 : st - 1);
    const double *ring = sm + st * SLAB;
    const bool last = (q % spl) == spl - 1;
    double *out = level + (blockIdx.x + (q / spl) * gridDim.x) * (int64_t)Rs;
    switch (wid) {
#define RCP_LS(G_)                                                      \
  case G_:                                                              \
    gram_staged_body<T, G_>(ring, nullptr, false, lane, acc);           \
    if (last) leaf_staged_flush<T, G_>(acc, R, lane, out);              \
    break;
      RCP_LS(0) RCP_LS(1) RCP_LS(2) RCP_LS(3) RCP_LS(4) RCP_LS(5) RCP_LS(6)
      default:
        gram_staged_body<T, 7>(ring, nullptr, false, lane, acc);
        if (last) leaf_staged_flush<T, 7>(acc, R, lane, out);
        break;
#undef RCP_LS
    }
    if (last && Rs > Rt && threadIdx.x == 0) out[Rt] = 0.0;
    st = st == kGsStages - 1 ? 0 : st + 1;
  }
  cpa_wait<0>();
}

template <int T>
int launch_leaf_staged(const double *U, int64_t n, int R, int leaf, int64_t nleaves, double *lvl,
                       cudaStream_t st) {
  const int smem = (int)(sizeof(double) * kGsStages * kGsRows * gs_stride<T>());
  static int per_sm = 0;
  if (!per_sm) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(sts_leaf_staged_kernel<T>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    RCP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sts_leaf_staged_kernel<T>, 256,
                                                               smem));
    if (per_sm < 1) per_sm = 1;
  }
  int64_t g = (int64_t)per_sm * sm_count();
  if (nleaves < g) g = nleaves;
  sts_leaf_staged_kernel<T><<<(unsigned)g, 256, smem, st>>>(U, n, R, leaf, nleaves, lvl);
  return RCP_OK;
}

__global__ void sts_zero_kernel(double *__restrict__ p, int64_t len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

// Up to three tree levels per launch: thread (v, e) of the top level reads the 2^L
// descendants of node v at the bottom level and writes every intermediate node, with the
// same pairwise additions as a level-by-level pass.  Level l nodes start at 2^l - 1.
__global__ void sts_levels_kernel(double *__restrict__ tree, int child_level, int L, int Rt) {
  const int top = child_level - L;
  const int64_t nodes = 1LL << top;
  const int64_t tot = nodes * Rt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / Rt, e = i % Rt;
    double acc[8];
    const int w = 1 << L;
    const double *ch = tree + ((1LL << child_level) - 1 + v * w) * Rt + e;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < w) acc[q] = ch[(int64_t)q * Rt];
    for (int l = 1; l <= L; ++l) {           // level child_level - l
      const int cnt = w >> l;
      double *lvl = tree + ((1LL << (child_level - l)) - 1 + v * cnt) * Rt + e;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < cnt) {
          acc[q] = acc[2 * q] + acc[2 * q + 1];
          lvl[(int64_t)q * Rt] = acc[q];
        }
    }
  }
}

__global__ void sts_cond_kernel(const double *__restrict__ cp, const double *__restrict__ grams,
                                int N, int i, int k, int R, double *__restrict__ M) {
  const int RR = R * R;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < RR; e += gridDim.x * blockDim.x) {
    double m = cp[e];
    for (int t = i + 1; t < N; ++t)
      if (t != k) m = m * grams[(int64_t)t * RR + e];
    M[e] = m;
  }
}

// One warp per sample over the (small) padded rank tree (ref samplers.py:423-451).
__global__ void sts_rank_walk_kernel(const double *__restrict__ ng, int depth, int P,
                                     const int32_t *__restrict__ leaf_rank,
                                     const double *__restrict__ M, const double *__restrict__ H,
                                     int64_t J, int R, uint64_t k0, uint64_t k1,
                                     const uint64_t *__restrict__ dk,
                                     const double *__restrict__ ov, int32_t *__restrict__ owner,
                                     double *__restrict__ rout, double *__restrict__ pmp,
                                     int *status) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= J) return;
  if (dk) {   // graph-replayed round: the key lives in device memory
    k0 = dk[0];
    k1 = dk[1];
  }
  double r = ov ? ov[s] : u64_to_unit(philox_word(k0, k1, (uint64_t)s));
  const double tiny = DBL_MIN;
  double prob = 1.0;
  int64_t v = 0;
  const int RR = R * R;
  for (int lev = 0; lev < depth; ++lev) {
    const double *Gv = ng + ((1LL << lev) - 1 + v) * (int64_t)RR;
    const double *Gl = ng + ((1LL << (lev + 1)) - 1 + 2 * v) * (int64_t)RR;
    double den = 0.0, num = 0.0;
    for (int e = lane; e < RR; e += 32) {
      const int a = e / R, b = e % R;
      const double hm = H[s * R + a] * H[s * R + b] * M[e];
      den = fma(Gv[e], hm, den);
      num = fma(Gl[e], hm, num);
    }
    den = warp_sum(den);
    num = warp_sum(num);
    if (!(den > 0.0)) {
      if (lane == 0) raise_status(status, RCP_ST_DEGENERATE);
      return;
    }
    double T = (num > 0.0 ? num : 0.0) / den;
    T = fmin(fmax(T, 0.0), 1.0);
    const bool right = r >= T;
    prob *= right ? (1.0 - T) : T;
    r = right ? (r - T) / fmax(1.0 - T, tiny) : r / fmax(T, tiny);
    r = fmin(fmax(r, 0.0), one_below());
    v = 2 * v + (right ? 1 : 0);
    const int64_t width = 1LL << (depth - 1 - lev);
    const int64_t lo = v * width;
    const int64_t nreal = min((v + 1) * width, (int64_t)P) - lo;
    if (nreal <= 0) {
      if (lane == 0) raise_status(status, RCP_ST_DEGENERATE);
      return;
    }
  }
  if (lane == 0) {
    owner[s] = depth ? leaf_rank[v] : leaf_rank[0];
    rout[s] = r;
    pmp[s] = prob;
  }
}

// Packed rank tree (ref samplers.py:239-275): leaf v of a complete tree over `width` leaves
// holds the packed upper triangle of block Gram order[v] (zero padding past P), every inner
// node the sum of its two children; the node layout is the local trees' (level order,
// stride tri_stride(R)), so the run-grouped walk reads it unchanged.
__global__ void sts_rank_tree_kernel(const double *__restrict__ blocks,
                                     const int64_t *__restrict__ order, int P, int R, int depth,
                                     double *__restrict__ tree) {
  const int Rt = R * (R + 1) / 2, Rs = tri_stride(R);
  const int64_t width = 1LL << depth;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < Rs; e += gridDim.x * blockDim.x) {
    int a = 0, rem = e;
    if (e < Rt)
      while (rem >= R - a) {
        rem -= R - a;
        ++a;
      }
    const int b = a + rem;
    double *leafs = tree + (width - 1) * (int64_t)Rs;
    for (int64_t v = 0; v < width; ++v) {
      double g = 0.0;
      if (e < Rt && v < P) {
        const int64_t src = order ? order[v] : v;
        g = blocks[(src * R + a) * R + b];
      }
      leafs[v * Rs + e] = g;
    }
    for (int lev = depth - 1; lev >= 0; --lev) {
      double *up = tree + ((1LL << lev) - 1) * (int64_t)Rs;
      const double *dn = tree + ((1LL << (lev + 1)) - 1) * (int64_t)Rs;
      for (int64_t v = 0; v < (1LL << lev); ++v)
        up[v * Rs + e] = dn[(2 * v) * Rs + e] + dn[(2 * v + 1) * Rs + e];
    }
  }
}

// Rank-level walk when every sample shares H = ones (the first constant mode): each CTA
// evaluates the mass <G_v (.) M', 1 1^T> of every rank-tree node once (warp per node over
// the packed triangle), then its threads descend one sample each with
// T = max(q_left, 0) / q_node (ref samplers.py:423-451).
constexpr int kOneGroupMaxNodes = 2047;
__global__ void __launch_bounds__(1024)
rank_walk_ones_kernel(const double *__restrict__ tree, int depth, const int32_t *__restrict__ leaf_rank,
                      const double *__restrict__ M, int R, int64_t J, uint64_t k0, uint64_t k1,
                      const uint64_t *__restrict__ dk, const double *__restrict__ ov,
                      int32_t *__restrict__ owner, double *__restrict__ rout,
                      double *__restrict__ pmp, int *status) {
  __shared__ double q[kOneGroupMaxNodes];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int Rt = R * (R + 1) / 2, Rs = tri_stride(R);
  const int nnodes = (2 << depth) - 1;
  for (int v = wid; v < nnodes; v += nw) {
    const double *g = tree + (int64_t)v * Rs;
    double acc = 0.0;
    // lane's first element and its (a, b); then step 32 elements along the packed rows
    int e = lane, a = 0, rem = lane;
    while (e < Rt && rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    while (e < Rt) {
      const int b = a + rem;
      const double m = M[a * R + b];
      acc = fma(g[e], a == b ? m : 2.0 * m, acc);
      e += 32;
      rem += 32;
      while (e < Rt && rem >= R - a) {
        rem -= R - a;
        ++a;
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) q[v] = acc;
  }
  __syncthreads();
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  if (dk) {
    k0 = dk[0];
    k1 = dk[1];
  }
  double r = ov ? ov[s] : u64_to_unit(philox_word(k0, k1, (uint64_t)s));
  const double tiny = DBL_MIN;
  double prob = 1.0;
  int v = 0;
  for (int lev = 0; lev < depth; ++lev) {
    const double den = q[(1 << lev) - 1 + v];
    const double num = q[(1 << (lev + 1)) - 1 + 2 * v];
    if (!(den > 0.0)) {
      raise_status(status, RCP_ST_DEGENERATE);
      owner[s] = -1;
      return;
    }
    double T = (num > 0.0 ? num : 0.0) / den;
    T = fmin(fmax(T, 0.0), 1.0);
    const bool right = r >= T;
    prob *= right ? (1.0 - T) : T;
    r = right ? (r - T) / fmax(1.0 - T, tiny) : r / fmax(T, tiny);
    r = fmin(fmax(r, 0.0), one_below());
    v = 2 * v + (right ? 1 : 0);
  }
  const int32_t p = leaf_rank[v];
  if (p < 0) {   // "walk branched into an empty padded subtree"
    raise_status(status, RCP_ST_DEGENERATE);
    owner[s] = -1;
    return;
  }
  owner[s] = p;
  rout[s] = r;
  pmp[s] = prob;
}

// Local search of the first constant mode at P > 1 (every sample shares H = ones): the
// samples routed to this rank invert the CDF of its rows' masses with their residual
// (ref _leaf_search_batch samplers.py:313-345), multiplying the path probability.
__global__ void sts_flat_local_kernel(const double *__restrict__ cdf,
                                      const double *__restrict__ dist, int64_t n, int64_t row_lo,
                                      const double *__restrict__ tmass,
                                      const double *__restrict__ rin,
                                      const int32_t *__restrict__ sel, int32_t selv, int64_t J,
                                      int64_t *__restrict__ Xi, double *__restrict__ pmp,
                                      double *__restrict__ resid, int *status) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J || sel[s] != selv) return;
  if (n < 1 || !(tmass[0] > 0.0)) {   // routed to a rank without mass
    raise_status(status, RCP_ST_DEGENERATE);
    Xi[s] = -1;
    return;
  }
  const double u = rin[s];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
  }
  if (lo > n - 1) lo = n - 1;
  const double p = dist[lo];
  Xi[s] = row_lo + lo;
  pmp[s] *= p;
  if (resid) {
    const double below = lo > 0 ? cdf[lo - 1] : 0.0;
    double ro = p > 0.0 ? (u - below) / p : 0.0;
    resid[s] = fmin(fmax(ro, 0.0), one_below());
  }
}

// STS exchange (ref schedules.py:239-247): a rank's contribution to the J x (R + 3) sum
// all-reduce -- row, step probability, residual and factor row of the samples it owns,
// zeros elsewhere -- and, after the reduction, the fold of every sample's row into the
// running Hadamard rows.  One warp per sample.
__global__ void exchange_pack_kernel(const int64_t *__restrict__ Xi, const double *__restrict__ pmp,
                                     const double *__restrict__ resid,
                                     const double *__restrict__ U, int64_t n, int64_t row_lo,
                                     const int32_t *__restrict__ owner, int32_t rank, int64_t J,
                                     int R, double *__restrict__ buf) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= J) return;
  double *dst = buf + s * (int64_t)(R + 3);
  const int64_t row = Xi[s] - row_lo;
  const bool mine = owner[s] == rank && row >= 0 && row < n;
  if (lane == 0) {
    dst[0] = mine ? (double)Xi[s] : 0.0;
    dst[1] = mine ? pmp[s] : 0.0;
    dst[2] = mine ? resid[s] : 0.0;
  }
  const double *src = U + (mine ? row : 0) * R;
  for (int c = lane; c < R; c += 32) dst[3 + c] = mine ? src[c] : 0.0;
}

__global__ void exchange_unpack_kernel(const double *__restrict__ buf, int64_t J, int R, int init,
                                       int64_t *__restrict__ Xi, double *__restrict__ pmp,
                                       double *__restrict__ resid, double *__restrict__ H) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= J) return;
  const double *src = buf + s * (int64_t)(R + 3);
  if (lane == 0) {
    Xi[s] = (int64_t)src[0];
    pmp[s] = src[1];
    resid[s] = src[2];
  }
  double *h = H + s * (int64_t)R;
  for (int c = lane; c < R; c += 32) h[c] = init ? src[3 + c] : h[c] * src[3 + c];
}

}  // namespace

extern "C" {

size_t rcp_arls_build_ws_bytes(int64_t n, int R) {
  (void)R;
  return (size_t)4 * sm_count() * sizeof(double) + scan_ws_bytes(n) + 64;
}

int rcp_arls_build(const double *d_U, int64_t n, int R, const double *d_Gp, double *d_dist,
                   double *d_cdf, double *d_mass, void *d_ws, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || n < 0 || !d_Gp || !d_mass || (n > 0 && (!d_U || !d_dist || !d_cdf || !d_ws)))
    return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (n == 0) {
    RCP_CUDA_TRY(cudaMemsetAsync(d_mass, 0, sizeof(double), st));
    return RCP_OK;
  }
  int64_t want = ceil_div(n, 64);   // 8-row tiles, 8 warps per CTA
  int grid = (int)(want < 4LL * sm_count() ? want : 4LL * sm_count());
  double *part = (double *)d_ws;
  void *scan_ws = (char *)d_ws + (size_t)4 * sm_count() * sizeof(double);
#ifndef RCP_LEV_NBUF
#define RCP_LEV_NBUF 2   // with RCP_LEV_SMEM_KB 110: two CTAs per SM (swept: tools/lab/dense_lab.py)
#endif
#ifndef RCP_LEV_SMEM_KB
#define RCP_LEV_SMEM_KB 110
#endif
  // up to RCP_LEV_NBUF staged tiles per warp within the shared-memory budget
  int nbuf = RCP_LEV_NBUF;
  auto lev_smem = [&](int nb) {
    return sizeof(double) * ((size_t)lev_rn(R) * lev_zs(R) + 8 * (size_t)nb * 8 * lev_zs(R));
  };
  while (nbuf > 1 && lev_smem(nbuf) > RCP_LEV_SMEM_KB * 1024) --nbuf;
  const size_t sm = lev_smem(nbuf);
  static bool attr_set[17] = {};
#define RCP_LEV(K)                                                                              \
  case K:                                                                                       \
    if (!attr_set[K / 2]) {                                                                     \
      RCP_CUDA_TRY(cudaFuncSetAttribute(leverage_mma_kernel<K>,                                 \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
      attr_set[K / 2] = true;                                                                   \
    }                                                                                           \
    leverage_mma_kernel<K><<<grid, 256, sm, st>>>(d_U, n, R, d_Gp, d_dist, part, nbuf);         \
    break
  switch (lev_rn(R) / 4) {
    RCP_LEV(2); RCP_LEV(4); RCP_LEV(6); RCP_LEV(8); RCP_LEV(10); RCP_LEV(12); RCP_LEV(14);
    RCP_LEV(16); RCP_LEV(18); RCP_LEV(20); RCP_LEV(22); RCP_LEV(24); RCP_LEV(26); RCP_LEV(28);
    RCP_LEV(30); RCP_LEV(32);
    default: return RCP_ERR_ARG;
  }
#undef RCP_LEV
  RCP_LAUNCH_CHECK("leverage");
  mass_kernel<<<1, 256, 0, st>>>(part, grid, d_mass);
  RCP_LAUNCH_CHECK("leverage_mass");
  int64_t blocks = ceil_div(n, 256);
  if (blocks > 8LL * sm_count()) blocks = 8LL * sm_count();
  normalize_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_dist, n, d_mass);
  RCP_LAUNCH_CHECK("leverage_normalize");
  int rc = scan_f64_inclusive(d_dist, d_cdf, n, scan_ws, st);
  if (rc) return rc;
  cdf_div_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_cdf, n);
  RCP_LAUNCH_CHECK("cdf_normalize");
  return RCP_OK;
}

int rcp_arls_draw(const double *d_cdf, const double *d_dist, int64_t n, int64_t row_lo,
                  double mass_ratio, const double *d_total_mass, uint64_t key0, uint64_t key1,
                  const uint64_t *d_key, int64_t q, int64_t offset, int64_t *d_rows_out,
                  double *d_prob_out, const double *d_U, int R, double *d_urow_out, int *d_status,
                  void *stream) {
  if (q < 0 || n < 1 || !d_cdf || !d_dist || !d_rows_out || !d_prob_out) return RCP_ERR_ARG;
  if (d_urow_out && (!d_U || R < 1)) return RCP_ERR_ARG;
  if (q == 0) return RCP_OK;
  arls_draw_kernel<<<(unsigned)ceil_div(q, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_cdf, d_dist, n, row_lo, mass_ratio, d_total_mass, key0, key1, d_key, q, offset, d_rows_out,
      d_prob_out, d_U, R, d_urow_out, d_status, RCP_ST_ZERO_MASS);
  RCP_LAUNCH_CHECK("arls_draw");
  return RCP_OK;
}

int rcp_sts_flat_draw(const double *d_cdf, const double *d_dist, int64_t n, int64_t row_lo,
                      const double *d_total_mass, uint64_t key0, uint64_t key1,
                      const uint64_t *d_key, int64_t J,
                      int64_t *d_Xi, double *d_pmp_i, int *d_status, void *stream) {
  if (J < 0 || n < 1 || !d_cdf || !d_dist || !d_Xi || !d_pmp_i || !d_total_mass) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  arls_draw_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_cdf, d_dist, n, row_lo, 1.0, d_total_mass, key0, key1, d_key, J, 0, d_Xi, d_pmp_i, nullptr, 0,
      nullptr, d_status, RCP_ST_DEGENERATE);
  RCP_LAUNCH_CHECK("sts_flat_draw");
  return RCP_OK;
}

int rcp_batch_fold(const int64_t *d_perm, const int64_t *d_rows, const double *d_prob, int64_t J,
                   const double *d_U, int64_t u_row_lo, const double *d_urows, int R, int first,
                   int64_t *d_Xi, double *d_pmp_i, double *d_H, void *stream) {
  if (J < 0 || R < 1 || (J > 0 && (!d_rows || !d_prob || !d_Xi || !d_pmp_i || !d_H)))
    return RCP_ERR_ARG;
  if (!d_urows && !d_U && J > 0) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  batch_fold_kernel<<<(unsigned)ceil_div(J * 32, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_perm, d_rows, d_prob, J, d_U, u_row_lo, d_urows, R, first, d_Xi, d_pmp_i, d_H);
  RCP_LAUNCH_CHECK("batch_fold");
  return RCP_OK;
}

int rcp_sts_depth(int64_t n, int leaf) {
  if (n <= 0 || leaf < 1) return 0;
  int64_t nl = ceil_div(n, leaf);
  int d = 0;
  while ((1LL << d) < nl) ++d;
  return d;
}

size_t rcp_sts_tree_doubles(int64_t n, int leaf, int R) {
  if (n <= 0) return 0;
  int d = rcp_sts_depth(n, leaf);
  return (size_t)((2LL << d) - 1) * (size_t)tri_stride(R);
}

int rcp_sts_build(const double *d_U, int64_t n, int R, int leaf, double *d_tree, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || leaf < 1 || leaf > 64 || n < 0) return RCP_ERR_ARG;
  if (n == 0) return RCP_OK;
  if (!d_U || !d_tree) return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  const int Rt = tri_stride(R);   // node stride (even; pad entry zero)
  const int depth = rcp_sts_depth(n, leaf);
  const int64_t nleaves = ceil_div(n, leaf);
  const int64_t width = 1LL << depth;
  double *lvl = d_tree + (width - 1) * (int64_t)Rt;
  int64_t g = nleaves < 16LL * sm_count() ? nleaves : 16LL * sm_count();
  if (R <= 64) {
    int64_t gm = ceil_div(nleaves, 8);
    if (gm > 8LL * sm_count()) gm = 8LL * sm_count();
    const size_t msm = sizeof(double) * 8 * (size_t)Rt;
    static bool leaf_attr[9] = {};
#define RCP_LEAF(K)                                                                             \
  case K:                                                                                       \
    if (!leaf_attr[K]) {                                                                        \
      RCP_CUDA_TRY(cudaFuncSetAttribute(sts_leaf_mma_kernel<K>,                                 \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
      leaf_attr[K] = true;                                                                      \
    }                                                                                           \
    sts_leaf_mma_kernel<K><<<(unsigned)gm, 256, msm, st>>>(d_U, n, R, leaf, nleaves, lvl);      \
    break
    switch ((R + 7) / 8) {
      RCP_LEAF(1); RCP_LEAF(2); RCP_LEAF(3); RCP_LEAF(4); RCP_LEAF(5); RCP_LEAF(6); RCP_LEAF(7);
      default: RCP_LEAF(8);
    }
#undef RCP_LEAF
    RCP_LAUNCH_CHECK("sts_leaf_mma");
  } else if ((leaf == kGsRows || leaf == 2 * kGsRows) && !getenv_leaf_ffma() && !getenv_leaf_split()) {
    // fp64 tensor cores over shared-memory staged slabs
    int rc = RCP_OK;
    switch ((R + 7) / 8) {
      case 9: rc = launch_leaf_staged<9>(d_U, n, R, leaf, nleaves, lvl, st); break;
      case 10: rc = launch_leaf_staged<10>(d_U, n, R, leaf, nleaves, lvl, st); break;
      case 11: rc = launch_leaf_staged<11>(d_U, n, R, leaf, nleaves, lvl, st); break;
      case 12: rc = launch_leaf_staged<12>(d_U, n, R, leaf, nleaves, lvl, st); break;
      case 13: rc = launch_leaf_staged<13>(d_U, n, R, leaf, nleaves, lvl, st); break;
      case 14: rc = launch_leaf_staged<14>(d_U, n, R, leaf, nleaves, lvl, st); break;
      case 15: rc = launch_leaf_staged<15>(d_U, n, R, leaf, nleaves, lvl, st); break;
      default: rc = launch_leaf_staged<16>(d_U, n, R, leaf, nleaves, lvl, st); break;
    }
    if (rc) return rc;
    RCP_LAUNCH_CHECK("sts_leaf_staged");
  } else if (R <= 96 && !getenv_leaf_ffma()) {   // fp64 tensor cores, tile pairs split over warps
    const int T = (R + 7) / 8;
    const int G = 4, slots = 8 / G;
    int64_t gs = ceil_div(nleaves, (int64_t)slots);
    if (gs > 4LL * sm_count()) gs = 4LL * sm_count();
    const size_t ssm = sizeof(double) * (size_t)slots * Rt;
#define RCP_LEAFS(K)                                                                              \
  case K: {                                                                                       \
    static bool a_ = false;                                                                       \
    if (!a_) {                                                                                    \
      RCP_CUDA_TRY(cudaFuncSetAttribute(sts_leaf_split_kernel<K, 4>,                              \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));  \
      a_ = true;                                                                                  \
    }                                                                                             \
    sts_leaf_split_kernel<K, 4><<<(unsigned)gs, 256, ssm, st>>>(d_U, n, R, leaf, nleaves, lvl);   \
    break;                                                                                        \
  }
    switch (T) {
      RCP_LEAFS(9) RCP_LEAFS(10) RCP_LEAFS(11)
      default: RCP_LEAFS(12)
    }
#undef RCP_LEAFS
    RCP_LAUNCH_CHECK("sts_leaf_split");
    (void)G;
  } else {
  const size_t lsm = sizeof(double) * leaf * R + sizeof(uint16_t) * (size_t)R * (R + 1) / 2;
  static bool attr = false;
  if (!attr) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(sts_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      100 * 1024));
    attr = true;
  }
  sts_leaf_kernel<<<(unsigned)g, 128, lsm, st>>>(d_U, n, R, leaf, nleaves, lvl);
  RCP_LAUNCH_CHECK("sts_leaf");
  }
  if (width > nleaves) {
    int64_t len = (width - nleaves) * Rt;
    int64_t b = ceil_div(len, 256);
    if (b > 8LL * sm_count()) b = 8LL * sm_count();
    sts_zero_kernel<<<(unsigned)b, 256, 0, st>>>(lvl + nleaves * Rt, len);
    RCP_LAUNCH_CHECK("sts_pad");
  }
  for (int cl = depth; cl > 0;) {
    const int L = cl >= 3 ? 3 : cl;
    const int64_t nodes = 1LL << (cl - L);
    int64_t b = ceil_div(nodes * Rt, 256);
    if (b > 8LL * sm_count()) b = 8LL * sm_count();
    sts_levels_kernel<<<(unsigned)b, 256, 0, st>>>(d_tree, cl, L, Rt);
    RCP_LAUNCH_CHECK("sts_levels");
    cl -= L;
  }
  return RCP_OK;
}

int rcp_sts_cond(const double *d_chain_pinv, const double *d_grams, int N, int i, int k, int R,
                 double *d_M, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || N < 2 || !d_chain_pinv || !d_grams || !d_M) return RCP_ERR_ARG;
  sts_cond_kernel<<<(unsigned)ceil_div(R * R, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_chain_pinv, d_grams, N, i, k, R, d_M);
  RCP_LAUNCH_CHECK("sts_cond");
  return RCP_OK;
}

size_t rcp_sts_rank_tree_doubles(int P, int R) {
  if (P < 1 || R < 1) return 0;
  return (size_t)((2LL << rcp_sts_depth(P, 1)) - 1) * (size_t)tri_stride(R);
}

int rcp_sts_rank_tree(const double *d_block_grams, const int64_t *d_order, int P, int R,
                      double *d_tree, void *stream) {
  if (P < 1 || R < 1 || R > RCP_MAX_RANK || !d_block_grams || !d_tree) return RCP_ERR_ARG;
  const int depth = rcp_sts_depth(P, 1);
  sts_rank_tree_kernel<<<(unsigned)ceil_div(tri_stride(R), 128), 128, 0, RCP_STREAM(stream)>>>(
      d_block_grams, d_order, P, R, depth, d_tree);
  RCP_LAUNCH_CHECK("sts_rank_tree");
  return RCP_OK;
}

int rcp_sts_rank_walk_ones(const double *d_rank_tree, int P, const int32_t *d_leaf_rank, int R,
                           const double *d_M, int64_t J, uint64_t key0, uint64_t key1,
                           const uint64_t *d_key, const double *d_override, int32_t *d_owner,
                           double *d_r_out, double *d_pmp_i, int *d_status, void *stream) {
  if (P < 1 || R < 1 || R > RCP_MAX_RANK || J < 0 || !d_rank_tree || !d_leaf_rank || !d_M ||
      !d_owner || !d_r_out || !d_pmp_i)
    return RCP_ERR_ARG;
  const int depth = rcp_sts_depth(P, 1);
  if ((2 << depth) - 1 > kOneGroupMaxNodes) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  // few nodes: small CTAs (each CTA evaluates every node once); many: fewer, larger CTAs
  const int threads = depth <= 4 ? 256 : 1024;
  rank_walk_ones_kernel<<<(unsigned)ceil_div(J, threads), threads, 0, RCP_STREAM(stream)>>>(
      d_rank_tree, depth, d_leaf_rank, d_M, R, J, key0, key1, d_key, d_override, d_owner, d_r_out,
      d_pmp_i, d_status);
  RCP_LAUNCH_CHECK("sts_rank_walk_ones");
  return RCP_OK;
}

int rcp_sts_flat_local(const double *d_cdf, const double *d_dist, int64_t n, int64_t row_lo,
                       const double *d_total_mass, const double *d_rin, const int32_t *d_sel,
                       int32_t sel_value, int64_t J, int64_t *d_Xi, double *d_pmp_i,
                       double *d_resid, int *d_status, void *stream) {
  if (J < 0 || n < 0 || !d_total_mass || !d_rin || !d_sel || !d_Xi || !d_pmp_i) return RCP_ERR_ARG;
  if (n > 0 && (!d_cdf || !d_dist)) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  sts_flat_local_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_cdf, d_dist, n, row_lo, d_total_mass, d_rin, d_sel, sel_value, J, d_Xi, d_pmp_i, d_resid,
      d_status);
  RCP_LAUNCH_CHECK("sts_flat_local");
  return RCP_OK;
}

int rcp_exchange_pack(const int64_t *d_Xi, const double *d_pmp_i, const double *d_resid,
                      const double *d_U, int64_t n, int64_t row_lo, const int32_t *d_owner,
                      int32_t rank, int64_t J, int R, double *d_buf, void *stream) {
  if (J < 0 || R < 1 || n < 0) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (!d_Xi || !d_pmp_i || !d_resid || !d_owner || !d_buf || (n > 0 && !d_U)) return RCP_ERR_ARG;
  exchange_pack_kernel<<<(unsigned)ceil_div(J * 32, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_Xi, d_pmp_i, d_resid, d_U, n, row_lo, d_owner, rank, J, R, d_buf);
  RCP_LAUNCH_CHECK("exchange_pack");
  return RCP_OK;
}

int rcp_exchange_unpack(const double *d_buf, int64_t J, int R, int init, int64_t *d_Xi,
                        double *d_pmp_i, double *d_resid, double *d_H, void *stream) {
  if (J < 0 || R < 1) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (!d_buf || !d_Xi || !d_pmp_i || !d_resid || !d_H) return RCP_ERR_ARG;
  exchange_unpack_kernel<<<(unsigned)ceil_div(J * 32, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_buf, J, R, init, d_Xi, d_pmp_i, d_resid, d_H);
  RCP_LAUNCH_CHECK("exchange_unpack");
  return RCP_OK;
}

int rcp_sts_rank_walk(const double *d_node_grams, int depth, int P, const int32_t *d_leaf_rank,
                      const double *d_M, const double *d_H, int64_t J, int R, uint64_t key0,
                      uint64_t key1, const uint64_t *d_key, const double *d_override,
                      int32_t *d_owner, double *d_r_out, double *d_pmp_i, int *d_status,
                      void *stream) {
  if (J < 0 || R < 1 || depth < 0 || P < 1 || !d_leaf_rank || !d_owner || !d_r_out || !d_pmp_i)
    return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (depth > 0 && (!d_node_grams || !d_M || !d_H)) return RCP_ERR_ARG;
  sts_rank_walk_kernel<<<(unsigned)ceil_div(J * 32, 256), 256, 0, RCP_STREAM(stream)>>>(
      d_node_grams, depth, P, d_leaf_rank, d_M, d_H, J, R, key0, key1, d_key, d_override, d_owner,
      d_r_out, d_pmp_i, d_status);
  RCP_LAUNCH_CHECK("sts_rank_walk");
  return RCP_OK;
}

}  // extern "C"
