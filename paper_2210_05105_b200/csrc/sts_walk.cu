// STS-CP tree walk, run-grouped (ref sts_sample samplers.py:379-468; _inverse_cdf :291-310).
//
// Every sample of constant mode i descends the per-block binary tree of packed node Grams:
// at a node with children (L, R) it computes the child masses q = h^T (G_child (.) M) h,
// goes right iff r >= T = qL / (qL + qR), multiplies its probability by T or 1-T and
// rescales r exactly as the reference does; at a leaf block it inverts the CDF of its
// rows' masses (u (.) h)^T M (u (.) h).
//
// Samples whose running Hadamard rows h are equal (equal indices in the already-sampled
// modes) see identical node masses.  Sorting the samples by (key of those indices, r)
// makes each such group contiguous and ordered by r; at every node the left-goers are a
// prefix of the group.  A group at a node is a *run* [lo, hi) of the sorted array: its
// masses are computed once, the split point is found by binary search, and the run splits
// into a left and a right run.  A run carries its path (thresholds T and directions from
// the root) and the product of its step probabilities, which all its samples share, so no
// per-sample state is touched above the leaves: a sample's rescaled residual at any level
// is recomputed from its uniform by replaying the path's rescalings in the reference's
// order.  Runs flow through a device work queue served by persistent warps.  Work is
// proportional to the number of distinct (h, node) pairs, not samples x levels.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <float.h>

namespace cg = cooperative_groups;

#include "common.cuh"

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

constexpr int kMaxLeaf = 64;
constexpr int kWalkWarps = 8;
constexpr int kMaxDepth = 30;   // local tree depth limit (2^30 leaves)

struct Run {
  int32_t lo, hi;      // sorted positions [lo, hi)
  int32_t level;       // tree level of `node`
  int32_t node;        // node index within its level
  uint32_t dirs;       // bit l: direction taken at level l (1 = right)
  int32_t pad;
  double prob;         // product of the step probabilities so far
  double T[kMaxDepth]; // thresholds at levels 0 .. level-1
};

struct WalkWs {
  size_t o_key, o_key2, o_r, o_r2, o_idx, o_idx2, o_runs, o_ready, o_ctl, o_cub, total;
  size_t cub_bytes;
  int64_t nruns;
  WalkWs(int64_t J, int depth) {
    size_t b1 = 0, b2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, (const double *)nullptr, (double *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)J);
    cub::DeviceRadixSort::SortPairs(nullptr, b2, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)J);
    cub_bytes = b1 > b2 ? b1 : b2;
    size_t t = 0;
    auto add = [&](size_t bytes) {
      size_t o = (t + 255) & ~(size_t)255;
      t = o + bytes;
      return o;
    };
    // runs per level partition the samples: at most J per level, depth+1 levels
    nruns = J * (int64_t)(depth + 1) + 16;
    o_key = add(8 * J);
    o_key2 = add(8 * J);
    o_r = add(8 * J);
    o_r2 = add(8 * J);
    o_idx = add(4 * J);
    o_idx2 = add(4 * J);
    o_runs = add(sizeof(Run) * nruns);
    o_ready = add(4 * nruns);
    o_ctl = add(64);
    o_cub = add(cub_bytes + 256);
    total = t + 256;
  }
};

// Shared doubles per walker warp: P (node stride), h/u row, leaf masses, path; kept even
// so every warp's P is 16-byte aligned.
__host__ __device__ __forceinline__ size_t walk_per_warp(int R) {
  const size_t w = (size_t)tri_stride(R) + R + kMaxLeaf + kMaxDepth + 2;
  return (w + 1) & ~(size_t)1;
}

// control words: [0] queue tail, [1] queue head, [2] samples finished, [3] participants
__device__ __forceinline__ int ld_volatile(const int *p) { return *(volatile const int *)p; }

// The reference's per-level residual rescaling (ref samplers.py:436-440).
__device__ __forceinline__ double rescale(double r, double T, bool right) {
  const double tiny = DBL_MIN;
  const double y = right ? (r - T) / fmax(1.0 - T, tiny) : r / fmax(T, tiny);
  return fmin(fmax(y, 0.0), one_below());
}

__device__ __forceinline__ double replay(double r, const double *T, uint32_t dirs, int level) {
  for (int l = 0; l < level; ++l) r = rescale(r, T[l], (dirs >> l) & 1u);
  return r;
}

__global__ void walk_prepare_kernel(const int64_t *__restrict__ hkey_in, int64_t J, uint64_t k0,
                                    uint64_t k1, const double *__restrict__ ov,
                                    const double *__restrict__ rin, const int32_t *__restrict__ sel,
                                    int32_t selv, int64_t *__restrict__ key, double *__restrict__ r,
                                    int32_t *__restrict__ idx) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  double u;
  if (ov) u = ov[s];
  else if (rin) u = rin[s];
  else u = u64_to_unit(philox_word(k0, k1, (uint64_t)s));
  const bool mine = !sel || sel[s] == selv;
  r[s] = u;
  key[s] = mine ? (hkey_in ? hkey_in[s] : 0) : INT64_MAX;
  idx[s] = (int32_t)s;
}

__global__ void walk_gather_kernel(const int64_t *__restrict__ in, const int32_t *__restrict__ idx,
                                   int64_t J, int64_t *__restrict__ out) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < J) out[s] = in[idx[s]];
}

// One root run per distinct key; counts participants.
__global__ void walk_seed_kernel(const int64_t *__restrict__ key, const int32_t *__restrict__ idx,
                                 int64_t J, const double *__restrict__ pmp_in, Run *runs,
                                 int *ready, int *ctl) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  const int64_t k = key[s];
  if (k == INT64_MAX) return;
  atomicAdd(&ctl[3], 1);
  if (s > 0 && key[s - 1] == k) return;
  int64_t lo = s + 1, hi = J;   // first position with a larger key
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (key[mid] <= k) lo = mid + 1; else hi = mid;
  }
  const int t = atomicAdd(&ctl[0], 1);
  Run &rr = runs[t];
  rr.lo = (int32_t)s;
  rr.hi = (int32_t)lo;
  rr.level = 0;
  rr.node = 0;
  rr.dirs = 0u;
  // samples of one group share their rank-level path, hence this probability
  rr.prob = pmp_in ? pmp_in[idx[s]] : 1.0;
  (void)ready;
}

__global__ void row_keys_kernel(const int64_t *__restrict__ X, int N, int64_t J, Strides8 st,
                                int64_t *__restrict__ out) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  int64_t k = 0;
  for (int m = 0; m < N; ++m)
    if (st.s[m]) k += X[(int64_t)m * J + s] * st.s[m];
  out[s] = k;
}

// Warp-cooperative push of a child run (path of the parent + one step).  Runs entering the
// leaf level are cut into chunks so that the per-sample leaf work spreads over warps.
constexpr int32_t kLeafChunk = 256;

__device__ __forceinline__ void push_child(Run *runs, int *ready, int *ctl, const Run &par,
                                           int32_t lo, int32_t hi, double T, bool right,
                                           int depth, int lane) {
  const int lev = par.level;
  const int32_t chunk = (lev + 1 == depth) ? kLeafChunk : hi - lo;
  for (int32_t c0 = lo; c0 < hi; c0 += chunk) {
    int t = 0;
    if (lane == 0) t = atomicAdd(&ctl[0], 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    Run &c = runs[t];
    if (lane < lev) c.T[lane] = par.T[lane];
    if (lane == 0) {
      c.lo = c0;
      c.hi = min(hi, c0 + chunk);
      c.level = lev + 1;
      c.node = 2 * par.node + (right ? 1 : 0);
      c.dirs = par.dirs | ((right ? 1u : 0u) << lev);
      c.prob = par.prob * (right ? (1.0 - T) : T);
      c.T[lev] = T;
    }
    __syncwarp();
  }
  (void)ready;
}

__global__ void __launch_bounds__(kWalkWarps * 32)
walk_runs_kernel(const double *__restrict__ tree, const double *__restrict__ U, int64_t n, int R,
                 int leaf, int depth, int64_t row_lo, const double *__restrict__ Mfull,
                 const double *__restrict__ H, const int32_t *__restrict__ idx,
                 const double *__restrict__ r, Run *runs, int *ready, int *ctl, int64_t cap_runs,
                 int64_t *__restrict__ Xi, double *__restrict__ pmp, double *__restrict__ resid,
                 int *status) {
  extern __shared__ double sh[];
  const int Rt = R * (R + 1) / 2;
  const int Rs = tri_stride(R);                    // even node stride (zero pad)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t per_warp = walk_per_warp(R);
  double *Mp = sh;                                 // Rs: packed M, off-diagonals x2
  double *P = Mp + Rs + (size_t)wid * per_warp;    // per warp: Rs (16-byte aligned)
  double *uv = P + Rs;                             // R
  double *mass = uv + R;                           // leaf
  double *Tp = mass + kMaxLeaf;                    // path thresholds of the current run
  uint16_t *pairs = reinterpret_cast<uint16_t *>(Mp + Rs + (size_t)nw * per_warp);
  if (Rs > Rt && threadIdx.x == 0) Mp[Rt] = 0.0;
  for (int e = threadIdx.x; e < Rt; e += blockDim.x) {
    int a = 0, rem = e;
    while (rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    const int b = a + rem;
    pairs[e] = (uint16_t)(a | (b << 8));
    const double m = Mfull[a * R + b];
    Mp[e] = (a == b) ? m : 2.0 * m;
  }
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const int64_t gwarp = (int64_t)blockIdx.x * nw + wid;
  const int64_t nwarps = (int64_t)gridDim.x * nw;
  int64_t begin = 0;
  // Level-synchronous breadth: the runs of one tree level are [begin, end); their children
  // are appended behind `end` and become the next level after a grid-wide barrier.
  for (int lvl = 0; lvl <= depth; ++lvl) {
  const int64_t end = min((int64_t)ld_volatile(&ctl[0]), cap_runs);
  for (int64_t t = begin + gwarp; t < end; t += nwarps) {
    const Run &run = runs[t];
    const int32_t lo = run.lo, hi = run.hi, level = run.level;
    const uint32_t dirs = run.dirs;
    if (lane < level) Tp[lane] = run.T[lane];
    // P = (h h^T) (.) M' of the run's common Hadamard row
    const int32_t s0 = idx[lo];
    for (int c = lane; c < R; c += 32) uv[c] = H ? H[(int64_t)s0 * R + c] : 1.0;
    __syncwarp();
    for (int e = lane; e < Rs; e += 32) {
      const uint16_t ab = e < Rt ? pairs[e] : 0;
      P[e] = e < Rt ? uv[ab & 0xff] * uv[ab >> 8] * Mp[e] : 0.0;
    }
    __syncwarp();
    if (level < depth) {
      const int64_t v = run.node;
      const double2 *GL = reinterpret_cast<const double2 *>(
          tree + ((1LL << (level + 1)) - 1 + 2 * v) * (int64_t)Rs);
      const double2 *GR = GL + Rs / 2;
      const double2 *P2 = reinterpret_cast<const double2 *>(P);
      double qL = 0.0, qR = 0.0, qL2 = 0.0, qR2 = 0.0;
      const int n2 = Rs / 2;
#pragma unroll 4
      for (int e = lane; e < n2; e += 32) {
        const double2 gl = __ldg(GL + e);
        const double2 gr = __ldg(GR + e);
        const double2 p = P2[e];
        qL = fma(gl.x, p.x, qL);
        qL2 = fma(gl.y, p.y, qL2);
        qR = fma(gr.x, p.x, qR);
        qR2 = fma(gr.y, p.y, qR2);
      }
      qL += qL2;
      qR += qR2;
      qL = warp_sum(qL);
      qR = warp_sum(qR);
      qL = qL > 0.0 ? qL : 0.0;
      qR = qR > 0.0 ? qR : 0.0;
      const double tot = qL + qR;
      if (!(tot > 0.0)) {
        for (int32_t s = lo + lane; s < hi; s += 32) Xi[idx[s]] = -1;
        __syncwarp();
        if (lane == 0) {
          raise_status(status, RCP_ST_DEGENERATE);
          __threadfence();
          atomicAdd(&ctl[2], hi - lo);
        }
        continue;
      }
      double T = qL / tot;
      T = fmin(fmax(T, 0.0), 1.0);
      // left-goers (replayed r < T) are a prefix of the r-sorted run: 32-ary search
      int32_t a = lo, b = hi;   // answer in [a, b]
      while (b - a > 0) {
        const int32_t span = b - a;
        const int32_t step = (span + 31) / 32;
        const int32_t pos = a + lane * step;
        bool ge = true;   // "replayed r >= T" at pos (positions >= b count as true)
        if (pos < b) ge = replay(r[pos], Tp, dirs, level) >= T;
        const unsigned m = __ballot_sync(0xffffffffu, ge);
        if (m == 0u) {                     // every probe < T: answer beyond the last probe
          a = a + 31 * step + 1;
          continue;
        }
        const int first = __ffs(m) - 1;   // first lane whose probe is >= T
        if (first == 0) {
          b = a;
        } else {                           // answer in (probe[first-1], probe[first]]
          const int32_t na = a + (first - 1) * step + 1;
          b = min(b, a + first * step);
          a = na;
        }
      }
      const int32_t nl = a - lo;
      if (nl > 0) push_child(runs, ready, ctl, run, lo, lo + nl, T, false, depth, lane);
      if (hi - lo - nl > 0) push_child(runs, ready, ctl, run, lo + nl, hi, T, true, depth, lane);
      continue;
    }
    // ---- leaf block: masses of its rows, then each sample's inverse CDF
    const int64_t r0 = (int64_t)run.node * leaf;
    const int nr = (int)min((int64_t)leaf, n - r0);
    const double rprob = run.prob;
    bool bad = nr <= 0;
    double total_m = 0.0;
    if (!bad) {
      for (int q = 0; q < nr; ++q) {
        for (int c = lane; c < R; c += 32) uv[c] = U[(r0 + q) * R + c];
        __syncwarp();
        double m = 0.0;
        for (int e = lane; e < Rt; e += 32) {
          const uint16_t ab = pairs[e];
          m = fma(uv[ab & 0xff] * uv[ab >> 8], P[e], m);
        }
        m = warp_sum(m);
        if (lane == 0) mass[q] = m > 0.0 ? m : 0.0;
        __syncwarp();
      }
      if (lane == 0)
        for (int q = 0; q < nr; ++q) total_m += mass[q];
      total_m = __shfl_sync(0xffffffffu, total_m, 0);
      bad = !(total_m > 0.0);
    }
    if (bad) {
      for (int32_t s = lo + lane; s < hi; s += 32) Xi[idx[s]] = -1;
      __syncwarp();
      if (lane == 0) {
        raise_status(status, RCP_ST_DEGENERATE);
        __threadfence();
        atomicAdd(&ctl[2], hi - lo);
      }
      continue;
    }
    for (int32_t s = lo + lane; s < hi; s += 32) {
      const double target = replay(r[s], Tp, dirs, level) * total_m;
      double cdf = 0.0;
      int cnt = 0;
      for (int q = 0; q < nr; ++q) {
        cdf += mass[q];
        if (cdf <= target) ++cnt;
      }
      const int choice = cnt < nr - 1 ? cnt : nr - 1;
      double cdf_at = 0.0;
      for (int q = 0; q <= choice; ++q) cdf_at += mass[q];
      const double picked = mass[choice];
      double ro = picked > 0.0 ? (target - (cdf_at - picked)) / picked : 0.0;
      ro = fmin(fmax(ro, 0.0), one_below());
      const int32_t o = idx[s];
      Xi[o] = row_lo + r0 + choice;
      pmp[o] = rprob * (picked / total_m);
      if (resid) resid[o] = ro;
    }
    __syncwarp();
    if (lane == 0) atomicAdd(&ctl[2], hi - lo);
  }
  begin = end;
  grid.sync();
  }
}

// out[s,:] = U[X_i[s]-row_lo, :] (init) or out[s,:] *= U[...] for the selected samples:
// the H-row fold after a walk (ref samplers.py:464) and the owner's row payload at P > 1.
__global__ void fold_rows_kernel(double *__restrict__ out, const double *__restrict__ U, int64_t n,
                                 int R, int64_t row_lo, const int64_t *__restrict__ Xi, int64_t J,
                                 int init, const int32_t *__restrict__ sel, int32_t selv) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= J) return;
  if (sel && sel[s] != selv) return;
  const int64_t row = Xi[s] - row_lo;
  if (row < 0 || row >= n) return;
  const double *src = U + row * R;
  double *dst = out + s * R;
  for (int c = lane; c < R; c += 32) dst[c] = init ? src[c] : dst[c] * src[c];
}

size_t walk_smem(int R, int warps) {
  return sizeof(double) * ((size_t)tri_stride(R) + (size_t)warps * walk_per_warp(R)) +
         sizeof(uint16_t) * (size_t)tri_stride(R) + 64;
}

}  // namespace

extern "C" {

size_t rcp_sts_walk_ws_bytes(int64_t J, int64_t n, int leaf) {
  WalkWs w(J > 0 ? J : 1, rcp_sts_depth(n, leaf));
  return w.total;
}

int rcp_sts_walk(const double *d_tree, const double *d_U, int64_t n, int R, int leaf,
                 int64_t row_lo, const double *d_M, const double *d_H_in, const int64_t *d_hkey,
                 int64_t J, uint64_t key0, uint64_t key1, const double *d_override,
                 const double *d_rin, const int32_t *d_sel, int32_t sel_value, int64_t *d_Xi,
                 double *d_pmp_i, double *d_resid, void *d_ws, size_t ws_bytes, int *d_status,
                 void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || leaf < 1 || leaf > kMaxLeaf || J < 0 || n < 0 ||
      J >= (1LL << 31))
    return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (n == 0 || !d_tree || !d_U || !d_M || !d_Xi || !d_pmp_i || !d_ws) return RCP_ERR_ARG;
  const int depth = rcp_sts_depth(n, leaf);
  if (depth > kMaxDepth) return RCP_ERR_ARG;
  WalkWs L(J, depth);
  if (ws_bytes < L.total) return RCP_ERR_ARG;
  int warps = kWalkWarps;
  while (warps > 1 && walk_smem(R, warps) > 200 * 1024) --warps;
  const size_t smem = walk_smem(R, warps);
  if (smem > 220 * 1024) return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  char *w = (char *)d_ws;
  int64_t *key = (int64_t *)(w + L.o_key), *key2 = (int64_t *)(w + L.o_key2);
  double *r = (double *)(w + L.o_r), *r2 = (double *)(w + L.o_r2);
  int32_t *idx = (int32_t *)(w + L.o_idx), *idx2 = (int32_t *)(w + L.o_idx2);
  Run *runs = (Run *)(w + L.o_runs);
  int *ready = (int *)(w + L.o_ready);
  int *ctl = (int *)(w + L.o_ctl);
  void *cub_tmp = w + L.o_cub;
  const unsigned gb = (unsigned)ceil_div(J, 256);
  walk_prepare_kernel<<<gb, 256, 0, st>>>(d_hkey, J, key0, key1, d_override, d_rin, d_sel,
                                          sel_value, key, r, idx);
  RCP_LAUNCH_CHECK("walk_prepare");
  // sort by r, then stably by key: runs of equal key are contiguous and r-ordered
  size_t tb = L.cub_bytes;
  RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, r, r2, idx, idx2, (int)J, 0, 64, st));
  RCP_LAUNCH_CHECK("walk_sort_r");
  walk_gather_kernel<<<gb, 256, 0, st>>>(key, idx2, J, key2);
  RCP_LAUNCH_CHECK("walk_gather");
  tb = L.cub_bytes;
  RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, key2, key, idx2, idx, (int)J, 0, 64, st));
  RCP_LAUNCH_CHECK("walk_sort_key");
  walk_gather_kernel<<<gb, 256, 0, st>>>((const int64_t *)r, idx, J, (int64_t *)r2);
  RCP_LAUNCH_CHECK("walk_gather_r");
  RCP_CUDA_TRY(cudaMemsetAsync(ctl, 0, 64, st));
  walk_seed_kernel<<<gb, 256, 0, st>>>(key, idx, J, d_sel ? d_pmp_i : nullptr, runs, ready, ctl);
  RCP_LAUNCH_CHECK("walk_seed");
  static bool attr = false;
  if (!attr) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(walk_runs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      220 * 1024));
    attr = true;
  }
  int per_sm = 0;
  RCP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_runs_kernel,
                                                             warps * 32, smem));
  if (per_sm < 1) return RCP_ERR_ARG;
  // persistent: every CTA resident at once (workers wait on the shared queue)
  const int grid = per_sm * sm_count();
  // cooperative launch: every CTA co-resident, grid-wide barrier between tree levels
  const double *a_tree = d_tree, *a_U = d_U, *a_M = d_M, *a_H = d_H_in;
  const int32_t *a_idx = idx;
  const double *a_r = r2;
  int64_t a_n = n, a_row_lo = row_lo, a_cap = L.nruns;
  int a_R = R, a_leaf = leaf, a_depth = depth;
  void *args[] = {(void *)&a_tree, (void *)&a_U, (void *)&a_n, (void *)&a_R, (void *)&a_leaf,
                  (void *)&a_depth, (void *)&a_row_lo, (void *)&a_M, (void *)&a_H, (void *)&a_idx,
                  (void *)&a_r, (void *)&runs, (void *)&ready, (void *)&ctl, (void *)&a_cap,
                  (void *)&d_Xi, (void *)&d_pmp_i, (void *)&d_resid, (void *)&d_status};
  RCP_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)walk_runs_kernel, dim3(grid),
                                           dim3(warps * 32), args, smem, st));
  RCP_LAUNCH_CHECK("walk_runs");
  return RCP_OK;
}

int rcp_fold_rows(double *d_out, const double *d_U, int64_t n, int R, int64_t row_lo,
                  const int64_t *d_Xi, int64_t J, int init, const int32_t *d_sel,
                  int32_t sel_value, void *stream) {
  if (R < 1 || J < 0 || n < 0) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (!d_out || !d_U || !d_Xi) return RCP_ERR_ARG;
  const int64_t threads = J * 32;
  int64_t blocks = ceil_div(threads, 256);
  fold_rows_kernel<<<(unsigned)blocks, 256, 0, RCP_STREAM(stream)>>>(d_out, d_U, n, R, row_lo, d_Xi,
                                                                     J, init, d_sel, sel_value);
  RCP_LAUNCH_CHECK("fold_rows");
  return RCP_OK;
}

int rcp_row_keys(const int64_t *d_X, int N, int64_t J, const int64_t *h_strides, int64_t *d_out,
                 void *stream) {
  if (N < 1 || N > 8 || J < 0 || !h_strides) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  if (!d_X || !d_out) return RCP_ERR_ARG;
  Strides8 sd;
  for (int m = 0; m < 8; ++m) sd.s[m] = m < N ? h_strides[m] : 0;
  row_keys_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, RCP_STREAM(stream)>>>(d_X, N, J, sd, d_out);
  RCP_LAUNCH_CHECK("row_keys");
  return RCP_OK;
}

}  // extern "C"
