// STS-CP tree walk, run-grouped (ref sts_sample samplers.py:379-468; _inverse_cdf :291-310).
//
// Every sample of constant mode i descends the per-block binary tree of packed node Grams:
// at a node with children (L, R) it computes the child masses q = h^T (G_child (.) M) h,
// goes right iff r >= T = qL / (qL + qR), multiplies its probability by T or 1-T and
// rescales r exactly as the reference does; at a leaf block it inverts the CDF of its
// rows' masses (u (.) h)^T M (u (.) h).
//
// Samples whose running Hadamard rows h are equal (equal indices in the already-sampled
// modes) see identical node masses.  Sorting the samples by the key of those indices makes
// each such group contiguous.  A group at a node is a *run* [lo, hi) of the array: its
// child masses are computed once; its samples' residuals r are compared with the split
// T = qL / (qL + qR), rescaled exactly as the reference does (ref samplers.py:436-440), and
// partitioned into the left and right child runs of the next level (double-buffered
// (r, sample) arrays).  Work is proportional to the number of distinct (h, node) pairs
// plus one pass over the samples per level.
//
// Per walk, every node Gram is multiplied once by the packed conditioning matrix M'
// (GM = G (.) M'), so a child mass is <GM_child, h h^T> with h read from shared memory.
// Leaf row masses z^T M z (z = u (.) h) run on the fp64 tensor cores for R <= 64.  The
// levels are processed by one cooperative launch with a grid barrier between levels.
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
// Runs entering the leaf level are cut into chunks so that the per-sample leaf work
// spreads over warps; longer runs elsewhere are cut into pieces of at most kMaxRun samples
// (same key, same node): each piece recomputes the same child masses, but no warp
// partitions more than kMaxRun samples.
constexpr int32_t kLeafChunk = 256;
constexpr int32_t kMaxRun = 256;
#ifndef RCP_WALK_UNROLL
#define RCP_WALK_UNROLL 8   // child-mass loop: node loads in flight per lane (swept: 4/8/10)
#endif
#ifndef RCP_WALK_MIN_BLOCKS
#define RCP_WALK_MIN_BLOCKS 2
#endif
constexpr int kWalkUnroll = RCP_WALK_UNROLL;
#ifndef RCP_WALK_UNROLL_BIG
#define RCP_WALK_UNROLL_BIG 16
#endif
constexpr int kWalkUnrollBig = RCP_WALK_UNROLL_BIG;
// Diagnostics (per-level finish times, sample counters): off in the product build, where
// they cost same-address global atomics per sample, run and CTA; tools/lab/walk_trace.py
// builds with -DRCP_WALK_PROF=1.
#ifndef RCP_WALK_PROF
#ifdef RCP_WALK_TRACE
#define RCP_WALK_PROF 1
#else
#define RCP_WALK_PROF 0
#endif
#endif
#ifndef RCP_WALK_WARPS
#define RCP_WALK_WARPS 16
#endif
constexpr int kWalkWarps = RCP_WALK_WARPS;
constexpr int kMaxDepth = 30;   // local tree depth limit (2^30 leaves)
// control words: [0] seeded runs, [2] samples finished, [3] participants,
// [kGenBase + g] runs pushed during generation g (each generation has its own counter, so
// the extent of generation g + 1 is stable once every CTA has passed the barrier)
constexpr int kGenBase = 8;
// per level: [start time, runs] at 2 l, then [last warp finish, ~first warp finish] at
// 2 (kMaxDepth + 2) + 2 l (global timer, ns).  With -DRCP_WALK_TRACE also, per level, the
// longest time any warp spent in each phase of one run (claim -> run record, -> h row,
// -> child mass, -> partition + push) at 4 (kMaxDepth + 2) + 4 l (diagnostics only).
#ifdef RCP_WALK_TRACE
constexpr size_t kProfBytes = 64 * (kMaxDepth + 2);
#else
constexpr size_t kProfBytes = 32 * (kMaxDepth + 2);
#endif
constexpr size_t kCtlBytes = sizeof(int) * (kGenBase + kMaxDepth + 8);

struct Run {
  int32_t lo, hi;      // positions [lo, hi) in the level's (r, sample) buffer
  int32_t hrow;        // a sample of the run's group: the row of H all its samples share
  int32_t node;        // node index within its level (the level is the pass's: runs are
                       // processed level-synchronously)
  double prob;         // product of the step probabilities so far
  double qv;           // h'(G_node (.) M)h when known (left children inherit it), else NaN
};

struct WalkWs {
  size_t o_key, o_key2, o_r, o_r2, o_idx, o_idx2, o_idx3, o_runs, o_ctl, o_mp, o_pairs, o_gm,
      o_cub, o_prof, total;
  size_t cub_bytes;
  int64_t nruns;
  WalkWs(int64_t J, int depth, int R) {
    size_t b1 = 0, b2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b2, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)J);
    cub_bytes = b1 > b2 ? b1 : b2;
    size_t t = 0;
    auto add = [&](size_t bytes) {
      size_t o = (t + 255) & ~(size_t)255;
      t = o + bytes;
      return o;
    };
    // runs of one level partition that level's samples: at most J per level
    nruns = J * (int64_t)(depth + 1) + 16;
    const size_t Rs = (size_t)tri_stride(R);
    o_key = add(8 * J);
    o_key2 = add(8 * J);
    o_r = add(8 * J);
    o_r2 = add(8 * J);
    o_idx = add(4 * J);
    o_idx2 = add(4 * J);
    o_idx3 = add(4 * J);
    o_runs = add(sizeof(Run) * nruns);
    o_ctl = add(kCtlBytes);
    o_mp = add(8 * Rs);
    o_pairs = add(4 * Rs);
    o_gm = add(8 * Rs * (size_t)((2LL << depth) - 1));   // G (.) M' for every tree node
    o_cub = add(cub_bytes + 256);
    o_prof = add(kProfBytes);   // per level: global timer at the level start, runs
    total = t + 256;
  }
};

// Leaf masses on the fp64 tensor cores (mma.m8n8k4) when R <= kMmaMaxR: Y = Z M for a
// tile of 8 leaf rows Z = U_leaf (.) h, mass_q = <Y_q, Z_q>.
constexpr int kMmaMaxR = 128;
static_assert(kMmaMaxR >= RCP_MAX_RANK, "leaf masses run on the tensor cores for every rank");
__host__ __device__ __forceinline__ int mma_rn(int R) { return (R + 7) & ~7; }
// Row strides of the leaf tile Z and of M in shared memory: Rn + 4 is 4 or 12 mod 16 doubles,
// so the mma fragment reads (8 rows x 4 k of Z, 4 k x 8 columns of M) hit 16 distinct
// double-banks per half-warp (Rn + 2 and Rn were 2-way conflicted: 4 wavefronts per load).
__host__ __device__ __forceinline__ int mma_zs(int R) { return mma_rn(R) + 4; }
__host__ __device__ __forceinline__ int mma_ms(int R) { return mma_rn(R) + 4; }

// Shared doubles per walker warp: h, leaf rows z = u (.) h (a batch, or an 8-row mma
// tile), leaf masses, path.
__host__ __device__ __forceinline__ size_t walk_per_warp(int R) {
  const size_t zb = (size_t)8 * mma_zs(R);
  const size_t w = (size_t)R + zb + kMaxLeaf;
  return (w + 1) & ~(size_t)1;
}

// The inner levels alone need the run's Hadamard row only.
__host__ __device__ __forceinline__ size_t walk_per_warp_inner(int R) {
  return ((size_t)R + 1) & ~(size_t)1;
}

// Block-shared doubles: the full padded M (mma path) or packed M' (fallback).
__host__ __device__ __forceinline__ size_t walk_block_doubles(int R) {
  return (size_t)mma_rn(R) * mma_ms(R);
}

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int ld_volatile(const int *p) { return *(volatile const int *)p; }

// The reference's per-level residual rescaling (ref samplers.py:436-440).
__device__ __forceinline__ double rescale(double r, double T, bool right) {
  const double tiny = DBL_MIN;
  const double y = right ? (r - T) / fmax(1.0 - T, tiny) : r / fmax(T, tiny);
  return fmin(fmax(y, 0.0), one_below());
}

__global__ void walk_prepare_kernel(const int64_t *__restrict__ hkey_in, int64_t J,
                                    const int32_t *__restrict__ sel, int32_t selv,
                                    int64_t *__restrict__ key, int32_t *__restrict__ idx,
                                    int *__restrict__ ctl, unsigned long long *__restrict__ prof) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (blockIdx.x == 0) {   // control words and the per-level timing record
    for (int q = threadIdx.x; q < (int)(kCtlBytes / sizeof(int)); q += blockDim.x) ctl[q] = 0;
    for (int q = threadIdx.x; q < (int)(kProfBytes / 8); q += blockDim.x) prof[q] = 0ull;
  }
  if (s >= J) return;
  const bool mine = !sel || sel[s] == selv;
  key[s] = mine ? (hkey_in ? hkey_in[s] : 0) : INT64_MAX;
  idx[s] = (int32_t)s;
}

// Level-0 buffer: the uniform of each sample in key order.
__global__ void walk_fill_r_kernel(const int32_t *__restrict__ idx, int64_t J, uint64_t k0,
                                   uint64_t k1, const uint64_t *__restrict__ dkey,
                                   const double *__restrict__ ov,
                                   const double *__restrict__ rin, double *__restrict__ r) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= J) return;
  if (dkey) {   // stream key resident on the device (graph-replayed rounds)
    k0 = dkey[0];
    k1 = dkey[1];
  }
  const int32_t s = idx[i];
  double u;
  if (ov) u = ov[s];
  else if (rin) u = rin[s];
  else u = u64_to_unit(philox_word(k0, k1, (uint64_t)s));
  r[i] = u;
}

// One root run per distinct key; counts participants.
__global__ void walk_seed_kernel(const int64_t *__restrict__ key, const int32_t *__restrict__ idx,
                                 int64_t J, const double *__restrict__ pmp_in, Run *runs,
                                 int *ctl) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  const int64_t k = key[s];
  if (k == INT64_MAX) return;
#if RCP_WALK_PROF
  atomicAdd(&ctl[3], 1);
#endif
  if (s > 0 && key[s - 1] == k) return;
  int64_t lo = s + 1, hi = J;   // first position with a larger key
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (key[mid] <= k) lo = mid + 1; else hi = mid;
  }
  // samples of one group share their rank-level path, hence this probability
  const double prob = pmp_in ? pmp_in[idx[s]] : 1.0;
  const int pieces = (int)((lo - s + kMaxRun - 1) / kMaxRun);
  const int t = atomicAdd(&ctl[0], pieces);
  for (int q = 0; q < pieces; ++q) {
    Run rr;
    rr.lo = (int32_t)(s + (int64_t)q * kMaxRun);
    rr.hi = (int32_t)min(lo, s + (int64_t)(q + 1) * kMaxRun);
    rr.hrow = idx[s];
    rr.node = 0;
    rr.prob = prob;
    rr.qv = __longlong_as_double(0x7ff8000000000000LL);   // unknown
    runs[t + q] = rr;
  }
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

// Packed M' (off-diagonals doubled, zero pad to the even stride) and the (a, b) index pair
// of every packed position.
// Tables are stored in split-half order: position 2i holds packed element i, position
// 2i+1 element i + Rs/2, so a lane's double2 at index i covers two elements whose (a, b)
// indices run consecutively across lanes (conflict-free h[b] reads in shared memory).
__host__ __device__ __forceinline__ int split_pos(int e, int n2) {
  return e < n2 ? 2 * e : 2 * (e - n2) + 1;
}

__global__ void walk_tables_kernel(const double *__restrict__ Mfull, int R, double *__restrict__ Mp,
                                   uint32_t *__restrict__ pairs) {
  const int Rt = R * (R + 1) / 2, Rs = tri_stride(R), n2 = Rs / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < Rs; e += gridDim.x * blockDim.x) {
    const int ps = split_pos(e, n2);
    if (e >= Rt) {
      Mp[ps] = 0.0;
      pairs[ps] = 0u;
      continue;
    }
    int a = 0, rem = e;
    while (rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    const int b = a + rem;
    const double m = Mfull[a * R + b];
    Mp[ps] = (a == b) ? m : 2.0 * m;
    pairs[ps] = (uint32_t)a | ((uint32_t)b << 16);
  }
}

// GM[node] = G[node] (.) M' for one walk (split-half order): a node's child mass is then
// <GM, h h^T>.  n2: double2 slots over all nodes; Rs2 = Rs / 2 slots per node.
__global__ void walk_gm_kernel(const double *__restrict__ tree, const double2 *__restrict__ Mp,
                               int64_t n2, int Rs2, double2 *__restrict__ gm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = i / Rs2, j = i - node * Rs2;
    const double *g = tree + node * 2 * Rs2;
    const double2 m = Mp[j];
    gm[i] = make_double2(g[j] * m.x, g[j + Rs2] * m.y);
  }
}

// Warp-cooperative push of a child run (path of the parent + one step) into the next
// level's generation.  Runs entering the leaf level are cut into chunks so that the
// per-sample leaf work spreads over warps.


// Child runs are staged in a per-CTA shared buffer and published with one global
// reservation per CTA and level (a global counter taking one atomic per child run
// serialised ~2*10^4 same-address atomics per level); a full buffer falls back to the
// global counter.
constexpr int kStage = 224;   // two CTAs of 16 walker warps per SM at R = 50

struct Stage {
  Run buf[kStage];
  int count;
  int base;
};

__device__ __forceinline__ void push_child(Run *runs, int *gen_cnt, int64_t base, int64_t cap,
                                           int *status, Stage &stg, const Run &par, int32_t lo,
                                           int32_t hi, double T, bool right, double qv, int depth,
                                           int lev, int lane) {
  const int32_t chunk = (lev + 1 == depth) ? kLeafChunk : kMaxRun;
  for (int32_t c0 = lo; c0 < hi; c0 += chunk) {
    if (lane == 0) {
      Run c;
      c.lo = c0;
      c.hi = min(hi, c0 + chunk);
      c.hrow = par.hrow;
      c.node = 2 * par.node + (right ? 1 : 0);
      c.prob = par.prob * (right ? (1.0 - T) : T);
      c.qv = qv;
      const int t = atomicAdd(&stg.count, 1);
      if (t < kStage) {
        stg.buf[t] = c;
      } else {
        const int g = atomicAdd(gen_cnt, 1);
        if (base + g >= cap) raise_status(status, RCP_ST_CAPACITY);   // cannot happen: one
        else runs[base + g] = c;   // level holds at most J disjoint runs
      }
    }
  }
  __syncwarp();
}

// End of a level: the CTA's staged children go to the next level's array.
__device__ __forceinline__ void publish_children(Run *runs, int *gen_cnt, int64_t base,
                                                 int64_t cap, int *status, Stage &stg) {
  __syncthreads();
  const int n = min(stg.count, kStage);
  if (threadIdx.x == 0) stg.base = n ? atomicAdd(gen_cnt, n) : 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t o = base + stg.base + i;
    if (o >= cap) raise_status(status, RCP_ST_CAPACITY);
    else runs[o] = stg.buf[i];
  }
  if (threadIdx.x == 0) stg.count = 0;
}

// A degenerate run (zero node or leaf mass: ref DegenerateWalkError samplers.py:428-430)
// marks its samples' indices -1 and zeroes their Hadamard output rows, so nothing after
// it in the solve reads unset memory; the status flag is raised for the host.
__device__ __forceinline__ void fail_run(int32_t lo, int32_t hi, const int32_t *__restrict__ idx,
                                         int64_t *__restrict__ Xi, double *__restrict__ Hout,
                                         int R, int *status, int *ctl, int lane,
                                         int32_t *__restrict__ owner = nullptr) {
  for (int32_t s = lo + lane; s < hi; s += 32) {
    if (Xi) Xi[idx[s]] = -1;
    if (owner) owner[idx[s]] = -1;   // rank mode: no rank finishes these samples
  }
  if (Hout)
    for (int32_t s = lo; s < hi; ++s) {
      double *dst = Hout + (int64_t)idx[s] * R;
      for (int c = lane; c < R; c += 32) dst[c] = 0.0;
    }
  __syncwarp();
  if (lane == 0) {
    raise_status(status, RCP_ST_DEGENERATE);
    __threadfence();
    atomicAdd(&ctl[2], hi - lo);
  }
}

// kMinB / kUn: resident CTAs per SM the register budget is set for, and node loads in flight
// per lane in the child-mass loop.  <RCP_WALK_MIN_BLOCKS, kWalkUnroll> where shared memory lets
// two CTAs share an SM (R <= 64: node tables mostly L2-resident); <1, kWalkUnrollBig> above,
// where one CTA fits anyway and the 10^1 KB node tables of million-row trees stream from HBM:
// twice the registers buy twice the loads in flight (same FMA order, same results).
// kPhase: 0 = every level in one launch; 1 = the inner levels only, with the slim shared
// layout (h rows and the pair table: no M, no leaf tile), so that at R > 64 two CTAs still
// share an SM while the walk is bound by the latency chain of each run; 2 = the leaf level
// alone (full layout), started from the level extents phase 1 left in the control words.
template <int kMinB, int kUn, int kPhase>
__global__ void __launch_bounds__(kWalkWarps * 32, kMinB)
walk_runs_kernel(const double *__restrict__ gm, const double *__restrict__ U, int64_t n, int R,
                 int leaf, int depth, int64_t row_lo,
                 const double *__restrict__ Mfull,
                 const uint32_t *__restrict__ pairs_g, const double *__restrict__ H,
                 double *__restrict__ rA, double *__restrict__ rB, int32_t *__restrict__ iA,
                 int32_t *__restrict__ iB, Run *runs,
                 int *ctl, int64_t cap_runs, int64_t *__restrict__ Xi, double *__restrict__ pmp,
                 double *__restrict__ resid, double *__restrict__ Hout, int *status,
                 unsigned long long *prof, const int32_t *__restrict__ leaf_rank,
                 int32_t *__restrict__ owner) {
  extern __shared__ double sh[];
  const int Rs = tri_stride(R);                    // even node stride (zero pad)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int Rn = mma_rn(R), Zs = mma_zs(R), Ms = mma_ms(R);
  const size_t bd = kPhase == 1 ? 0 : walk_block_doubles(R);
  double *Mp = sh;                                 // full M, zero-padded to Rn x Ms
  // R: the run's Hadamard row
  double *hv = sh + bd + (size_t)wid * (kPhase == 1 ? walk_per_warp_inner(R) : walk_per_warp(R));
  double *zb = hv + R;                             // leaf rows (.) h
  double *mass = zb + 8 * Zs;                      // leaf
  uint32_t *pairs = reinterpret_cast<uint32_t *>(
      sh + bd + (size_t)nw * (kPhase == 1 ? walk_per_warp_inner(R) : walk_per_warp(R)));
  if (kPhase != 2)
    for (int e = threadIdx.x; e < Rs; e += blockDim.x) pairs[e] = pairs_g[e];
  if (kPhase != 1)
    for (int e = threadIdx.x; e < Rn * Ms; e += blockDim.x) {
      const int k = e / Ms, c = e - k * Ms;
      // leaf masses sum only the k-tiles at or above an n-tile's diagonal block: blocks
      // above the diagonal carry 2 M (M is symmetric, like the nodes' packed M')
      Mp[e] = (k < R && c < R) ? ((k >> 3) < (c >> 3) ? 2.0 * Mfull[k * R + c] : Mfull[k * R + c]) : 0.0;
    }
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  // Level-synchronous: the runs of level l are [begin, end); their children go to level
  // l + 1 through that level's own counter, whose value is stable after the grid barrier.
  __shared__ int claim;
  __shared__ Stage stg;
#if RCP_WALK_PROF
  __shared__ unsigned long long fin_last, fin_first_inv;   // this CTA's warps, this level
#endif
#ifdef RCP_WALK_TRACE
  __shared__ unsigned long long ph_max[4];
  auto gtime = []() {
    unsigned long long x;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x));
    return x;
  };
#endif
  if (threadIdx.x == 0) stg.count = 0;
  int64_t begin = 0, end = min((int64_t)ld_volatile(&ctl[0]), cap_runs);
  int lvl0 = 0;
  if (kPhase == 2) {   // the leaf level's extent, as the inner levels' launch left it
    while (lvl0 < depth && end > begin) {
      const int64_t pushed_n = ld_volatile(&ctl[kGenBase + lvl0]);
      begin = end;
      end = min(end + pushed_n, cap_runs);
      ++lvl0;
    }
    if (lvl0 < depth) return;   // an inner level ended without runs (grid-uniform)
  }
  for (int lvl = lvl0; lvl <= (kPhase == 1 ? depth - 1 : depth) && end > begin; ++lvl) {
    int *gen_cnt = &ctl[kGenBase + lvl];
    // this CTA's runs begin + blockIdx.x + k gridDim.x (spread over the level), claimed one
    // by one by its warps
    if (threadIdx.x == 0) {
      claim = 0;
#if RCP_WALK_PROF
      fin_last = 0ull;
      fin_first_inv = 0ull;
#endif
#ifdef RCP_WALK_TRACE
      ph_max[0] = ph_max[1] = ph_max[2] = ph_max[3] = 0ull;
#endif
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) {   // level start time and run count
      unsigned long long tnow;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
      prof[2 * lvl] = tnow;
      prof[2 * lvl + 1] = (unsigned long long)(end - begin);
    }
    __syncthreads();
    while (true) {
      int tc = 0;
      if (lane == 0) tc = atomicAdd(&claim, 1);
      const int64_t t = begin + blockIdx.x + (int64_t)__shfl_sync(0xffffffffu, tc, 0) * gridDim.x;
      if (t >= end) {
#if RCP_WALK_PROF
        if (lane == 0) {   // this warp's finish time for the per-level record
          unsigned long long tnow;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
          atomicMax(&fin_last, tnow);
          atomicMax(&fin_first_inv, ~tnow);
        }
#endif
        break;
      }
#ifdef RCP_WALK_TRACE
      const unsigned long long tr0 = gtime();
#endif
      const Run run = runs[t];
      const int32_t lo = run.lo, hi = run.hi, level = lvl;
      const double *rs = (level & 1) ? rB : rA;
      const int32_t *is = (level & 1) ? iB : iA;
      const int32_t s0 = run.hrow;   // no dependent load of the run's first sample
#ifdef RCP_WALK_TRACE
      const unsigned long long tr1 = gtime();
#endif
      for (int c = lane; c < R; c += 32) hv[c] = H ? H[(int64_t)s0 * R + c] : 1.0;
      __syncwarp();
#ifdef RCP_WALK_TRACE
      const unsigned long long tr2 = gtime();
#endif
      if (kPhase != 2 && (kPhase == 1 || level < depth)) {
        // child masses <GM_child, h h^T> over the packed triangle, two positions per step
        // T = max(q_left, 0) / q_node (ref samplers.py:423-451).  q_node is inherited from
        // the parent by left children; right children and seeds compute it here, in the
        // same pass as q_left.
        const int64_t v = run.node;
        const double2 *GL = reinterpret_cast<const double2 *>(
            gm + ((1LL << (level + 1)) - 1 + 2 * v) * (int64_t)Rs);
        const double2 *GV = reinterpret_cast<const double2 *>(
            gm + ((1LL << level) - 1 + v) * (int64_t)Rs);
        const uint2 *PR = reinterpret_cast<const uint2 *>(pairs);
        const bool known = !isnan(run.qv);
        double qL = 0.0, qV = 0.0, qL2 = 0.0, qV2 = 0.0;
        const int n2 = Rs / 2;
        if (known) {
#pragma unroll (kUn)
          for (int e = lane; e < n2; e += 32) {
            const double2 gl = __ldg(GL + e);
            const uint2 ab = PR[e];
            const double h0 = hv[ab.x & 0xffffu] * hv[ab.x >> 16];
            const double h1 = hv[ab.y & 0xffffu] * hv[ab.y >> 16];
            qL = fma(gl.x, h0, qL);
            qL2 = fma(gl.y, h1, qL2);
          }
        } else {
#pragma unroll (kUn)
          for (int e = lane; e < n2; e += 32) {
            const double2 gl = __ldg(GL + e);
            const double2 gv = __ldg(GV + e);
            const uint2 ab = PR[e];
            const double h0 = hv[ab.x & 0xffffu] * hv[ab.x >> 16];
            const double h1 = hv[ab.y & 0xffffu] * hv[ab.y >> 16];
            qL = fma(gl.x, h0, qL);
            qL2 = fma(gl.y, h1, qL2);
            qV = fma(gv.x, h0, qV);
            qV2 = fma(gv.y, h1, qV2);
          }
        }
        qL = warp_sum(qL + qL2);
#ifdef RCP_WALK_TRACE
        const unsigned long long tr3 = gtime();
#endif
        const double qnode = known ? run.qv : warp_sum(qV + qV2);
        if (!(qnode > 0.0)) {
          fail_run(lo, hi, is, Xi, Hout, R, status, ctl, lane, owner);
          continue;
        }
        double T = (qL > 0.0 ? qL : 0.0) / qnode;
        T = fmin(fmax(T, 0.0), 1.0);
        // partition the run's samples into the children's ranges of the next level's
        // buffer (left from the front, right from the back), rescaling each residual
        double *rd = (level & 1) ? rA : rB;
        int32_t *id = (level & 1) ? iA : iB;
        int32_t nl = 0, nr = 0;
        const unsigned below = (1u << lane) - 1u;
        constexpr int kPU = 4;   // 32-sample groups with loads in flight per step
        for (int32_t q0 = lo; q0 < hi; q0 += 32 * kPU) {
          double rv[kPU];
          int32_t sv[kPU];
#pragma unroll
          for (int u = 0; u < kPU; ++u) {
            const int32_t q = q0 + 32 * u + lane;
            rv[u] = q < hi ? rs[q] : 0.0;
            sv[u] = q < hi ? is[q] : 0;
          }
#pragma unroll
          for (int u = 0; u < kPU; ++u) {
            const int32_t q = q0 + 32 * u + lane;
            const bool valid = q < hi;
            const bool right = rv[u] >= T;
            const unsigned ml = __ballot_sync(0xffffffffu, valid && !right);
            const unsigned mr = __ballot_sync(0xffffffffu, valid && right);
            if (valid) {
              const int32_t o =
                  right ? hi - 1 - (nr + __popc(mr & below)) : lo + nl + __popc(ml & below);
              rd[o] = rescale(rv[u], T, right);
              id[o] = sv[u];
            }
            nl += __popc(ml);
            nr += __popc(mr);
          }
        }
        const double unknown = __longlong_as_double(0x7ff8000000000000LL);
        if (nl > 0)
          push_child(runs, gen_cnt, end, cap_runs, status, stg, run, lo, lo + nl, T, false, qL, depth,
                     level, lane);
        if (nr > 0)
          push_child(runs, gen_cnt, end, cap_runs, status, stg, run, lo + nl, hi, T, true, unknown,
                     depth, level, lane);
#ifdef RCP_WALK_TRACE
        if (lane == 0) {
          const unsigned long long tr4 = gtime();
          atomicMax(&ph_max[0], tr1 - tr0);
          atomicMax(&ph_max[1], tr2 - tr1);
          atomicMax(&ph_max[2], tr3 - tr2);
          atomicMax(&ph_max[3], tr4 - tr3);
        }
#endif
        continue;
      }
      if (kPhase == 1) continue;   // (not reached: phase 1 ends above the leaf level)
      if (leaf_rank) {
        // ---- rank mode (the tree's leaves are ranks, ref samplers.py:423-451): every
        // sample of the run is finished by the rank owning the leaf; its residual and the
        // probability of its path go on to that rank's local search
        const int32_t p = leaf_rank[run.node];
        if (p < 0) {   // "walk branched into an empty padded subtree"
          fail_run(lo, hi, is, Xi, Hout, R, status, ctl, lane, owner);
          continue;
        }
        for (int32_t s = lo + lane; s < hi; s += 32) {
          const int32_t o = is[s];
          owner[o] = p;
          resid[o] = rs[s];
          pmp[o] = run.prob;
        }
        continue;
      }
      // ---- leaf block: masses z^T M' z of its rows z = u (.) h, then each sample's
      // inverse CDF
      const int64_t r0 = (int64_t)run.node * leaf;
      const int nrow = (int)min((int64_t)leaf, n - r0);
      const double rprob = run.prob;
      bool bad = nrow <= 0;
      double total_m = 0.0;
      if (!bad) {
        // 8-row tiles: Y = Z M' on the fp64 tensor cores (M' = the block upper triangle of M
        // with the off-diagonal blocks doubled: z'Mz over half the tile products),
        // mass_q = <Y_q, Z_q>
        const int row = lane >> 2, quad = lane & 3;
        for (int q0 = 0; q0 < nrow; q0 += 8) {
          const int nb = min(8, nrow - q0);
          for (int c = lane; c < 8 * Zs; c += 32) {
            const int j = c / Zs, col = c - j * Zs;
            zb[c] = (j < nb && col < R) ? U[(r0 + q0 + j) * R + col] * hv[col] : 0.0;
          }
          __syncwarp();
          const double *zr = zb + row * Zs;
          double msum = 0.0;
          for (int nt = 0; nt < Rn; nt += 8) {
            double c0 = 0.0, c1 = 0.0;
            for (int ks = 0; ks < nt + 8; ks += 4)   // k-tiles <= this n-tile (upper blocks of M')
              dmma_8x8x4(c0, c1, zr[ks + quad], Mp[(ks + quad) * Ms + nt + row]);
            msum = fma(c0, zr[nt + 2 * quad], msum);
            msum = fma(c1, zr[nt + 2 * quad + 1], msum);
          }
          msum += __shfl_xor_sync(0xffffffffu, msum, 1);
          msum += __shfl_xor_sync(0xffffffffu, msum, 2);
          if (quad == 0 && row < nb) mass[q0 + row] = msum > 0.0 ? msum : 0.0;
          __syncwarp();
        }
      }
      if (!bad) {
        if (lane == 0)
          for (int q = 0; q < nrow; ++q) total_m += mass[q];
        total_m = __shfl_sync(0xffffffffu, total_m, 0);
        bad = !(total_m > 0.0);
      }
      if (bad) {
        fail_run(lo, hi, is, Xi, Hout, R, status, ctl, lane, owner);
        continue;
      }
      // blocks of kLeafChunk samples: lanes pick rows, then (optionally) the warp writes the
      // folded Hadamard rows from the staged leaf rows z = u (.) h
      const bool zrows = nrow <= 8;   // zb holds every row of this leaf
      for (int32_t b0 = lo; b0 < hi; b0 += kLeafChunk) {
        const int32_t b1 = min(hi, b0 + kLeafChunk);
        for (int32_t s = b0 + lane; s < b1; s += 32) {
          const double target = rs[s] * total_m;
          double cdf = 0.0;
          int cnt = 0;
          for (int q = 0; q < nrow; ++q) {
            cdf += mass[q];
            if (cdf <= target) ++cnt;
          }
          const int choice = cnt < nrow - 1 ? cnt : nrow - 1;
          double cdf_at = 0.0;
          for (int q = 0; q <= choice; ++q) cdf_at += mass[q];
          const double picked = mass[choice];
          double ro = picked > 0.0 ? (target - (cdf_at - picked)) / picked : 0.0;
          ro = fmin(fmax(ro, 0.0), one_below());
          const int32_t o = is[s];
          Xi[o] = row_lo + r0 + choice;
          pmp[o] = rprob * (picked / total_m);
          if (resid) resid[o] = ro;
          if (Hout) {   // fold the chosen factor row into the sample's Hadamard row
            double *dst = Hout + (int64_t)o * R;
            if (zrows) {
              const double *z = zb + choice * Zs;
              for (int c = 0; c < R; ++c) dst[c] = z[c];
            } else {
              const double *u = U + (r0 + choice) * R;
              for (int c = 0; c < R; ++c) dst[c] = u[c] * hv[c];
            }
          }
        }
        __syncwarp();
      }
#if RCP_WALK_PROF
      if (lane == 0) atomicAdd(&ctl[2], hi - lo);
#endif
    }
    publish_children(runs, gen_cnt, end, cap_runs, status, stg);
#if RCP_WALK_PROF
    if (threadIdx.x == 0) {   // (publish_children synchronised the CTA)
      atomicMax(&prof[2 * (kMaxDepth + 2) + 2 * lvl], fin_last);
      atomicMax(&prof[2 * (kMaxDepth + 2) + 2 * lvl + 1], fin_first_inv);
#ifdef RCP_WALK_TRACE
      for (int q = 0; q < 4; ++q) atomicMax(&prof[4 * (kMaxDepth + 2) + 4 * lvl + q], ph_max[q]);
#endif
    }
#endif
    grid.sync();
    const int64_t pushed_n = ld_volatile(gen_cnt);
    begin = end;
    end = min(end + pushed_n, cap_runs);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long tnow;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
    prof[2 * (kMaxDepth + 1)] = tnow;
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

size_t walk_smem_inner(int R, int warps) {
  return sizeof(double) * ((size_t)warps * walk_per_warp_inner(R)) +
         sizeof(uint32_t) * (size_t)tri_stride(R) + 64;
}

size_t walk_smem(int R, int warps) {
  return sizeof(double) * (walk_block_doubles(R) + (size_t)warps * walk_per_warp(R)) +
         sizeof(uint32_t) * (size_t)tri_stride(R) + 64;
}

}  // namespace

extern "C" {

size_t rcp_sts_walk_ws_bytes(int64_t J, int64_t n, int leaf, int R) {
  if (R < 1 || R > RCP_MAX_RANK || leaf < 1) return 0;
  WalkWs w(J > 0 ? J : 1, rcp_sts_depth(n, leaf), R);
  return w.total;
}

}  // extern "C"

namespace {

int walk_gm_tables(const double *d_tree, const double *d_M, int R, int depth, double *Mp,
                   uint32_t *pairs, double *gm, cudaStream_t st) {
  walk_tables_kernel<<<(unsigned)ceil_div(tri_stride(R), 128), 128, 0, st>>>(d_M, R, Mp, pairs);
  RCP_LAUNCH_CHECK("walk_tables");
  const int Rs = tri_stride(R);
  const int64_t n2 = ((2LL << depth) - 1) * (int64_t)(Rs / 2);
  int64_t g = ceil_div(n2, 256);
  if (g > 8LL * sm_count()) g = 8LL * sm_count();
  walk_gm_kernel<<<(unsigned)g, 256, 0, st>>>(d_tree, (const double2 *)Mp, n2, Rs / 2,
                                               (double2 *)gm);
  RCP_LAUNCH_CHECK("walk_gm");
  return RCP_OK;
}

// The run-grouped walk.  d_leaf_rank != nullptr selects the rank mode: the tree's leaves are
// ranks (leaf = 1, n = P, no factor rows); every sample gets its owner, its residual and the
// probability of its path instead of a row.
int walk_impl(const double *d_tree, const double *d_U, int64_t n, int R, int leaf,
              int64_t row_lo, const double *d_M, const double *d_H_in, const int64_t *d_hkey,
              int key_bits, int64_t J, uint64_t key0, uint64_t key1, const uint64_t *d_key,
              const double *d_override,
              const double *d_rin, const int32_t *d_sel, int32_t sel_value, int64_t *d_Xi,
              double *d_pmp_i, double *d_resid, double *d_H_out, void *d_ws, size_t ws_bytes,
              int *d_status, const int32_t *d_leaf_rank, int32_t *d_owner,
              void *stream, bool gm_ready = false) {
  if (R < 1 || R > RCP_MAX_RANK || leaf < 1 || leaf > kMaxLeaf || J < 0 || n < 0 ||
      J >= (1LL << 31) || key_bits < 1)
    return RCP_ERR_ARG;
  if (key_bits > 64 || !d_hkey) key_bits = 64;
  if (J == 0) return RCP_OK;
  if (n == 0 || !d_tree || !d_M || !d_pmp_i || !d_ws) return RCP_ERR_ARG;
  if (d_leaf_rank) {
    if (!d_owner || !d_resid || leaf != 1) return RCP_ERR_ARG;
  } else if (!d_U || !d_Xi) {
    return RCP_ERR_ARG;
  }
  if (d_H_out && d_H_out == d_H_in) return RCP_ERR_ARG;   // groups read a shared row of H_in
  const int depth = rcp_sts_depth(n, leaf);
  if (depth > kMaxDepth) return RCP_ERR_ARG;
  WalkWs L(J, depth, R);
  if (ws_bytes < L.total) return RCP_ERR_ARG;
  int warps = kWalkWarps;
  while (warps > 1 && walk_smem(R, warps) > 200 * 1024) --warps;
  const size_t smem = walk_smem(R, warps);
  if (smem > 200 * 1024) return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  char *w = (char *)d_ws;
  int64_t *key = (int64_t *)(w + L.o_key), *key2 = (int64_t *)(w + L.o_key2);
  double *r = (double *)(w + L.o_r), *r2 = (double *)(w + L.o_r2);
  int32_t *idx = (int32_t *)(w + L.o_idx), *idx2 = (int32_t *)(w + L.o_idx2);
  Run *runs = (Run *)(w + L.o_runs);
  int *ctl = (int *)(w + L.o_ctl);
  double *Mp = (double *)(w + L.o_mp);
  uint32_t *pairs = (uint32_t *)(w + L.o_pairs);
  double *gm = (double *)(w + L.o_gm);
  void *cub_tmp = w + L.o_cub;
  const unsigned gb = (unsigned)ceil_div(J, 256);
  // no key and no selection: every sample is in one group, already "sorted"
  const bool one_group = !d_hkey && !d_sel;
  walk_prepare_kernel<<<gb, 256, 0, st>>>(d_hkey, J, d_sel, sel_value, one_group ? key2 : key,
                                          one_group ? idx2 : idx, ctl,
                                          (unsigned long long *)(w + L.o_prof));
  RCP_LAUNCH_CHECK("walk_prepare");
  // group samples by key (only the key's bits); level 0 holds their uniforms in that order
  int32_t *idx3 = (int32_t *)(w + L.o_idx3);
  size_t tb = L.cub_bytes;
  if (!one_group) {
    RCP_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, key, key2, idx, idx2, (int)J, 0,
                                                 key_bits, st));
    RCP_LAUNCH_CHECK("walk_sort_key");
  }
  walk_fill_r_kernel<<<gb, 256, 0, st>>>(idx2, J, key0, key1, d_key, d_override, d_rin, r);
  RCP_LAUNCH_CHECK("walk_fill_r");
  walk_seed_kernel<<<gb, 256, 0, st>>>(key2, idx2, J, d_sel ? d_pmp_i : nullptr, runs, ctl);
  RCP_LAUNCH_CHECK("walk_seed");
  // this walk's M' tables and G (.) M' for every node (unless rcp_sts_walk_gm made them)
  if (!gm_ready) {
    const int rc = walk_gm_tables(d_tree, d_M, R, depth, Mp, pairs, gm, st);
    if (rc != RCP_OK) return rc;
  }
  using WalkFn = void (*)(const double *, const double *, int64_t, int, int, int, int64_t, const double *,
                          const uint32_t *, const double *, double *, double *, int32_t *, int32_t *,
                          Run *, int *, int64_t, int64_t *, double *, double *, double *, int *,
                          unsigned long long *, const int32_t *, int32_t *);
  const WalkFn fn_all = walk_runs_kernel<RCP_WALK_MIN_BLOCKS, kWalkUnroll, 0>;
  const WalkFn fn_all_big = walk_runs_kernel<1, kWalkUnrollBig, 0>;
  const WalkFn fn_inner = walk_runs_kernel<RCP_WALK_MIN_BLOCKS, kWalkUnroll, 1>;
  const WalkFn fn_leaf = walk_runs_kernel<1, kWalkUnrollBig, 2>;
  static bool attr = false;
  if (!attr) {
    for (WalkFn f : {fn_all, fn_all_big, fn_inner, fn_leaf})
      RCP_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  // RCP_WALK_WIDE=0: never the wide-register / split variants (A/B runs)
  static const int wide_ok = [] {
    const char *e = getenv("RCP_WALK_WIDE");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  int per_sm = 0;
  RCP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn_all, warps * 32, smem));
  // Shared memory admits one CTA of the full layout per SM (R > 64): the inner levels run
  // as their own launch with the slim layout (two CTAs of 16 warps per SM again), the leaf
  // level after it with the full one.
  const bool split = wide_ok && per_sm <= 1 && depth >= 2;
  WalkFn fn = fn_all, fn2 = nullptr;
  int warps1 = warps;
  size_t smem1 = smem;
  if (split) {
    fn = fn_inner;
    fn2 = fn_leaf;
    warps1 = kWalkWarps;
    smem1 = walk_smem_inner(R, warps1);
  } else if (wide_ok && per_sm <= 1) {
    fn = fn_all_big;
  }
  RCP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, warps1 * 32, smem1));
  if (per_sm < 1) return RCP_ERR_ARG;
  // persistent: every CTA resident at once (workers wait on the shared queue)
  const int grid = per_sm * sm_count();
  // cooperative launch: every CTA co-resident, grid-wide barrier between tree levels
  const double *a_gm = gm, *a_U = d_U, *a_H = d_H_in, *a_Mf = d_M;
  const uint32_t *a_pairs = pairs;
  double *a_rA = r, *a_rB = r2;
  int32_t *a_iA = idx2, *a_iB = idx3;
  unsigned long long *a_prof = (unsigned long long *)(w + L.o_prof);
  int64_t a_n = n, a_row_lo = row_lo, a_cap = L.nruns;
  int a_R = R, a_leaf = leaf, a_depth = depth;
  void *args[] = {(void *)&a_gm, (void *)&a_U, (void *)&a_n, (void *)&a_R, (void *)&a_leaf,
                  (void *)&a_depth, (void *)&a_row_lo, (void *)&a_Mf,
                  (void *)&a_pairs,
                  (void *)&a_H, (void *)&a_rA, (void *)&a_rB, (void *)&a_iA, (void *)&a_iB,
                  (void *)&runs, (void *)&ctl,
                  (void *)&a_cap, (void *)&d_Xi, (void *)&d_pmp_i, (void *)&d_resid, (void *)&d_H_out,
                  (void *)&d_status, (void *)&a_prof, (void *)&d_leaf_rank, (void *)&d_owner};
  RCP_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)fn, dim3(grid),
                                           dim3(warps1 * 32), args, smem1, st));
  RCP_LAUNCH_CHECK("walk_runs");
  if (fn2) {
    int per_sm2 = 0;
    RCP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, fn2, warps * 32, smem));
    if (per_sm2 < 1) return RCP_ERR_ARG;
    RCP_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)fn2, dim3(per_sm2 * sm_count()),
                                             dim3(warps * 32), args, smem, st));
    RCP_LAUNCH_CHECK("walk_leaf");
  }
  return RCP_OK;
}

}  // namespace

extern "C" {

int rcp_sts_walk(const double *d_tree, const double *d_U, int64_t n, int R, int leaf,
                 int64_t row_lo, const double *d_M, const double *d_H_in, const int64_t *d_hkey,
                 int key_bits, int64_t J, uint64_t key0, uint64_t key1, const uint64_t *d_key,
                 const double *d_override,
                 const double *d_rin, const int32_t *d_sel, int32_t sel_value, int64_t *d_Xi,
                 double *d_pmp_i, double *d_resid, double *d_H_out, void *d_ws, size_t ws_bytes,
                 int *d_status,
                 void *stream) {
  return walk_impl(d_tree, d_U, n, R, leaf, row_lo, d_M, d_H_in, d_hkey, key_bits, J, key0, key1,
                   d_key, d_override, d_rin, d_sel, sel_value, d_Xi, d_pmp_i, d_resid, d_H_out, d_ws,
                   ws_bytes, d_status, nullptr, nullptr, stream);
}

// The walk's conditioning pass alone (M' tables and G (.) M' for every node, written into
// the walk workspace): depends only on the tree and M, so a caller can run it on another
// stream ahead of the walk (rcp_sts_walk_prepared) while earlier modes are still sampled.
int rcp_sts_walk_gm(const double *d_tree, int64_t n, int R, int leaf, const double *d_M, int64_t J,
                    void *d_ws, size_t ws_bytes, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || leaf < 1 || leaf > kMaxLeaf || J < 1 || n < 1 || !d_tree ||
      !d_M || !d_ws)
    return RCP_ERR_ARG;
  const int depth = rcp_sts_depth(n, leaf);
  if (depth > kMaxDepth) return RCP_ERR_ARG;
  WalkWs L(J, depth, R);
  if (ws_bytes < L.total) return RCP_ERR_ARG;
  char *w = (char *)d_ws;
  return walk_gm_tables(d_tree, d_M, R, depth, (double *)(w + L.o_mp), (uint32_t *)(w + L.o_pairs),
                        (double *)(w + L.o_gm), RCP_STREAM(stream));
}

// rcp_sts_walk on a workspace whose conditioning pass rcp_sts_walk_gm already made (same
// tree, M, J, n, leaf, R).
int rcp_sts_walk_prepared(const double *d_tree, const double *d_U, int64_t n, int R, int leaf,
                          int64_t row_lo, const double *d_M, const double *d_H_in,
                          const int64_t *d_hkey, int key_bits, int64_t J, uint64_t key0,
                          uint64_t key1, const uint64_t *d_key, const double *d_override,
                          const double *d_rin, const int32_t *d_sel, int32_t sel_value,
                          int64_t *d_Xi, double *d_pmp_i, double *d_resid, double *d_H_out,
                          void *d_ws, size_t ws_bytes, int *d_status, void *stream) {
  return walk_impl(d_tree, d_U, n, R, leaf, row_lo, d_M, d_H_in, d_hkey, key_bits, J, key0, key1,
                   d_key, d_override, d_rin, d_sel, sel_value, d_Xi, d_pmp_i, d_resid, d_H_out, d_ws,
                   ws_bytes, d_status, nullptr, nullptr, stream, true);
}

size_t rcp_sts_rank_walk_ws_bytes(int64_t J, int P, int R) {
  if (R < 1 || R > RCP_MAX_RANK || P < 1) return 0;
  WalkWs w(J > 0 ? J : 1, rcp_sts_depth(P, 1), R);
  return w.total;
}

// Rank-level walk of every sample over the packed rank tree (rcp_sts_rank_tree), grouped
// by the key of the modes already sampled like the local walk (ref samplers.py:423-451):
// owner, residual and path probability per sample.
int rcp_sts_rank_walk_grouped(const double *d_rank_tree, int P, const int32_t *d_leaf_rank,
                              int R, const double *d_M, const double *d_H_in,
                              const int64_t *d_hkey, int key_bits, int64_t J, uint64_t key0,
                              uint64_t key1, const uint64_t *d_key, const double *d_override,
                              int32_t *d_owner, double *d_r_out, double *d_pmp_i, void *d_ws,
                              size_t ws_bytes, int *d_status, void *stream) {
  if (P < 1 || !d_leaf_rank || !d_owner || !d_r_out) return RCP_ERR_ARG;
  return walk_impl(d_rank_tree, nullptr, P, R, 1, 0, d_M, d_H_in, d_hkey, key_bits, J, key0, key1,
                   d_key, d_override, nullptr, nullptr, 0, nullptr, d_pmp_i, d_r_out, nullptr, d_ws,
                   ws_bytes, d_status, d_leaf_rank, d_owner, stream);
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
