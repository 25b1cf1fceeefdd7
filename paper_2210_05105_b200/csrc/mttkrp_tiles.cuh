// Row-tile x fiber sampled MTTKRP (included by mttkrp.cu inside its anonymous namespace).
//
// The mode-k store is column-major (CSC analogue, ref matricization.py:67-128): the entries
// of one fiber are contiguous and their rows ascend.  Cutting the output rows into tiles of
// TR = 2^TS rows, the entries of a sampled fiber that fall in one tile are therefore one
// contiguous run of at most TR entries — a "pair" (tile, fiber).  Instead of transposing
// every gathered entry into row order (the reference's sparse transpose,
// mttkrp.py:131-155), this path moves only the pairs (8 bytes each, ~2-3 entries per pair at
// C3), and reads the entries straight from the store:
//
//   pass 1  tile_hist      per CTA, pairs per tile (CTA-private shared-memory histogram)
//   prefix  cta_prefix     per tile, exclusive prefix over CTAs + tile totals -> tptr
//   pass 2  pair_scatter   pairs written to their tile's range in a deterministic order
//   units   tile_units     tiles cut into parts of <= kTilePart pairs
//   spmm    tile_spmm      per part: 8 warps split its pairs; each warp keeps the tile's TR
//                          output rows in registers, loads the fiber's scaled KRP row Hs_d
//                          ONCE per pair and applies every entry of the pair to it
//                          (row selected by a warp-uniform switch); warps and parts are
//                          combined in a fixed order (no atomics on the output)
//
// Every order is a function of the input only, so results are bit-reproducible run to run
// (ref tests/test_mttkrp.py:60-67,163-172 require bit-identity across worker counts).
// Pair record: store position (36 bits) | count - 1 (6 bits) | distinct fiber id (22 bits).

#include "tile_apply_ptx.cuh"


constexpr int kTilePart = 2048;         // pairs per spmm part (4 warps x 512)
constexpr int kTileWarps = 4;
constexpr int kScatterItems = 1024;     // items per pair_scatter chunk (spans cached in smem)
constexpr int kTileMaxRowsShift = 5;    // TR <= 32: a pair's end is always inside the next window
constexpr int kTileMaxTiles = 4096;     // tiles per mode (tile_units scans them in one CTA)

__device__ __forceinline__ uint64_t pack_pair(int64_t pos, int cnt, int64_t d) {
  return ((uint64_t)pos << 28) | ((uint64_t)(cnt - 1) << 22) | (uint64_t)d;
}
__device__ __forceinline__ int64_t pair_pos(uint64_t p) { return (int64_t)(p >> 28); }
__device__ __forceinline__ int pair_cnt(uint64_t p) { return (int)((p >> 22) & 63u) + 1; }
__device__ __forceinline__ int pair_fib(uint64_t p) { return (int)(p & 0x3FFFFFu); }

// ---------------------------------------------------------------- deterministic dedup order
// Distinct fibers are numbered in the order of their representative (smallest) sample id,
// not in hash-slot order (which depends on the order of the CAS races in hash_insert).
__global__ void rep_flag_kernel(const int64_t *__restrict__ X, int N, int64_t J, int k, Strides st,
                                int64_t tmask, const unsigned long long *__restrict__ tkey,
                                const int32_t *__restrict__ trep, int64_t *__restrict__ flag,
                                int32_t *__restrict__ sslot) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  const unsigned long long key = (unsigned long long)sample_key(X, N, J, k, st, s);
  uint64_t h = mix64((uint64_t)key) & (uint64_t)tmask;
  while (tkey[h] != key) h = (h + 1) & (uint64_t)tmask;
  flag[s] = trep[h] == (int32_t)s ? 1 : 0;
  sslot[s] = (int32_t)h;
}

__global__ void rep_compact_kernel(const int64_t *__restrict__ flag, const int64_t *__restrict__ fpos,
                                   int64_t J, const int32_t *__restrict__ sslot,
                                   const unsigned long long *__restrict__ tkey,
                                   const int32_t *__restrict__ tcnt,
                                   const unsigned long long *__restrict__ twmin,
                                   const unsigned long long *__restrict__ twmax,
                                   const double *__restrict__ twsum, int64_t *__restrict__ dkey,
                                   int32_t *__restrict__ dcnt, int32_t *__restrict__ drep,
                                   double *__restrict__ dsc, int64_t *__restrict__ S) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s == 0) S[0] = fpos[J];
  if (s >= J || !flag[s]) return;
  const int64_t d = fpos[s];
  const int32_t h = sslot[s];
  dkey[d] = (int64_t)tkey[h];
  dcnt[d] = tcnt[h];
  drep[d] = (int32_t)s;
  dsc[d] = twmin[h] == twmax[h] ? (double)tcnt[h] * __longlong_as_double((long long)twmin[h]) : twsum[h];
}

// ---------------------------------------------------------------- pass 1: pairs per tile
// A warp loads all (<= kItemE / 32) windows of its item at once, then flags run starts.
constexpr int kItemWin = (int)(kItemE / 32);

constexpr int kPairThreads = 512;   // pair passes: 16 warps x 2 CTAs per SM

template <int TS>
__global__ void __launch_bounds__(kPairThreads, 2)
tile_hist_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                 const int32_t *__restrict__ ifib, const int64_t *__restrict__ dlo,
                 const int64_t *__restrict__ dlen, const int32_t *__restrict__ rows, int n_tiles,
                 int32_t *__restrict__ cmat) {
  extern __shared__ int32_t hist[];
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t it = i0 + wid; it < i1; it += nw) {
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    const int64_t fs = dlo[sp.d];
    int32_t t[kItemWin];
#pragma unroll
    for (int q = 0; q < kItemWin; ++q) {
      const int64_t pos = sp.a + 32 * q + lane;
      t[q] = pos < sp.b ? (rows[pos] >> TS) : -1;
    }
    const int32_t t0 = (lane == 0 && sp.a > fs) ? (rows[sp.a - 1] >> TS) : -1;
#pragma unroll
    for (int q = 0; q < kItemWin; ++q) {
      int32_t pt = __shfl_up_sync(0xffffffffu, t[q], 1);
      const int32_t last = q ? __shfl_sync(0xffffffffu, t[q ? q - 1 : 0], 31) : t0;
      if (lane == 0) pt = last;
      if (t[q] >= 0 && t[q] != pt) atomicAdd(&hist[t[q]], 1);
    }
  }
  __syncthreads();
  int32_t *mine = cmat + (int64_t)blockIdx.x * n_tiles;
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) mine[i] = hist[i];
}

// Block-wide exclusive scan of n <= 4 * blockDim.x int32 values in shared memory (in place);
// returns the total.  blockDim.x a multiple of 32, <= 1024.
__device__ int block_scan_excl(int32_t *a, int n) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t total;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  int32_t v[4], s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = 4 * t + q;
    v[q] = i < n ? a[i] : 0;
    s += v[q];
  }
  int32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    int32_t z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z - w;
    if (lane == 31) total = z;
  }
  __syncthreads();
  int32_t run = wsum[wid] + x - s;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = 4 * t + q;
    if (i < n) a[i] = run;
    run += v[q];
  }
  __syncthreads();
  return total;
}

// ---------------------------------------------------------------- pass 2: pair scatter
// The CTA's items are cut into units of up to kUnitWin consecutive 32-entry windows of one
// item; one unit per warp forms a batch.  Within a batch a tile receives at most one
// pair per unit (a fiber has one pair per tile), ranked by warp index through a per-tile
// bit mask; the batch order and the unit -> warp assignment are fixed, so every pair's slot
// is a function of the input only.  Item spans are cached in shared memory per chunk.
constexpr int kUnitWin = 4;

template <int TS>
__global__ void __launch_bounds__(kPairThreads, 2)
pair_scatter_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                    const int32_t *__restrict__ ifib, const int64_t *__restrict__ dlo,
                    const int64_t *__restrict__ dlen, const int32_t *__restrict__ rows,
                    int n_tiles, const int64_t *__restrict__ tptr,
                    const int32_t *__restrict__ cmat, uint64_t *__restrict__ pairs) {
  extern __shared__ int64_t smem_i64[];
  int64_t *cur = smem_i64;                                 // n_tiles
  int64_t *ia = cur + n_tiles;                             // item start   [kScatterItems]
  int64_t *ib = ia + kScatterItems;                        // item end
  int64_t *ifs = ib + kScatterItems;                       // fiber start
  int64_t *ife = ifs + kScatterItems;                      // fiber end
  uint32_t *mask = reinterpret_cast<uint32_t *>(ife + kScatterItems);   // n_tiles
  int32_t *idd = reinterpret_cast<int32_t *>(mask + n_tiles);          // fiber id
  int32_t *upre = idd + kScatterItems;                                  // kScatterItems + 1
  const int64_t S = Sp[0];
  int64_t i0, i1;
  cta_items(ioff[S], i0, i1);
  const int32_t *mine = cmat + (int64_t)blockIdx.x * n_tiles;
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
    cur[i] = tptr[i] + mine[i];
    mask[i] = 0u;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned below = (1u << wid) - 1u;
  constexpr int UE = 32 * kUnitWin;
  for (int64_t ci = i0; ci < i1; ci += kScatterItems) {
    const int ni = (int)min((int64_t)kScatterItems, i1 - ci);
    __syncthreads();
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
      const ItemSpan sp = item_span(ci + i, ioff, ifib, dlo, dlen);
      ia[i] = sp.a;
      ib[i] = sp.b;
      ifs[i] = dlo[sp.d];
      ife[i] = dlo[sp.d] + dlen[sp.d];
      idd[i] = (int32_t)sp.d;
      upre[i] = (int32_t)ceil_div(sp.b - sp.a, (int64_t)UE);
    }
    __syncthreads();
    const int nu = block_scan_excl(upre, ni);
    if (threadIdx.x == 0) upre[ni] = nu;
    __syncthreads();
    // unit loads for batch ub are issued before the barriers of batch ub - 32
    struct UnitLoad {
      int32_t t[kUnitWin + 1];
      int32_t tp;
      int64_t base, b, fs, fe;
      int32_t d;
      bool ok;
    };
    auto load_unit = [&](int u) {
      UnitLoad L;
      L.ok = u < nu;
      L.base = L.b = L.fs = L.fe = 0;
      L.d = 0;
      L.tp = -1;
#pragma unroll
      for (int v = 0; v <= kUnitWin; ++v) L.t[v] = INT_MAX;
      if (L.ok) {   // warp-uniform
        int lo = 0, hi = ni;   // largest i with upre[i] <= u
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (upre[mid] <= u) lo = mid; else hi = mid;
        }
        L.b = ib[lo];
        L.fs = ifs[lo];
        L.fe = ife[lo];
        L.d = idd[lo];
        L.base = ia[lo] + (int64_t)UE * (u - upre[lo]);
        // windows 0..kUnitWin-1 of the unit and one more (a run ends <= TR <= 32 later),
        // read to the fiber's end (past the item's end when needed)
#pragma unroll
        for (int v = 0; v <= kUnitWin; ++v) {
          const int64_t pos = L.base + 32 * v + lane;
          if (pos < L.fe) L.t[v] = rows[pos];
        }
        if (lane == 0 && L.base > L.fs) L.tp = rows[L.base - 1];
      }
      return L;
    };
    const int nwarp = (int)(blockDim.x >> 5);   // units per batch (one per warp)
    UnitLoad cu = load_unit(wid);
    for (int ub = 0; ub < nu; ub += nwarp) {
      unsigned own = 0u;        // bit v: this lane owns the pair starting in window v
      int32_t tl[kUnitWin];
      int cnt[kUnitWin];
      if (cu.ok) {   // warp-uniform
        int32_t t[kUnitWin + 1];
#pragma unroll
        for (int v = 0; v <= kUnitWin; ++v) t[v] = cu.t[v] == INT_MAX ? INT_MAX : (cu.t[v] >> TS);
        const int32_t tp = cu.tp < 0 ? -1 : (cu.tp >> TS);
        unsigned bnd[kUnitWin + 1], st[kUnitWin + 1];
#pragma unroll
        for (int v = 0; v <= kUnitWin; ++v) {
          const int64_t pos = cu.base + 32 * v + lane;
          int32_t pt = __shfl_up_sync(0xffffffffu, t[v], 1);
          const int32_t last = v ? __shfl_sync(0xffffffffu, t[v ? v - 1 : 0], 31) : tp;
          if (lane == 0) pt = last;
          const bool s_ = pos < cu.fe && t[v] != pt;
          st[v] = s_ ? 1u : 0u;
          bnd[v] = __ballot_sync(0xffffffffu, s_ || pos >= cu.fe);
        }
#pragma unroll
        for (int v = 0; v < kUnitWin; ++v) {
          const int64_t pos = cu.base + 32 * v + lane;
          tl[v] = t[v];
          cnt[v] = 0;
          if (st[v] && pos < cu.b) {
            const unsigned above = bnd[v] & ~((2u << lane) - 1u);
            const int64_t end = above ? cu.base + 32 * v + (__ffs(above) - 1)
                                      : cu.base + 32 * (v + 1) + (__ffs(bnd[v + 1]) - 1);
            cnt[v] = (int)(end - pos);
            own |= 1u << v;
            atomicOr(&mask[t[v]], 1u << wid);
          }
        }
      }
      const int64_t base = cu.base;
      const int32_t d = cu.d;
      cu = load_unit(ub + nwarp + wid);   // next batch's loads fly during the barriers
      __syncthreads();
      unsigned m[kUnitWin];
#pragma unroll
      for (int v = 0; v < kUnitWin; ++v) {
        m[v] = 0u;
        if (own >> v & 1u) {
          m[v] = mask[tl[v]];
          pairs[cur[tl[v]] + __popc(m[v] & below)] = pack_pair(base + 32 * v + lane, cnt[v], d);
        }
      }
      __syncthreads();
#pragma unroll
      for (int v = 0; v < kUnitWin; ++v)
        if ((own >> v & 1u) && (m[v] & below) == 0u) {   // the tile's lowest warp advances
          cur[tl[v]] += __popc(m[v]);
          mask[tl[v]] = 0u;
        }
      __syncthreads();
    }
  }
}

inline size_t pair_scatter_smem(int n_tiles) {
  return 12 * (size_t)n_tiles + (size_t)kScatterItems * (4 * 8 + 4) + 4 * (kScatterItems + 1);
}

// ---------------------------------------------------------------- work units
// Tile t is cut into ceil(n_t / kTilePart) parts (at least one: empty tiles still write
// their zero rows).  uoff[t] = first unit of tile t; sbase[t] = first scratch slot of a
// multi-part tile.  One CTA of 1024 threads, n_tiles <= 4096.
__global__ void __launch_bounds__(1024)
tile_units_kernel(const int64_t *__restrict__ tcnt, int n_tiles, int32_t *__restrict__ uoff,
                  int32_t *__restrict__ sbase) {
  __shared__ int32_t a[4096 + 1], b[4096 + 1];
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int32_t np = (int32_t)max((int64_t)1, ceil_div(tcnt[t], (int64_t)kTilePart));
    a[t] = np;
    b[t] = np > 1 ? np : 0;
  }
  __syncthreads();
  const int nu = block_scan_excl(a, n_tiles);
  const int ns = block_scan_excl(b, n_tiles);
  (void)ns;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    uoff[t] = a[t];
    sbase[t] = b[t];
  }
  if (threadIdx.x == 0) uoff[n_tiles] = nu;
}

// ---------------------------------------------------------------- per-tile SpMM
// Accumulator row g of the warp's tile: acc[g] += v * h (g warp-uniform), through the
// generated brx.idx jump table (tile_apply_ptx.cuh).
template <int TR, int NP>
__device__ __forceinline__ void tile_apply(double2 (&a)[TR][NP], int g, double v, const double2 (&h)[NP]);

template <>
__device__ __forceinline__ void tile_apply<16, 1>(double2 (&a)[16][1], int g, double v, const double2 (&h)[1]) {
  tile_apply_ptx_16_1(a[0][0].x, a[0][0].y, a[1][0].x, a[1][0].y, a[2][0].x, a[2][0].y, a[3][0].x, a[3][0].y,
                      a[4][0].x, a[4][0].y, a[5][0].x, a[5][0].y, a[6][0].x, a[6][0].y, a[7][0].x, a[7][0].y,
                      a[8][0].x, a[8][0].y, a[9][0].x, a[9][0].y, a[10][0].x, a[10][0].y, a[11][0].x, a[11][0].y,
                      a[12][0].x, a[12][0].y, a[13][0].x, a[13][0].y, a[14][0].x, a[14][0].y, a[15][0].x, a[15][0].y,
                      g, v, h[0].x, h[0].y);
}

template <>
__device__ __forceinline__ void tile_apply<8, 2>(double2 (&a)[8][2], int g, double v, const double2 (&h)[2]) {
  tile_apply_ptx_8_2(a[0][0].x, a[0][0].y, a[0][1].x, a[0][1].y, a[1][0].x, a[1][0].y, a[1][1].x, a[1][1].y,
                     a[2][0].x, a[2][0].y, a[2][1].x, a[2][1].y, a[3][0].x, a[3][0].y, a[3][1].x, a[3][1].y,
                     a[4][0].x, a[4][0].y, a[4][1].x, a[4][1].y, a[5][0].x, a[5][0].y, a[5][1].x, a[5][1].y,
                     a[6][0].x, a[6][0].y, a[6][1].x, a[6][1].y, a[7][0].x, a[7][0].y, a[7][1].x, a[7][1].y,
                     g, v, h[0].x, h[0].y, h[1].x, h[1].y);
}

// Per-warp ring of kTileRing pair slots filled by cp.async: the fiber's scaled KRP row (the
// lane's column pairs) and the pair's rows and values.  Pair i + kTileRing is requested while
// pair i is applied, so every warp keeps kTileRing pairs' loads in flight.
// Per-warp ring of 2 x BS pair slots filled by cp.async, BS pairs per batch: batch b + 1 is
// requested while batch b is applied.  Each pair is requested by 32 / BS lanes of its own
// (the lanes split its Hs row's 16-byte chunks and its entries), so issuing a batch costs a
// few instructions per pair.  Slot: the fiber's scaled KRP row (512 NP bytes), then one
// 16-byte record {value, row} per entry.
template <int TR, int NP>
struct TileSlotLayout {
  static constexpr int BS = NP == 1 ? 8 : 4;        // pairs per batch
  static constexpr int LPP = 32 / BS;               // lanes per pair
  static constexpr uint32_t E = 512u * NP;          // entry records
  static constexpr uint32_t bytes = E + 16u * (TR + 1);   // +1: the loop reads one record ahead
};

__device__ __forceinline__ void cpa16_u32(uint32_t s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cpa8_u32(uint32_t s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cpa4_u32(uint32_t s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t s) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(s) : "memory");
  return v;
}

template <int TS, int NP>
constexpr size_t tile_spmm_smem() {
  using SL = TileSlotLayout<(1 << TS), NP>;
  constexpr size_t ring = (size_t)kTileWarps * 2 * SL::BS * SL::bytes;
  constexpr size_t red = (size_t)kTileWarps * (1 << TS) * 32 * NP * sizeof(double2);
  return ring > red ? ring : red;
}

template <int TS, int NP>
__global__ void __launch_bounds__(kTileWarps * 32, 4)
tile_spmm_kernel(const int64_t *__restrict__ tptr, int n_tiles, int64_t n_rows,
                 const int32_t *__restrict__ uoff, const int32_t *__restrict__ sbase,
                 const uint64_t *__restrict__ pairs, const int32_t *__restrict__ rows,
                 const double *__restrict__ vals, const double *__restrict__ Hs, int R,
                 double *__restrict__ out, double2 *__restrict__ scratch,
                 int32_t *__restrict__ tile_done, uint32_t *__restrict__ tile_mask,
                 int64_t *__restrict__ stats) {
  constexpr int TR = 1 << TS;
  constexpr int W = 32 * NP;   // double2 columns per row
  using SL = TileSlotLayout<TR, NP>;
  constexpr int BS = SL::BS, LPP = SL::LPP;
  constexpr uint32_t kSlot = SL::bytes, kSlotE = SL::E;
  extern __shared__ __align__(16) unsigned char tsm[];
  double2 *red = reinterpret_cast<double2 *>(tsm);                 // [kTileWarps][TR][W]
  __shared__ uint32_t s_mask;
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t ring_u32 = (uint32_t)__cvta_generic_to_shared(tsm) + (uint32_t)(wid * 2 * BS) * kSlot;
  const int Rp2 = hs_stride(R) >> 1;
  const double2 *H2 = reinterpret_cast<const double2 *>(Hs);
  const int U = uoff[n_tiles];
  unsigned long long hit_total = 0;
  if (threadIdx.x == 0) s_mask = 0u;
  __syncthreads();
  for (int u = blockIdx.x; u < U; u += gridDim.x) {
    int lo = 0, hi = n_tiles;   // tile: largest t with uoff[t] <= u
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (uoff[mid] <= u) lo = mid; else hi = mid;
    }
    const int t = lo;
    const int part = u - uoff[t], nparts = uoff[t + 1] - uoff[t];
    const int64_t p0 = tptr[t], p1 = tptr[t + 1];
    const int64_t per = ceil_div(p1 - p0, (int64_t)nparts);
    const int64_t a = p0 + part * per, b = min(a + per, p1);
    const int64_t wper = ceil_div(b - a, (int64_t)kTileWarps);
    const int64_t wa = min(a + wid * wper, b), wb = min(wa + wper, b);
    const int n = (int)(wb - wa);
    double2 acc[TR][NP];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[r][j] = make_double2(0.0, 0.0);
    uint32_t hmask = 0u;
    // lane -> (pair jp of the batch, sub-lane sub): the lane requests the pair's 16-byte
    // Hs chunks sub, sub + LPP, ... and its entries sub, sub + LPP, ...
    const int jp = lane / LPP, sub = lane % LPP;
    const int nch = (R + 1) >> 1;                                   // 16-byte chunks per row
    const int nb = (int)ceil_div((int64_t)n, (int64_t)BS);
    int cnt_nx = 0, cnt_cu = 0;   // this lane's pair count in the requested / applied batch
    // Pair records come from registers: rc holds the records of 32-pair group g0, rn of
    // group g0 + 1 (loaded a group ahead).  The store entries of batch bi + kPF are
    // prefetched into L2 while batch bi + 1 is copied, so the copies hit L2.
    constexpr int kPF = 3;
    int g0 = 0;
    uint64_t rc = lane < n ? pairs[wa + lane] : 0ull;
    uint64_t rn = 32 + lane < n ? pairs[wa + 32 + lane] : 0ull;
    auto rec_of = [&](int ip) {   // ip in [32 g0, 32 g0 + 64)
      const uint64_t x = __shfl_sync(0xffffffffu, rc, ip & 31);
      const uint64_t y = __shfl_sync(0xffffffffu, rn, ip & 31);
      return (ip >> 5) == g0 ? x : y;
    };
    auto issue = [&](int bi) {
      if (bi * BS >= 32 * (g0 + 1)) {   // warp-uniform: advance the record window
        ++g0;
        rc = rn;
        rn = 32 * (g0 + 1) + lane < n ? pairs[wa + 32 * (g0 + 1) + lane] : 0ull;
      }
      const int ip = bi * BS + jp;
      const uint64_t pr = rec_of(ip);
      const int ipf = (bi + kPF) * BS + jp;
      const uint64_t pf = rec_of(ipf);
      const uint32_t sl = ring_u32 + (uint32_t)((bi & 1) * BS + jp) * kSlot;
      int c = 0;
      if (ip < n) {
        c = pair_cnt(pr);
        const double2 *hs = H2 + (int64_t)pair_fib(pr) * Rp2;
#pragma unroll
        for (int q = 0; q < 32 * NP / LPP; ++q) {
          const int ch = q * LPP + sub;
          if (ch < nch) cpa16_u32(sl + 16u * ch, hs + ch);
        }
        const int64_t pe = pair_pos(pr);
        for (int e = sub; e < c; e += LPP) {
          cpa8_u32(sl + kSlotE + 16u * e, vals + pe + e);
          cpa4_u32(sl + kSlotE + 16u * e + 8u, rows + pe + e);
        }
      }
      if (ipf < n && sub < 2) {
        const int64_t pe = pair_pos(pf);
        if (sub == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(vals + pe));
        else asm volatile("prefetch.global.L2 [%0];" ::"l"(rows + pe));
      }
      cpa_commit();
      return c;
    };
    if (nb > 0) cnt_nx = issue(0);
    for (int bi = 0; bi < nb; ++bi) {
      cnt_cu = cnt_nx;
      cnt_nx = bi + 1 < nb ? issue(bi + 1) : (cpa_commit(), 0);
      cpa_wait<1>();
      __syncwarp();
      const uint32_t base = ring_u32 + (uint32_t)((bi & 1) * BS) * kSlot;
      const int np_ = min(BS, n - bi * BS);
      for (int j = 0; j < np_; ++j) {
        const uint32_t sl = base + (uint32_t)j * kSlot;
        double2 h[NP];
#pragma unroll
        for (int jj = 0; jj < NP; ++jj) h[jj] = lds_f64x2(sl + 16u * lane + 512u * jj);
        const int c = __shfl_sync(0xffffffffu, cnt_cu, j * LPP);
        uint32_t ea = sl + kSlotE;
        double2 rec = lds_f64x2(ea);   // the next record is loaded before this one's branch
        for (int e = 0; e < c; ++e) {
          ea += 16u;
          const double2 nx = lds_f64x2(ea);   // (past the last entry: unused slot bytes)
          const int g = __double2loint(rec.y) & (TR - 1);
          hmask |= 1u << g;
          tile_apply<TR, NP>(acc, g, rec.x, h);
          rec = nx;
        }
      }
      __syncwarp();
    }
    cpa_wait<0>();
    __syncthreads();   // every warp is done with its ring: the area becomes the reduction buffer
    // fixed-order combine of the warps' partial tiles
    double2 *mine = red + (size_t)wid * TR * W;
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int j = 0; j < NP; ++j) mine[r * W + lane + 32 * j] = acc[r][j];
    if (lane == 0 && hmask) atomicOr(&s_mask, hmask);
    __syncthreads();
    const int64_t row0 = (int64_t)t * TR;
    double2 *slot = nparts > 1 ? scratch + ((size_t)sbase[t] + part) * TR * W : nullptr;
    for (int i = threadIdx.x; i < TR * W; i += blockDim.x) {
      double2 s = red[i];
#pragma unroll
      for (int w = 1; w < kTileWarps; ++w) {
        const double2 x = red[(size_t)w * TR * W + i];
        s.x += x.x;
        s.y += x.y;
      }
      if (slot) {
        __stcg(slot + i, s);
      } else {
        const int64_t row = row0 + i / W;
        const int c = 2 * (i % W);
        if (row < n_rows && c < R) {
          out[row * R + c] = s.x;
          if (c + 1 < R) out[row * R + c + 1] = s.y;
        }
      }
    }
    if (nparts == 1) {
      if (threadIdx.x == 0) hit_total += __popc(s_mask);
    } else {
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        atomicOr(&tile_mask[t], s_mask);
        s_last = atomicAdd(&tile_done[t], 1) == nparts - 1;
      }
      __syncthreads();
      if (s_last) {   // the last part to finish sums every part in part order
        __threadfence();
        const double2 *base = scratch + (size_t)sbase[t] * TR * W;
        for (int i = threadIdx.x; i < TR * W; i += blockDim.x) {
          double2 s = __ldcg(base + i);
          for (int q = 1; q < nparts; ++q) {
            const double2 x = __ldcg(base + (size_t)q * TR * W + i);
            s.x += x.x;
            s.y += x.y;
          }
          const int64_t row = row0 + i / W;
          const int c = 2 * (i % W);
          if (row < n_rows && c < R) {
            out[row * R + c] = s.x;
            if (c + 1 < R) out[row * R + c + 1] = s.y;
          }
        }
        if (threadIdx.x == 0) {
          hit_total += __popc(atomicExch(&tile_mask[t], 0u));
          tile_done[t] = 0;
        }
      }
    }
    if (threadIdx.x == 0) s_mask = 0u;
    __syncthreads();
  }
  if (threadIdx.x == 0 && hit_total) atomicAdd((unsigned long long *)&stats[4], hit_total);
}

// ---------------------------------------------------------------- many row tiles
// Modes with more than kTileMaxTiles row tiles (C4/C5 factor modes: 10^5..10^6 tiles): the
// pairs are emitted per item in item order (count, scan, emit: fiber order, ascending tile
// inside a fiber), then stably radix-sorted by tile -- inside a tile they stay in fiber
// order, the same canonical order as the CTA-histogram passes produce -- and the tile
// pointers are found by binary search in the sorted tiles.
template <int TS>
__global__ void pair_count_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                                  const int32_t *__restrict__ ifib, const int64_t *__restrict__ dlo,
                                  const int64_t *__restrict__ dlen, const int32_t *__restrict__ rows,
                                  int64_t *__restrict__ icnt, int64_t *__restrict__ nit) {
  const int64_t n_items = ioff[Sp[0]];
  if (blockIdx.x == 0 && threadIdx.x == 0) nit[0] = n_items;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < n_items; it += nw) {
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    const int64_t fs = dlo[sp.d];
    int64_t c = 0;
    for (int64_t base = sp.a; base < sp.b; base += 32) {
      const int64_t pos = base + lane;
      const int32_t t = pos < sp.b ? (rows[pos] >> TS) : -1;
      int32_t pt = __shfl_up_sync(0xffffffffu, t, 1);
      if (lane == 0) pt = pos > fs ? (rows[pos - 1] >> TS) : -1;
      c += __popc(__ballot_sync(0xffffffffu, pos < sp.b && (pos == fs || t != pt)));
    }
    if (lane == 0) icnt[it] = c;
  }
}

template <int TS>
__global__ void pair_emit_kernel(const int64_t *__restrict__ ioff, const int64_t *__restrict__ Sp,
                                 const int32_t *__restrict__ ifib, const int64_t *__restrict__ dlo,
                                 const int64_t *__restrict__ dlen, const int32_t *__restrict__ rows,
                                 const int64_t *__restrict__ ipos, uint32_t *__restrict__ tkeys,
                                 uint64_t *__restrict__ pairs) {
  const int64_t n_items = ioff[Sp[0]];
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned below = (1u << lane) - 1u;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < n_items; it += nw) {
    const ItemSpan sp = item_span(it, ioff, ifib, dlo, dlen);
    const int64_t fs = dlo[sp.d], fe = fs + dlen[sp.d];
    int64_t o = ipos[it];
    for (int64_t base = sp.a; base < sp.b; base += 32) {
      const int64_t pos = base + lane;
      // this window and the next (a run ends at most TR <= 32 entries later), to the fiber end
      const int32_t t1 = pos < fe ? (rows[pos] >> TS) : INT_MAX;
      const int32_t t2 = pos + 32 < fe ? (rows[pos + 32] >> TS) : INT_MAX;
      int32_t p1 = __shfl_up_sync(0xffffffffu, t1, 1);
      if (lane == 0) p1 = pos > fs ? (rows[pos - 1] >> TS) : -1;
      int32_t p2 = __shfl_up_sync(0xffffffffu, t2, 1);
      const int32_t last1 = __shfl_sync(0xffffffffu, t1, 31);
      if (lane == 0) p2 = last1;
      const bool s1 = pos < fe && t1 != p1;
      const bool s2 = pos + 32 < fe && t2 != p2;
      const unsigned b1 = __ballot_sync(0xffffffffu, s1 || pos >= fe);
      const unsigned b2 = __ballot_sync(0xffffffffu, s2 || pos + 32 >= fe);
      const bool own = s1 && pos < sp.b;
      const unsigned m = __ballot_sync(0xffffffffu, own);
      if (own) {
        const unsigned above = b1 & ~((2u << lane) - 1u);
        const int64_t end = above ? base + (__ffs(above) - 1) : base + 32 + (__ffs(b2) - 1);
        const int64_t q = o + __popc(m & below);
        tkeys[q] = (uint32_t)t1;
        pairs[q] = pack_pair(pos, (int)(end - pos), sp.d);
      }
      o += __popc(m);
    }
  }
}

// tptr[t] = first pair of tile t in the tile-sorted pairs (t = 0..n_tiles)
__global__ void tile_bounds_kernel(const uint32_t *__restrict__ tkeys, const int64_t *__restrict__ np,
                                   int64_t n_tiles, int64_t *__restrict__ tptr) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > n_tiles) return;
  int64_t lo = 0, hi = np[0];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)tkeys[mid] < t) lo = mid + 1; else hi = mid;
  }
  tptr[t] = lo;
}

// Per tile: parts (>= 1) and multi-part parts, as int64 counts for the scans.
__global__ void tile_parts_kernel(const int64_t *__restrict__ tptr, int64_t n_tiles,
                                  int64_t *__restrict__ up, int64_t *__restrict__ sp) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const int64_t np = max((int64_t)1, ceil_div(tptr[t + 1] - tptr[t], (int64_t)kTilePart));
  up[t] = np;
  sp[t] = np > 1 ? np : 0;
}

__global__ void tile_parts_i32_kernel(const int64_t *__restrict__ uo, const int64_t *__restrict__ so,
                                      int64_t n_tiles, int32_t *__restrict__ uoff,
                                      int32_t *__restrict__ sbase) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > n_tiles) return;
  uoff[t] = (int32_t)uo[t];
  if (t < n_tiles) sbase[t] = (int32_t)so[t];
}

// ---------------------------------------------------------------- ordered sample weights
// Deterministic mode: a distinct fiber whose samples carry unequal weights (an injected batch;
// sampler output has equal weights, whose merged weight count * w^2 is exact) gets its sum
// of w^2 in sample order instead of the hash table's atomic sum.
__global__ void sample_fiber_kernel(const int32_t *__restrict__ sslot, const int32_t *__restrict__ trep,
                                    const int64_t *__restrict__ fpos, int64_t J,
                                    uint32_t *__restrict__ key, uint32_t *__restrict__ val) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  key[s] = (uint32_t)fpos[trep[sslot[s]]];
  val[s] = (uint32_t)s;
}

__global__ void fiber_start_kernel(const uint32_t *__restrict__ key, int64_t J,
                                   int32_t *__restrict__ start) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= J) return;
  if (i == 0 || key[i] != key[i - 1]) start[key[i]] = (int32_t)i;
}

__global__ void ordered_w2_kernel(const int64_t *__restrict__ Sp, const int32_t *__restrict__ start,
                                  const int32_t *__restrict__ dcnt, const uint32_t *__restrict__ val,
                                  const double *__restrict__ w, const int32_t *__restrict__ drep,
                                  const int32_t *__restrict__ sslot,
                                  const unsigned long long *__restrict__ twmin,
                                  const unsigned long long *__restrict__ twmax,
                                  double *__restrict__ dsc) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= Sp[0]) return;
  const int32_t h = sslot[drep[d]];
  if (twmin[h] == twmax[h]) return;   // equal weights: count * w^2 already exact
  double s = 0.0;
  const int32_t b = start[d], e = b + dcnt[d];
  for (int32_t i = b; i < e; ++i) {
    const double x = w[val[i]];
    s = fma(x, x, s);
  }
  dsc[d] = s;
}
