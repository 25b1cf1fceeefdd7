// Deterministic sampled MTTKRP (included by mttkrp.cu inside its anonymous namespace).
//
// The mode-k store is column-major (CSC analogue, ref matricization.py:67-128): the entries
// of one fiber are contiguous and their rows ascend.  Cutting the output rows into tiles of
// TR = 2^TS rows, the entries of a sampled fiber that fall in one tile are one contiguous
// run of at most TR entries -- a "pair" (tile, fiber).  The deterministic mode orders the
// pairs canonically (by tile, then by fiber) and derives every later order from that one:
//
//   pairs   <= 4096 tiles: tile_hist (pairs per (CTA, tile)) -> cta_prefix -> pair_scatter
//           (slots from per-tile warp masks in fixed batches);  more tiles: pair_count ->
//           scan -> pair_emit (item order) -> stable radix sort by tile
//   entries tile_entries + scan (entry offset of every tile); 32-pair chunks: chunk_rows
//           (entries per row) -> tile_rowscan (each chunk's slot per row, stable) ->
//           chunk_write: row-sorted entries, pair order inside a row
//   spmm    the fast path's segmented SpMM, except that rows split across its chunks leave
//           per-chunk partials which spmm_fix sums in chunk order (no red.add)
//
// Every order is a function of the input only, so results are bit-reproducible run to run
// (ref tests/test_mttkrp.py:60-67,163-172 require bit-identity across worker counts).
// Pair record: store position (36 bits) | count - 1 (6 bits) | distinct fiber id (22 bits).

constexpr int kScatterItems = 1024;     // items per pair_scatter chunk (spans cached in smem)
constexpr int kTileMaxTiles = 4096;     // CTA-private tile histograms up to this many tiles

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

// ---------------------------------------------------------------- canonical row order
// The deterministic mode's pairs (tile order, fiber order inside a tile) expanded into the
// row-sorted entries of the segmented SpMM: per tile a stable counting sort by row, so the
// entries of a row keep pair order.  The SpMM then combines rows split across its chunks
// in chunk order (spmm_packed_kernel<NP, true> + spmm_fix_kernel) instead of red.add.
__global__ void tile_entries_kernel(const int64_t *__restrict__ tptr, int64_t n_tiles,
                                    const uint64_t *__restrict__ pairs, int64_t *__restrict__ te) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += nw) {
    int64_t c = 0;
    for (int64_t p = tptr[t] + lane; p < tptr[t + 1]; p += 32) c += pair_cnt(pairs[p]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) te[t] = c;
  }
}

// Rows the deterministic SpMM split across chunks: their chunk partials summed in chunk order.
template <int NP>
__global__ void spmm_fix_kernel(const int64_t *__restrict__ rptr, int64_t n_rows,
                                const double2 *__restrict__ slotF, const double2 *__restrict__ slotL,
                                int R, double *__restrict__ out) {
  constexpr int CH = kSpmmChunk;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    const int64_t rs = rptr[r], re = rptr[r + 1];
    if (re <= rs) continue;
    const int64_t c0 = rs / CH, c1 = (re - 1) / CH;
    if (c0 == c1) continue;   // whole in one chunk: stored by the SpMM
    double2 s[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) s[j] = make_double2(0.0, 0.0);
    for (int64_t c = c0; c <= c1; ++c) {
      const double2 *sl = (rs < c * CH ? slotF : slotL) + c * (32 * NP);
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const double2 v = sl[lane + 32 * j];
        s[j].x += v.x;
        s[j].y += v.y;
      }
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int c = 2 * (lane + 32 * j);
      if (c < R) {
        out[r * R + c] = s[j].x;
        if (c + 1 < R) out[r * R + c + 1] = s[j].y;
      }
    }
  }
}

// Parallel form of the expansion: 32-pair chunks of each tile (one warp each) count their
// entries per row, a per-tile pass turns the counts into each chunk's slot per row (chunk
// order = pair order: stable), and the chunks write their entries.
__global__ void tile_chunks_kernel(const int64_t *__restrict__ tptr, int64_t n_tiles,
                                   int64_t *__restrict__ nch) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n_tiles) nch[t] = ceil_div(tptr[t + 1] - tptr[t], (int64_t)32);
}

__device__ __forceinline__ int64_t chunk_tile(const int64_t *__restrict__ choff, int64_t n_tiles,
                                              int64_t c) {
  int64_t lo = 0, hi = n_tiles;   // largest t with choff[t] <= c
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (choff[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

template <int TS>
__global__ void chunk_rows_kernel(const int64_t *__restrict__ tptr, const int64_t *__restrict__ choff,
                                  int64_t n_tiles, const uint64_t *__restrict__ pairs,
                                  const int32_t *__restrict__ rows, int64_t *__restrict__ cc) {
  constexpr int TR = 1 << TS;
  const int lane = threadIdx.x & 31;
  const int64_t n_ch = choff[n_tiles];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < n_ch; c += nw) {
    const int64_t t = chunk_tile(choff, n_tiles, c);
    const int64_t p = tptr[t] + 32 * (c - choff[t]) + lane;
    uint32_t m = 0;
    if (p < tptr[t + 1]) {
      const uint64_t pr = pairs[p];
      const int64_t pos = pair_pos(pr);
      const int cn = pair_cnt(pr);
      for (int e = 0; e < cn; ++e) m |= 1u << (rows[pos + e] & (TR - 1));
    }
    int mine = 0;
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int n = __popc(__ballot_sync(0xffffffffu, (m >> r) & 1u));
      if (lane == r) mine = n;
    }
    if (lane < TR) cc[c * TR + lane] = mine;
  }
}

// Per tile (warp): row r's chunks' counts -> their absolute first slots; row pointers.
template <int TS>
__global__ void tile_rowscan_kernel(const int64_t *__restrict__ choff, int64_t n_tiles, int64_t n_rows,
                                    const int64_t *__restrict__ eoff, int64_t *__restrict__ cc,
                                    int64_t *__restrict__ rptr, int64_t *__restrict__ stats) {
  constexpr int TR = 1 << TS;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long hit = 0;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += nw) {
    const int64_t c0 = choff[t], c1 = choff[t + 1];
    int64_t tot = 0;   // lane r: entries of row r in the tile
    if (lane < TR)
      for (int64_t c = c0; c < c1; ++c) tot += cc[c * TR + lane];
    int64_t x = lane < TR ? tot : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    int64_t run = eoff[t] + x - (lane < TR ? tot : 0);
    const int64_t row = t * TR + lane;
    if (lane < TR && row < n_rows) rptr[row] = run;
    if (lane < TR && row == n_rows - 1) rptr[n_rows] = run + tot;
    hit += __popc(__ballot_sync(0xffffffffu, lane < TR && tot > 0));
    if (lane < TR)
      for (int64_t c = c0; c < c1; ++c) {
        const int64_t v = cc[c * TR + lane];
        cc[c * TR + lane] = run;
        run += v;
      }
  }
  if (lane == 0 && hit) atomicAdd((unsigned long long *)&stats[4], hit);
}

template <int TS>
__global__ void chunk_write_kernel(const int64_t *__restrict__ tptr, const int64_t *__restrict__ choff,
                                   int64_t n_tiles, const uint64_t *__restrict__ pairs,
                                   const int32_t *__restrict__ rows, const double *__restrict__ vals,
                                   const int64_t *__restrict__ cc, double2 *__restrict__ ent) {
  constexpr int TR = 1 << TS;
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const int64_t n_ch = choff[n_tiles];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < n_ch; c += nw) {
    const int64_t t = chunk_tile(choff, n_tiles, c);
    const int64_t p = tptr[t] + 32 * (c - choff[t]) + lane;
    uint32_t m = 0;
    int64_t pos = 0;
    int d = 0;
    if (p < tptr[t + 1]) {
      const uint64_t pr = pairs[p];
      pos = pair_pos(pr);
      d = pair_fib(pr);
      const int cn = pair_cnt(pr);
      for (int e = 0; e < cn; ++e) m |= 1u << (rows[pos + e] & (TR - 1));
    }
    const int64_t mybase = lane < TR ? cc[c * TR + lane] : 0;
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const bool has = (m >> r) & 1u;
      const unsigned b = __ballot_sync(0xffffffffu, has);
      const int64_t base = __shfl_sync(0xffffffffu, mybase, r);
      if (has) {
        const int e = __popc(m & ((1u << r) - 1u));
        ent[base + __popc(b & below)] = make_double2(__longlong_as_double((long long)d), vals[pos + e]);
      }
    }
  }
}
