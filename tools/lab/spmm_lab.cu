// Experiment harness (not product code): variants of the sampled-MTTKRP segmented SpMM,
// run on the workspace a real rcp_sampled_mttkrp call left behind.  Built by
// tools/lab/run_lab.py into tools/lab/libspmm_lab.so together with the product sources.
#include "../../paper_2210_05105_b200/csrc/mttkrp.cu"

namespace {

// load policies for the Hs-row gather
template <int P>
__device__ __forceinline__ double2 ldh(const double2 *p) {
  if constexpr (P == 0) {
    return *p;
  } else if constexpr (P == 1) {
    return __ldcg(p);
  } else if constexpr (P == 2) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
  } else if constexpr (P == 3) {
    return __ldg(p);
  } else {
    double2 r;
    asm("ld.global.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
  }
}

template <int NP, int P, int U>
__global__ void __launch_bounds__(256)
lab_spmm_kernel(const int64_t *__restrict__ rptr, int64_t n_rows, const int64_t *__restrict__ nnzp,
                const double2 *__restrict__ ent, const double *__restrict__ Hs, int R,
                double *__restrict__ out) {
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
    int64_t row = floor_index(rptr, n_rows + 1, c0);
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
        while (base + q >= re) {
          flush();
          ++row;
          rs = re;
          re = rptr[row + 1];
        }
        const int run = (int)min((int64_t)(nb - q), re - (base + q));
        int t = 0;
        for (; t + U <= run; t += U) {
          int dq[U];
          double vq[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            dq[u] = __shfl_sync(0xffffffffu, md, q + t + u);
            vq[u] = __shfl_sync(0xffffffffu, mv, q + t + u);
          }
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            const int c2 = lane + 32 * j;
            if (2 * c2 < R) {
              double2 h[U];
#pragma unroll
              for (int u = 0; u < U; ++u) h[u] = ldh<P>(&H2[(int64_t)dq[u] * Rp2 + c2]);
#pragma unroll
              for (int u = 0; u < U; ++u) {
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
              const double2 h = ldh<P>(&H2[(int64_t)d * Rp2 + c2]);
              acc[j].x = fma(v, h.x, acc[j].x);
              acc[j].y = fma(v, h.y, acc[j].y);
            }
          }
        }
        q += run;
      }
    }
    flush();
  }
}

// ---------------------------------------------------------------- fused pass B + SpMM
// Work item = a chunk of kFC consecutive entries of the bucketed array `tmp` (pass A
// output: bucket b's entries, rows mixed, at [rptr[b<<sh], rptr[(b+1)<<sh])).  Per bucket
// segment of the chunk the CTA counting-sorts the entries by row in shared memory, splits
// the sorted segment evenly over its warps, and each warp reduces its rows' runs in
// registers; a run that is the whole row is stored, else added with red.global.
constexpr int kFC = 3072;
constexpr int kFThreads = 512;
constexpr int kFMaxRows = 256;

template <int NP, int P, int U>
__global__ void __launch_bounds__(kFThreads)
lab_fused_kernel(const double2 *__restrict__ tmp, const int64_t *__restrict__ rptr,
                 int64_t n_rows, int sh, const int64_t *__restrict__ nnzp,
                 const double *__restrict__ Hs, int R, double *__restrict__ out) {
  __shared__ int32_t sfib[kFC];
  __shared__ double sval[kFC];
  __shared__ int32_t hist[kFMaxRows + 1];
  __shared__ int32_t start[kFMaxRows + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = kFThreads / 32;
  const int Rp2 = hs_stride(R) >> 1;
  const double2 *H2 = reinterpret_cast<const double2 *>(Hs);
  const int64_t nnz = nnzp[0];
  const int64_t nchunks = ceil_div(nnz, kFC);
  const int64_t nb = ceil_div(n_rows, (int64_t)1 << sh);
  const int brows = 1 << sh;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = ch * kFC, c1 = min(c0 + kFC, nnz);
    // bucket holding c0: largest b with rptr[b << sh] <= c0
    int64_t lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (rptr[mid << sh] <= c0) lo = mid; else hi = mid;
    }
    int64_t b = lo;
    int64_t s0 = c0;
    while (s0 < c1) {
      const int64_t r0 = b << sh;
      const int64_t bend = rptr[min(n_rows, r0 + brows)];
      const int64_t s1 = min(c1, bend);
      const int n = (int)(s1 - s0);
      if (n <= 0) { ++b; continue; }
      for (int i = threadIdx.x; i <= brows; i += kFThreads) hist[i] = 0;
      __syncthreads();
      // load + rank within row
      constexpr int PER = kFC / kFThreads;
      int rl[PER], rk[PER], fb[PER];
      double vv[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int i = u * kFThreads + threadIdx.x;
        rl[u] = -1;
        if (i < n) {
          const double2 e = tmp[s0 + i];
          const uint64_t key = (uint64_t)__double_as_longlong(e.x);
          rl[u] = (int)((int64_t)(key >> 32) - r0);
          fb[u] = (int)(uint32_t)(key & 0xffffffffu);
          vv[u] = e.y;
        }
      }
#pragma unroll
      for (int u = 0; u < PER; ++u)
        if (rl[u] >= 0) rk[u] = atomicAdd(&hist[rl[u]], 1);
      __syncthreads();
      if (wid == 0) {   // exclusive scan of hist[0..brows) into start
        int carry = 0;
        for (int base = 0; base < brows; base += 32) {
          const int i = base + lane;
          int v = i < brows ? hist[i] : 0;
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          if (i < brows) start[i] = carry + x - v;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) start[brows] = carry;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < PER; ++u)
        if (rl[u] >= 0) {
          const int p = start[rl[u]] + rk[u];
          sfib[p] = fb[u];
          sval[p] = vv[u];
        }
      __syncthreads();
      // warp w reduces sorted positions [p0, p1)
      const int per = (n + NW - 1) / NW;
      const int p0 = min(n, wid * per), p1 = min(n, p0 + per);
      if (p0 < p1) {
        // row of p0: largest r with start[r] <= p0
        int rlo = 0, rhi = brows;
        while (rhi - rlo > 1) {
          const int mid = (rlo + rhi) >> 1;
          if (start[mid] <= p0) rlo = mid; else rhi = mid;
        }
        int row = rlo;
        double2 acc[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] = make_double2(0.0, 0.0);
        int rs = start[row], re = start[row + 1];
        auto flush = [&]() {
          const int a = max(rs, p0), z = min(re, p1);
          if (z > a) {
            const int64_t grow = r0 + row;
            const bool whole = (int64_t)(z - a) == rptr[grow + 1] - rptr[grow];
#pragma unroll
            for (int j = 0; j < NP; ++j) {
              const int c = 2 * (lane + 32 * j);
              if (c < R) {
                double *o = out + grow * R + c;
                if (whole) {
                  o[0] = acc[j].x;
                  if (c + 1 < R) o[1] = acc[j].y;
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
        for (int base = p0; base < p1; base += 32) {
          const int cnt = min(32, p1 - base);
          int md = 0;
          double mv = 0.0;
          if (lane < cnt) {
            md = sfib[base + lane];
            mv = sval[base + lane];
          }
          int q = 0;
          while (q < cnt) {
            while (base + q >= re) {
              flush();
              ++row;
              rs = re;
              re = start[row + 1];
            }
            const int run = min(cnt - q, re - (base + q));
            int t = 0;
            for (; t + U <= run; t += U) {
              int dq[U];
              double vq[U];
#pragma unroll
              for (int u = 0; u < U; ++u) {
                dq[u] = __shfl_sync(0xffffffffu, md, q + t + u);
                vq[u] = __shfl_sync(0xffffffffu, mv, q + t + u);
              }
#pragma unroll
              for (int j = 0; j < NP; ++j) {
                const int c2 = lane + 32 * j;
                if (2 * c2 < R) {
                  double2 h[U];
#pragma unroll
                  for (int u = 0; u < U; ++u) h[u] = ldh<P>(&H2[(int64_t)dq[u] * Rp2 + c2]);
#pragma unroll
                  for (int u = 0; u < U; ++u) {
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
                  const double2 h = ldh<P>(&H2[(int64_t)d * Rp2 + c2]);
                  acc[j].x = fma(v, h.x, acc[j].x);
                  acc[j].y = fma(v, h.y, acc[j].y);
                }
              }
            }
            q += run;
          }
        }
        flush();
      }
      __syncthreads();
      s0 = s1;
      ++b;
    }
  }
}

}  // namespace

extern "C" int lab_spmm(int variant, void *d_ws, size_t ws_bytes, int64_t J, int64_t n_rows,
                        int R, double *d_out, int reps, float *ms_out, int grid_mul) {
  const int64_t cap = mttkrp_cap(J, n_rows, R, ws_bytes);
  MttkrpLayout L(J, cap, n_rows, R);
  char *w = (char *)d_ws;
  const int64_t *rptr = (const int64_t *)(w + L.o_rptr);
  const int64_t *nnz = (const int64_t *)(w + L.o_nnz);
  const double2 *ent = (const double2 *)(w + L.o_ent);
  const double2 *tmp = (const double2 *)(w + L.o_tmp);
  const double *Hs = (const double *)(w + L.o_Hs);
  int sh = 0;
  while ((ceil_div(n_rows, (int64_t)1 << sh)) > kBucketMax) ++sh;
  if ((1 << sh) > kFMaxRows && variant >= 10) return -2;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const unsigned sb = (unsigned)(grid_mul * sm_count());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaMemset(d_out, 0, sizeof(double) * n_rows * R);
    cudaEventRecord(a);
    switch (variant) {
      case 0: lab_spmm_kernel<1, 0, 4><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 1: lab_spmm_kernel<1, 1, 4><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 2: lab_spmm_kernel<1, 2, 4><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 3: lab_spmm_kernel<1, 3, 4><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 4: lab_spmm_kernel<1, 4, 4><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 5: lab_spmm_kernel<1, 1, 8><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 6: lab_spmm_kernel<1, 2, 8><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 7: lab_spmm_kernel<1, 0, 2><<<sb, 256>>>(rptr, n_rows, nnz, ent, Hs, R, d_out); break;
      case 10: lab_fused_kernel<1, 0, 4><<<sb, kFThreads>>>(tmp, rptr, n_rows, sh, nnz, Hs, R, d_out); break;
      case 11: lab_fused_kernel<1, 1, 4><<<sb, kFThreads>>>(tmp, rptr, n_rows, sh, nnz, Hs, R, d_out); break;
      case 12: lab_fused_kernel<1, 2, 4><<<sb, kFThreads>>>(tmp, rptr, n_rows, sh, nnz, Hs, R, d_out); break;
      default: return -1;
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms_out = best;
  return (int)cudaGetLastError();
}


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
