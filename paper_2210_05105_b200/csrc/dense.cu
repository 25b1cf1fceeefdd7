// Small dense fp64 algebra on the hot path: Gram matrices, the R x R pseudo-inverse,
// the factor update GEMM with its column norms, renormalisation, sample weights.
// Ref: linalg.py:64-111, schedules.py:104-128, samplers.py:89-96, als.py:129-138.
#include <algorithm>

#include <stdlib.h>

#include "common.cuh"
#include "gram_mma.cuh"

using namespace rcp;

namespace {

int g_sms = 0;
int sm_count() {
  if (!g_sms) {
    g_sms = rcp_device_sms();
    if (!g_sms) g_sms = 148;
  }
  return g_sms;
}

// ------------------------------------------------------------------------------ Gram
// G = sum_r s_r^2 u_r u_r^T over n rows (U row-major n x R).  One CTA per SM streams
// 64-row chunks (contiguous 64 R doubles) into shared memory with cp.async, double
// buffered; each thread accumulates 4x4 tiles of the upper triangle for one row group;
// row groups are combined in a fixed order, CTA partials by sum_partials (deterministic).
constexpr int kGramRows = 64;      // rows per staged chunk
constexpr int kGramThreads = 256;
// tile pairs per thread: (R/4)(R/4+1)/2 <= 3*256 for R <= 128 (template parameter)

#ifndef RCP_GRAM_CTAS
#define RCP_GRAM_CTAS 2   // CTAs per SM of the Gram kernels (swept 1/2/3: tools/lab/dense_lab.py)
#endif
#ifndef RCP_GRAM_MINB
#define RCP_GRAM_MINB 2   // __launch_bounds__ min blocks of gram_mma_kernel (<= 128 registers)
#endif
int getenv_flag(const char *name) {   // 1 when the variable is set to "1" (read once per name use)
  const char *e = getenv(name);
  return e && e[0] == '1' ? 1 : 0;
}

int gram_grid(int64_t n) {
  int64_t tiles = ceil_div(n, kGramRows);
  // large factors: more CTAs hide the load latency; small ones keep fewer partials
#ifndef RCP_GRAM_BIG_ROWS
#define RCP_GRAM_BIG_ROWS (1LL << 20)
#endif
  int64_t g = (int64_t)(n >= RCP_GRAM_BIG_ROWS ? RCP_GRAM_CTAS : 1) * sm_count();
  if (tiles < g) g = tiles;
  return (int)(g < 1 ? 1 : g);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

size_t gram_smem(int R) {
  const int nT = (R + 3) / 4;
  const size_t chunk = 2 * ((size_t)kGramRows * R + 8) + 2 * kGramRows;
  const size_t red = (size_t)kGramThreads * 16;   // row-group partials
  (void)nT;
  return sizeof(double) * (chunk > red ? chunk : red) + 64;
}

template <int kGramMaxPairs>
__global__ void __launch_bounds__(kGramThreads)
gram_partial_kernel(const double *__restrict__ U, const double *__restrict__ scale, int64_t n,
                    int R, int aligned16, double *__restrict__ part) {
  extern __shared__ __align__(16) double sh[];
  const int nT = (R + 3) / 4;
  const int npairs = nT * (nT + 1) / 2;
  const int cs = kGramRows * R + 8;                 // chunk stride (doubles), even
  double *buf0 = sh, *buf1 = sh + cs;
  double *sc0 = sh + 2 * cs, *sc1 = sc0 + kGramRows;
  // thread -> (row group, pair list)
  const int groups = npairs <= kGramThreads ? kGramThreads / npairs : 1;
  const int grp = npairs <= kGramThreads ? (int)threadIdx.x / npairs : 0;
  int pa[kGramMaxPairs], pb[kGramMaxPairs];
  double acc[kGramMaxPairs][4][4];
#pragma unroll
  for (int p = 0; p < kGramMaxPairs; ++p) {
    int id = npairs <= kGramThreads ? (p == 0 ? (int)threadIdx.x % npairs : npairs)
                                    : (int)threadIdx.x + p * kGramThreads;
    if (grp >= groups) id = npairs;
    pa[p] = -1;
    pb[p] = -1;
    if (id < npairs) {  // decode upper-triangular tile pair (ta <= tb)
      int ta = 0, rem = id;
      while (rem >= nT - ta) {
        rem -= nT - ta;
        ++ta;
      }
      pa[p] = ta;
      pb[p] = ta + rem;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[p][x][y] = 0.0;
  }
  const int64_t nchunks = ceil_div(n, kGramRows);
  auto issue = [&](int64_t c, double *dst, double *scd) {
    const int64_t r0 = c * kGramRows;
    const int rows = (int)min((int64_t)kGramRows, n - r0);
    const int64_t cnt = (int64_t)rows * R;          // doubles, contiguous from U + r0 R
    const double *src = U + r0 * R;   // 16-byte aligned when U is (r0 R is even)
    if (aligned16) {
      const int64_t n16 = cnt >> 1;
      for (int64_t e = threadIdx.x; e < n16; e += blockDim.x) cp_async16(dst + 2 * e, src + 2 * e);
      if ((cnt & 1) && threadIdx.x == 0) cp_async8(dst + cnt - 1, src + cnt - 1);
    } else {
      for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) cp_async8(dst + e, src + e);
    }
    for (int q = threadIdx.x; q < kGramRows; q += blockDim.x) {
      double v = 0.0;
      if (q < rows) {
        v = scale ? scale[r0 + q] : 1.0;
        v *= v;
      }
      scd[q] = v;
    }
    cp_async_commit();
  };
  int cur = 0;
  if ((int64_t)blockIdx.x < nchunks) issue(blockIdx.x, buf0, sc0);
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t nx = c + gridDim.x;
    if (nx < nchunks) {
      issue(nx, cur ? buf0 : buf1, cur ? sc0 : sc1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double *tile = cur ? buf1 : buf0;
    const double *scw = cur ? sc1 : sc0;
    const int rows = (int)min((int64_t)kGramRows, n - c * kGramRows);
#pragma unroll
    for (int p = 0; p < kGramMaxPairs; ++p) {
      if (pa[p] < 0) continue;
      const int a0 = pa[p] * 4, b0 = pb[p] * 4;
      for (int rr = grp; rr < rows; rr += groups) {
        const double *row = tile + rr * R;
        const double w = scw[rr];
        double av[4], bv[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          av[x] = row[a0 + x] * w;   // columns >= R read the next row: discarded below
          bv[x] = row[b0 + x];
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[p][x][y] = fma(av[x], bv[y], acc[p][x][y]);
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  double *out = part + (int64_t)blockIdx.x * R * R;
  if (groups > 1) {
    // combine the row groups in group order (deterministic), pair-major layout
    double *red = sh;
    if (pa[0] >= 0) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) red[((size_t)grp * npairs + threadIdx.x % npairs) * 16 + x * 4 + y] = acc[0][x][y];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < npairs * 16; e += blockDim.x) {
      const int pr = e >> 4, xy = e & 15;
      double v = 0.0;
      for (int g = 0; g < groups; ++g) v += red[((size_t)g * npairs + pr) * 16 + xy];
      int ta = 0, rem = pr;
      while (rem >= nT - ta) {
        rem -= nT - ta;
        ++ta;
      }
      const int a = ta * 4 + (xy >> 2), b = (ta + rem) * 4 + (xy & 3);
      if (a < R && b < R) {
        out[a * R + b] = v;
        out[b * R + a] = v;
      }
    }
    return;
  }
#pragma unroll
  for (int p = 0; p < kGramMaxPairs; ++p) {
    if (pa[p] < 0) continue;
    const int a0 = pa[p] * 4, b0 = pb[p] * 4;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        int a = a0 + x, b = b0 + y;
        if (a < R && b < R) {
          out[a * R + b] = acc[p][x][y];
          out[b * R + a] = acc[p][x][y];
        }
      }
  }
}

__global__ void sum_partials_kernel(const double *__restrict__ part, int nparts, int64_t len,
                                    double *__restrict__ out) {
  // block = 32 elements x 8 slices; slice s sums partials p = s, s+8, ... (x4 unrolled),
  // then the 8 slice sums are combined in a fixed order: deterministic.
  __shared__ double red[8][33];
  const int el = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int64_t e = blockIdx.x * 32LL + el;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (e < len) {
    const double *p0 = part + e;
    int p = sl;
    for (; p + 24 < nparts; p += 32) {
      a0 += p0[(int64_t)p * len];
      a1 += p0[(int64_t)(p + 8) * len];
      a2 += p0[(int64_t)(p + 16) * len];
      a3 += p0[(int64_t)(p + 24) * len];
    }
    for (; p < nparts; p += 8) a0 += p0[(int64_t)p * len];
  }
  red[sl][el] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (sl == 0 && e < len) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += red[q][el];
    out[e] = s;
  }
}

// --------------------------------------------------------------------------- pinv
constexpr int kPinvThreads = 512;

__device__ double block_reduce(double v, double *red, bool is_max) {
  // all threads participate; result broadcast
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : v + w;
  }
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    v = lane < nw ? red[lane] : (is_max ? -1.0 / 0.0 : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmax(v, w) : v + w;
    }
    if (lane == 0) red[32] = v;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

// Load (chain of) input into A (stride LD), symmetric check; returns false if asymmetric.
__device__ void load_input(const double *in, int n_chain, int skip, int R, int LD, double *A,
                           double *chain_out) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double v;
    if (n_chain <= 0) {
      v = in[e];
    } else {
      bool have = false;
      v = 0.0;
      for (int m = 0; m < n_chain; ++m) {
        if (m == skip) continue;
        double g = in[(int64_t)m * R * R + e];
        v = have ? v * g : g;
        have = true;
      }
    }
    A[(e / R) * LD + (e % R)] = v;
    if (chain_out) chain_out[e] = v;
  }
}

__device__ __forceinline__ double fast_rcp(double x) {
  // reciprocal to ~1 ulp: hardware approximation + two Newton steps (no slow path)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Gauss-Jordan inverse of the SPD matrix in A (no pivoting).  Warp w owns rows
// w + 16a (a < RA), lane l owns columns l + 32b (b < RB); the RA x RB entries stay in
// registers for the whole inversion.  Pivot k needs only row k and column k, which their
// owners publish to a double-buffered shared row/column before the single barrier of the
// step.  Returns false (uniformly) on a non-positive pivot; A then holds garbage.
template <int RA, int RB>
__device__ bool gj_registers(double *A, int LD, int R, double *rcb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double v[RA][RB];
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int i = w + 16 * a, j = lane + 32 * b;
      v[a][b] = (i < R && j < R) ? A[i * LD + j] : 0.0;
    }
  for (int q = threadIdx.x; q < R; q += blockDim.x) {
    rcb[q] = A[q];                // row 0
    rcb[2 * R + q] = A[q * LD];   // column 0
  }
  __syncthreads();
  for (int k = 0; k < R; ++k) {
    const int pb = k & 1;
    const double *rowk = rcb + pb * R, *colk = rcb + 2 * R + pb * R;
    double *rown = rcb + (pb ^ 1) * R, *coln = rcb + 2 * R + (pb ^ 1) * R;
    const double pk = rowk[k];
    if (!(pk > 0.0)) return false;   // every thread reads the same pivot
    const double rk = fast_rcp(pk);
    // all shared reads of the step first (the publishes below alias nothing read here,
    // but the compiler cannot prove it and would serialise the rows otherwise)
    double rj[RB], ci[RA];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int j = lane + 32 * b;
      rj[b] = j < R ? rowk[j] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < RA; ++a) {
      const int i = w + 16 * a;
      ci[a] = i < R ? colk[i] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < RA; ++a) {
      const int i = w + 16 * a;
      const double f = ci[a] * rk;
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        const bool jk = lane + 32 * b == k;
        const double x = v[a][b];
        const double row = jk ? rk : x * rk;          // i == k
        const double oth = jk ? -f : fma(-f, rj[b], x);
        v[a][b] = (i == k) ? row : oth;
      }
    }
#pragma unroll
    for (int a = 0; a < RA; ++a) {
      const int i = w + 16 * a;
      if (i == k + 1) {                          // publish the next pivot row
#pragma unroll
        for (int b = 0; b < RB; ++b)
          if (lane + 32 * b < R) rown[lane + 32 * b] = v[a][b];
      }
#pragma unroll
      for (int b = 0; b < RB; ++b)               // and the next pivot column
        if (i < R && lane + 32 * b == k + 1) coln[i] = v[a][b];
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int i = w + 16 * a, j = lane + 32 * b;
      if (i < R && j < R) A[i * LD + j] = v[a][b];
    }
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kPinvThreads)
pinv_kernel(const double *__restrict__ in, int n_chain, int skip, int R, double cutoff,
            double *__restrict__ chain_out, double *__restrict__ out, int *status) {
  extern __shared__ double sh[];
  const int LD = R + 1;
  double *A = sh;                       // R x LD
  double *red = A + R * LD;             // 33
  double *diag = red + 40;              // R (eigenvalues)
  double *cs = diag + R + 1;            // R/2+1 cosines
  double *sn = cs + (R / 2 + 2);        // sines
  int *pr = reinterpret_cast<int *>(sn + (R / 2 + 2));  // pairs (2*(R/2+1))
  double *rcb = sn + (R / 2 + 2) + (R / 2 + 2) + 2;  // 4R + 2: pivot row/column (x2), 1/pivot
  __shared__ int flag;

  load_input(in, n_chain, skip, R, LD, A, chain_out);
  __syncthreads();
  // symmetry check on the raw input (ref linalg.py:92-95)
  double mx = 0.0, asym = 0.0;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    int a = e / R, b = e % R;
    mx = fmax(mx, fabs(A[a * LD + b]));
    asym = fmax(asym, fabs(A[a * LD + b] - A[b * LD + a]));
  }
  mx = block_reduce(mx, red, true);
  asym = block_reduce(asym, red, true);
  if (asym > 1e-8 * fmax(mx, 1.0)) {
    if (threadIdx.x == 0) raise_status(status, RCP_ST_ASYMMETRIC);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = 0.0;
    return;
  }
  // symmetrise: S = (G + G^T)/2 (upper triangle computed once, mirrored)
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    int a = e / R, b = e % R;
    if (a < b) {
      double s = 0.5 * (A[a * LD + b] + A[b * LD + a]);
      A[a * LD + b] = s;
      A[b * LD + a] = s;
    }
  }
  __syncthreads();
  double fro = 0.0;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double v = A[(e / R) * LD + (e % R)];
    fro += v * v;
  }
  fro = sqrt(block_reduce(fro, red, false));

  // ---- fast path: Gauss-Jordan inverse (no pivoting; valid for SPD) ----
  // Every thread keeps its entries (e = tid + 512 m) in registers for the whole inversion;
  // pivot k needs only row k and column k, which their owners publish to a double-buffered
  // shared row/column before the single barrier of the step.
  if (threadIdx.x == 0) flag = (fro > 0.0) ? 1 : 0;
  __syncthreads();
  if (flag) {
    bool ok;
    if (R <= 16) ok = gj_registers<1, 1>(A, LD, R, rcb);
    else if (R <= 32) ok = gj_registers<2, 1>(A, LD, R, rcb);
    else if (R <= 48) ok = gj_registers<3, 2>(A, LD, R, rcb);
    else if (R <= 64) ok = gj_registers<4, 2>(A, LD, R, rcb);
    else if (R <= 80) ok = gj_registers<5, 3>(A, LD, R, rcb);
    else if (R <= 96) ok = gj_registers<6, 3>(A, LD, R, rcb);
    else if (R <= 112) ok = gj_registers<7, 4>(A, LD, R, rcb);
    else ok = gj_registers<8, 4>(A, LD, R, rcb);
    if (!ok && threadIdx.x == 0) flag = 0;
    __syncthreads();
  }
  double *Ainv = A;
  if (flag) {
    double ifro = 0.0;
    bool finite = true;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      double v = Ainv[(e / R) * LD + (e % R)];
      ifro += v * v;
      if (!isfinite(v)) finite = false;
    }
    double bad = block_reduce(finite ? 0.0 : 1.0, red, true);
    ifro = sqrt(block_reduce(ifro, red, false));
    // kappa_2 <= ||S||_F ||S^-1||_F ; below 1e8 every eigenvalue clears 1e-10 * lambda_max
    if (bad == 0.0 && fro * ifro < 1e8 && cutoff <= 1e-9) {
      for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        int a = e / R, b = e % R;
        out[e] = 0.5 * (Ainv[a * LD + b] + Ainv[b * LD + a]);
      }
      return;
    }
  }
  // ---- robust path: parallel cyclic Jacobi eigendecomposition, reference cutoff ----
  __syncthreads();
  load_input(in, n_chain, skip, R, LD, A, nullptr);
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    int a = e / R, b = e % R;
    if (a < b) {
      double s = 0.5 * (A[a * LD + b] + A[b * LD + a]);
      A[a * LD + b] = s;
      A[b * LD + a] = s;
    }
  }
  double *Vt = out;  // eigenvectors as rows, kept in global scratch
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Vt[e] = (e / R == e % R) ? 1.0 : 0.0;
  __syncthreads();
  const int m = (R + 1) & ~1;  // even count with a dummy index R when R is odd
  const int half = m / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      int a = e / R, b = e % R;
      double v = A[a * LD + b];
      if (a != b) off += v * v; else dg += v * v;
    }
    off = block_reduce(off, red, false);
    dg = block_reduce(dg, red, false);
    if (off <= 1e-32 * dg || off == 0.0) break;
    for (int step = 0; step < m - 1; ++step) {
      // round-robin pairing: slot 0 fixed, others rotate by `step`
      for (int i = threadIdx.x; i < half; i += blockDim.x) {
        int s1 = i, s2 = m - 1 - i;
        auto who = [&](int slot) { return slot == 0 ? 0 : 1 + (slot - 1 + step) % (m - 1); };
        int p = who(s1), q = who(s2);
        if (p > q) { int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < R) {
          double apq = A[p * LD + q];
          if (apq != 0.0) {
            double th = (A[q * LD + q] - A[p * LD + p]) / (2.0 * apq);
            double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        }
        cs[i] = c;
        sn[i] = s;
        pr[2 * i] = p;
        pr[2 * i + 1] = q;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < half * R; e += blockDim.x) {  // rows: A <- J^T A ; Vt
        int i = e / R, j = e % R;
        int p = pr[2 * i], q = pr[2 * i + 1];
        if (q >= R || sn[i] == 0.0) continue;
        double c = cs[i], s = sn[i];
        double ap = A[p * LD + j], aq = A[q * LD + j];
        A[p * LD + j] = c * ap - s * aq;
        A[q * LD + j] = s * ap + c * aq;
        double vp = Vt[p * R + j], vq = Vt[q * R + j];
        Vt[p * R + j] = c * vp - s * vq;
        Vt[q * R + j] = s * vp + c * vq;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < half * R; e += blockDim.x) {  // cols: A <- A J
        int i = e / R, j = e % R;
        int p = pr[2 * i], q = pr[2 * i + 1];
        if (q >= R || sn[i] == 0.0) continue;
        double c = cs[i], s = sn[i];
        double ap = A[j * LD + p], aq = A[j * LD + q];
        A[j * LD + p] = c * ap - s * aq;
        A[j * LD + q] = s * ap + c * aq;
      }
      __syncthreads();
    }
  }
  for (int a = threadIdx.x; a < R; a += blockDim.x) diag[a] = A[a * LD + a];
  __syncthreads();
  double lmax = -1.0 / 0.0;
  for (int a = threadIdx.x; a < R; a += blockDim.x) lmax = fmax(lmax, diag[a]);
  lmax = block_reduce(lmax, red, true);
  // reuse A for Vt (global -> shared) before overwriting `out`
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) A[(e / R) * LD + (e % R)] = Vt[e];
  __syncthreads();
  for (int a = threadIdx.x; a < R; a += blockDim.x) {
    double w = diag[a];
    diag[a] = (lmax > 0.0 && w > cutoff * lmax) ? 1.0 / (w > 0.0 ? w : 1.0) : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    int a = e / R, b = e % R;
    double s = 0.0;
    for (int t = 0; t < R; ++t) s += A[t * LD + a] * diag[t] * A[t * LD + b];
    out[e] = s;
  }
}

// ------------------------------------------------------------------- update GEMM
constexpr int kUpdThreads = 256;

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// U = M B on the fp64 tensor cores (mma.m8n8k4), R <= 64: each warp takes 8-row tiles of
// M (staged in shared memory, zero padded to Rn = R rounded up to 8), keeps the tile's A
// fragments in registers and sweeps the n-tiles of B (block-shared, padded).  Column sums
// of squares per lane -> fixed-order warp/CTA reduction (deterministic).
template <int KS>   // k-steps = Rn / 4
__global__ void __launch_bounds__(kUpdThreads)
update_mma_kernel(const double *__restrict__ M, int64_t n, int R, const double *__restrict__ B,
                  double *__restrict__ U, double *__restrict__ part, int *status, int nbuf) {
  extern __shared__ double sh[];
  const int Rn = KS * 4;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int row = lane >> 2, quad = lane & 3;
  // row strides Rn + 4 (4 or 12 mod 16 doubles): conflict-free fragment reads
  const int Ss = Rn + 4;
  double *Bs = sh;                                   // Rn x Ss
  double *Mbase = sh + Rn * Ss + (size_t)wid * nbuf * 8 * Ss;   // per warp: nbuf x 8 x Ss
  for (int e = threadIdx.x; e < Rn * Ss; e += blockDim.x) {
    const int k = e / Ss, c = e - k * Ss;
    Bs[e] = (k < R && c < R) ? B[k * R + c] : 0.0;
  }
  for (int c = lane; c < nbuf * 8 * Ss; c += 32) Mbase[c] = 0.0;   // padding columns stay 0
  __syncthreads();
  double sq[KS / 2][2];   // this lane's columns nt*8 + 2 quad + {0,1}, nt < Rn/8
#pragma unroll
  for (int t = 0; t < KS / 2; ++t) sq[t][0] = sq[t][1] = 0.0;
  bool bad = false;
  const int64_t ntiles = ceil_div(n, (int64_t)8);
  const int64_t stride = (int64_t)gridDim.x * nw, t0 = (int64_t)blockIdx.x * nw + wid;
  // nbuf-stage cp.async pipeline: the tiles nbuf - 1 ahead load while this one computes
  auto stage = [&](int64_t tl, int slot) {
    if (tl < ntiles)
      stage_tile8(Mbase + slot * 8 * Ss, M, tl * 8, (int)min((int64_t)8, n - tl * 8), R, Ss, lane);
    cpa_commit();
  };
  for (int s = 0; s < nbuf - 1; ++s) stage(t0 + s * stride, s);
  int slot = 0;
  for (int64_t tile = t0; tile < ntiles; tile += stride) {
    stage(tile + (nbuf - 1) * stride, slot == 0 ? nbuf - 1 : slot - 1);
    cpa_wait_stages(nbuf);
    __syncwarp();
    const int64_t r0 = tile * 8;
    const int nr = (int)min((int64_t)8, n - r0);
    const double *Ms = Mbase + slot * 8 * Ss;
    double a[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[ks] = Ms[row * Ss + ks * 4 + quad];
    auto emit = [&](int nt, double c0, double c1) {
      const int col = nt * 8 + 2 * quad;
      if (row < nr) {
        if (col < R) {
          U[(r0 + row) * R + col] = c0;
          sq[nt][0] = fma(c0, c0, sq[nt][0]);
          if (!isfinite(c0)) bad = true;
        }
        if (col + 1 < R) {
          U[(r0 + row) * R + col + 1] = c1;
          sq[nt][1] = fma(c1, c1, sq[nt][1]);
          if (!isfinite(c1)) bad = true;
        }
      }
    };
    // two n-tiles at a time: two independent accumulator chains per warp
#pragma unroll
    for (int nt = 0; nt < KS / 2; nt += 2) {
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        dmma_8x8x4(c0, c1, a[ks], Bs[(ks * 4 + quad) * Ss + nt * 8 + row]);
        if (nt + 1 < KS / 2) dmma_8x8x4(d0, d1, a[ks], Bs[(ks * 4 + quad) * Ss + (nt + 1) * 8 + row]);
      }
      emit(nt, c0, c1);
      if (nt + 1 < KS / 2) emit(nt + 1, d0, d1);
    }
    __syncwarp();   // every lane is done with this slot before it is refilled
    slot = slot + 1 == nbuf ? 0 : slot + 1;
  }
  cpa_wait<0>();
  if (bad) raise_status(status, RCP_ST_NONFINITE);
  // lanes with equal quad hold the same columns: reduce over the 8 rows, then warps
#pragma unroll
  for (int nt = 0; nt < KS / 2; ++nt)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      double v = sq[nt][u];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      sq[nt][u] = v;
    }
  __syncthreads();
  double *wsq = sh;   // reuse: nw x Rn
  if (row == 0) {
#pragma unroll
    for (int nt = 0; nt < KS / 2; ++nt) {
      wsq[wid * Rn + nt * 8 + 2 * quad] = sq[nt][0];
      wsq[wid * Rn + nt * 8 + 2 * quad + 1] = sq[nt][1];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < R; c += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += wsq[w * Rn + c];
    part[(int64_t)blockIdx.x * R + c] = v;
  }
}


__global__ void renorm_kernel(double *__restrict__ U, int64_t n, int R,
                              const double *__restrict__ colsq, double *__restrict__ sigma) {
  extern __shared__ double nrm[];
  for (int c = threadIdx.x; c < R; c += blockDim.x) {
    double s = sqrt(colsq[c]);
    nrm[c] = s > 0.0 ? s : 1.0;
    if (blockIdx.x == 0 && sigma) sigma[c] = s;
  }
  __syncthreads();
  int64_t tot = n * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x)
    U[e] /= nrm[e % R];
}

__global__ void weights_kernel(const double *__restrict__ pmp, int N, int64_t J,
                               double *__restrict__ prob, double *__restrict__ w, int *status) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= J) return;
  double p = pmp[s];
  for (int m = 1; m < N; ++m) p *= pmp[(int64_t)m * J + s];
  if (prob) prob[s] = p;
  if (!(p > 0.0)) raise_status(status, RCP_ST_ZERO_PROB);
  w[s] = 1.0 / sqrt((double)J * p);
}

// out[e] = ((p_0[e] + p_1[e]) + p_2[e]) + ... : the rank-ordered sum of P replicated
// contributions (block Grams, column norms; ref grid.py:295-297).
__global__ void ordered_sum_kernel(const double *__restrict__ parts, int nparts, int64_t len,
                                   double *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = parts[e];
    for (int p = 1; p < nparts; ++p) s += parts[(int64_t)p * len + e];
    out[e] = s;
  }
}

__global__ void hadamard_rows_kernel(double *__restrict__ H, const double *__restrict__ urow,
                                     int64_t tot, int init) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x)
    H[e] = init ? urow[e] : H[e] * urow[e];
}

// R <= 64: the same Gram on the fp64 tensor cores.  For a 4-row step of Z = diag(s) U,
// thread t of a warp holds Z[r0 + t%4][8 tile + t/4] for every 8-column tile -- at once
// the A fragment (Z^T, row-major 8x4) and the B fragment (Z, col-major 4x8) of
// mma.m8n8k4 -- and accumulates every upper tile pair (a <= b) of G from registers.
// Steps go to (CTA, warp) in a fixed order; warps are combined in a fixed order (the CTA
// partials then by sum_partials): deterministic.
template <int T>
__global__ void __launch_bounds__(256, RCP_GRAM_MINB)
gram_mma_kernel(const double *__restrict__ U, const double *__restrict__ scale, int64_t n, int R,
                double *__restrict__ part) {
  constexpr int NP = T * (T + 1) / 2;
  __shared__ double red[NP * 64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc[NP][2];
#pragma unroll
  for (int p = 0; p < NP; ++p) acc[p][0] = acc[p][1] = 0.0;
  const int64_t steps = (n + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * nw;
  const int kk = lane & 3, col = lane >> 2;
  // three 4-row steps in flight per warp (loads of the next ones overlap the MMAs)
  double f0[T], f1[T], f2[T];
  int64_t s = (int64_t)blockIdx.x * nw + wid;
  gram_load<T>(U, scale, 4 * s + kk, n, R, col, f0);
  gram_load<T>(U, scale, 4 * (s + stride) + kk, n, R, col, f1);
  gram_load<T>(U, scale, 4 * (s + 2 * stride) + kk, n, R, col, f2);
  for (; s < steps; s += 3 * stride) {
    gram_accum<T>(f0, acc);
    gram_load<T>(U, scale, 4 * (s + 3 * stride) + kk, n, R, col, f0);
    if (s + stride >= steps) break;
    gram_accum<T>(f1, acc);
    gram_load<T>(U, scale, 4 * (s + 4 * stride) + kk, n, R, col, f1);
    if (s + 2 * stride >= steps) break;
    gram_accum<T>(f2, acc);
    gram_load<T>(U, scale, 4 * (s + 5 * stride) + kk, n, R, col, f2);
  }
  for (int w = 0; w < nw; ++w) {   // fixed-order combination of the warps
    if (wid == w) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double *q = red + p * 64 + 2 * lane;
        q[0] = w ? q[0] + acc[p][0] : acc[p][0];
        q[1] = w ? q[1] + acc[p][1] : acc[p][1];
      }
    }
    __syncthreads();
  }
  double *out = part + (int64_t)blockIdx.x * R * R;
  for (int e = threadIdx.x; e < NP * 64; e += blockDim.x) {
    int p = e >> 6, a = 0;
    while (p >= T - a) {
      p -= T - a;
      ++a;
    }
    const int b = a + p;
    const int ln = (e & 63) >> 1, u = e & 1;
    const int ga = 8 * a + (ln >> 2), gb = 8 * b + 2 * (ln & 3) + u;
    if (ga < R && gb < R) {
      out[ga * R + gb] = red[e];
      out[gb * R + ga] = red[e];
    }
  }
}

// 64 < R <= 128: the same register fragments, with the T(T+1)/2 upper tile pairs split
// into G groups of warps (a warp's group is fixed, its pairs a compile-time range) so the
// accumulators fit the register file; every warp loads the whole 4-row step (the warps of
// a CTA read the same rows at nearly the same time: L1 hits).  Steps go to (CTA, warp of
// the group) in a fixed order; warps and CTAs are combined in fixed orders: deterministic.
template <int T, int G, int g>
__device__ __forceinline__ void gram_split_body(const double *__restrict__ U,
                                                const double *__restrict__ scale, int64_t n, int R,
                                                int sub, double *red) {
  constexpr int NP = T * (T + 1) / 2;
  constexpr int PPG = (NP + G - 1) / G;
  constexpr int WG = 8 / G;   // warps per group
  const int lane = threadIdx.x & 31;
  double acc[PPG][2];
#pragma unroll
  for (int p = 0; p < PPG; ++p) acc[p][0] = acc[p][1] = 0.0;
  const int64_t steps = (n + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * WG;
  const int kk = lane & 3, col = lane >> 2;
  double f0[T], f1[T];   // two 4-row steps in flight
  int64_t s = (int64_t)blockIdx.x * WG + sub;
  gram_load<T>(U, scale, 4 * s + kk, n, R, col, f0);
  gram_load<T>(U, scale, 4 * (s + stride) + kk, n, R, col, f1);
  for (; s < steps; s += 2 * stride) {
    gram_accum_group<T, G, g>(f0, acc);
    gram_load<T>(U, scale, 4 * (s + 2 * stride) + kk, n, R, col, f0);
    if (s + stride >= steps) break;
    gram_accum_group<T, G, g>(f1, acc);
    gram_load<T>(U, scale, 4 * (s + 3 * stride) + kk, n, R, col, f1);
  }
  for (int w = 0; w < WG; ++w) {   // fixed-order combination of the group's warps
    if (sub == w) {
#pragma unroll
      for (int p = 0; p < PPG; ++p) {
        if (g * PPG + p >= NP) break;
        double *q = red + (g * PPG + p) * 64 + 2 * lane;
        q[0] = w ? q[0] + acc[p][0] : acc[p][0];
        q[1] = w ? q[1] + acc[p][1] : acc[p][1];
      }
    }
    __syncthreads();
  }
}

template <int T, int G>
__global__ void __launch_bounds__(256, 1)
gram_mma_split_kernel(const double *__restrict__ U, const double *__restrict__ scale, int64_t n,
                      int R, double *__restrict__ part) {
  constexpr int NP = T * (T + 1) / 2;
  extern __shared__ double red[];   // NP x 64
  const int wid = threadIdx.x >> 5;
  const int grp = wid % G, sub = wid / G;
  static_assert(G == 2 || G == 4 || G == 8, "G divides the 8 warps");
  switch (grp) {
    case 0: gram_split_body<T, G, 0>(U, scale, n, R, sub, red); break;
    case 1: gram_split_body<T, G, (G > 1 ? 1 : 0)>(U, scale, n, R, sub, red); break;
    case 2: gram_split_body<T, G, (G > 2 ? 2 : 0)>(U, scale, n, R, sub, red); break;
    case 3: gram_split_body<T, G, (G > 3 ? 3 : 0)>(U, scale, n, R, sub, red); break;
    case 4: gram_split_body<T, G, (G > 4 ? 4 : 0)>(U, scale, n, R, sub, red); break;
    case 5: gram_split_body<T, G, (G > 5 ? 5 : 0)>(U, scale, n, R, sub, red); break;
    case 6: gram_split_body<T, G, (G > 6 ? 6 : 0)>(U, scale, n, R, sub, red); break;
    default: gram_split_body<T, G, (G > 7 ? 7 : 0)>(U, scale, n, R, sub, red); break;
  }
  double *out = part + (int64_t)blockIdx.x * R * R;
  for (int e = threadIdx.x; e < NP * 64; e += blockDim.x) {
    int p = e >> 6, a = 0;
    while (p >= T - a) {
      p -= T - a;
      ++a;
    }
    const int b = a + p;
    const int ln = (e & 63) >> 1, u = e & 1;
    const int ga = 8 * a + (ln >> 2), gb = 8 * b + 2 * (ln & 3) + u;
    if (ga < R && gb < R) {
      out[ga * R + gb] = red[e];
      out[gb * R + ga] = red[e];
    }
  }
}

template <int T, int G>
int launch_gram_split(const double *U, const double *scale, int64_t n, int R, double *part, int grid,
                      cudaStream_t st) {
  constexpr int NP = T * (T + 1) / 2;
  const int smem = NP * 64 * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(gram_mma_split_kernel<T, G>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  gram_mma_split_kernel<T, G><<<grid, 256, smem, st>>>(U, scale, n, R, part);
  return RCP_OK;
}

// 64 < R <= 128, staged: slabs of 32 rows go through a 3-stage cp.async ring in shared
// memory (row stride 8T + 4 doubles: conflict-free fragment reads); warp w of the 8 owns the
// tile pairs [w PPW, (w + 1) PPW) for every row of the CTA's slabs, so its accumulators stay
// in registers and no partial is combined across warps.  Per 4-row step a warp reads the T
// fragments from shared memory (T LDS per ~T(T+1)/16 mma) instead of every warp of a group
// re-reading the rows from L1/L2.  Slabs go to CTAs round-robin, CTA partials are combined
// by sum_partials: deterministic.
template <int T>
size_t gram_staged_smem() {
  const size_t ring = (size_t)kGsStages * (kGsRows * gs_stride<T>() + kGsRows);
  const size_t red = (size_t)(T * (T + 1) / 2) * 64;
  return sizeof(double) * (ring > red ? ring : red);
}

template <int T>
__global__ void __launch_bounds__(256, 1)
gram_mma_staged_kernel(const double *__restrict__ U, const double *__restrict__ scale, int64_t n, int R,
                       double *__restrict__ part) {
  constexpr int NP = T * (T + 1) / 2;
  constexpr int PPW = (NP + 7) / 8;
  constexpr int ST = gs_stride<T>();
  constexpr int SLAB = kGsRows * ST + kGsRows;   // rows, then the 32 row scales
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool scaled = scale != nullptr;
  double acc[PPW][2];
#pragma unroll
  for (int p = 0; p < PPW; ++p) acc[p][0] = acc[p][1] = 0.0;
  // pad columns are never written by the copies
  for (int e = threadIdx.x; e < kGsStages * kGsRows * (ST - R); e += blockDim.x) {
    const int st = e / (kGsRows * (ST - R)), q = e - st * (kGsRows * (ST - R));
    const int r = q / (ST - R), c = R + (q - r * (ST - R));
    sm[st * SLAB + r * ST + c] = 0.0;
  }
  const int64_t slabs = (n + kGsRows - 1) / kGsRows;
  const int crow = threadIdx.x >> 3, c0 = threadIdx.x & 7;   // 8 threads per row
  auto issue = [&](int64_t sl, int st) {
    if (sl < slabs) {
      const int64_t r = sl * kGsRows + crow;
      const bool ok = r < n;
      const double *src = U + (ok ? r : 0) * (int64_t)R;
      double *dst = sm + st * SLAB + crow * ST;
      for (int c = c0; c < R; c += 8) cpa8_zfill(dst + c, src + c, ok);
      if (scaled && c0 == 0) cpa8_zfill(sm + st * SLAB + kGsRows * ST + crow, scale + (ok ? r : 0), ok);
    }
    cpa_commit();
  };
  int64_t sl = blockIdx.x;
  issue(sl, 0);
  issue(sl + gridDim.x, 1);
  int st = 0;
  for (; sl < slabs; sl += gridDim.x) {
    cpa_wait<1>();
    __syncthreads();   // the slab is visible; every warp is done with the stage refilled next
    issue(sl + 2 * (int64_t)gridDim.x, st == 0 ? 2 : st - 1);
    const double *ring = sm + st * SLAB;
    const double *sc = ring + kGsRows * ST;
    switch (wid) {
      case 0: gram_staged_body<T, 0>(ring, sc, scaled, lane, acc); break;
      case 1: gram_staged_body<T, 1>(ring, sc, scaled, lane, acc); break;
      case 2: gram_staged_body<T, 2>(ring, sc, scaled, lane, acc); break;
      case 3: gram_staged_body<T, 3>(ring, sc, scaled, lane, acc); break;
      case 4: gram_staged_body<T, 4>(ring, sc, scaled, lane, acc); break;
      case 5: gram_staged_body<T, 5>(ring, sc, scaled, lane, acc); break;
      case 6: gram_staged_body<T, 6>(ring, sc, scaled, lane, acc); break;
      default: gram_staged_body<T, 7>(ring, sc, scaled, lane, acc); break;
    }
    st = st == kGsStages - 1 ? 0 : st + 1;
  }
  cpa_wait<0>();
  __syncthreads();
  double *red = sm;   // NP x 64, each pair written by its one owner
#pragma unroll
  for (int p = 0; p < PPW; ++p) {
    const int gp = wid * PPW + p;
    if (gp < NP) {
      red[gp * 64 + 2 * lane] = acc[p][0];
      red[gp * 64 + 2 * lane + 1] = acc[p][1];
    }
  }
  __syncthreads();
  double *out = part + (int64_t)blockIdx.x * R * R;
  for (int e = threadIdx.x; e < NP * 64; e += blockDim.x) {
    int p = e >> 6, a = 0;
    while (p >= T - a) {
      p -= T - a;
      ++a;
    }
    const int b = a + p;
    const int ln = (e & 63) >> 1, u = e & 1;
    const int ga = 8 * a + (ln >> 2), gb = 8 * b + 2 * (ln & 3) + u;
    if (ga < R && gb < R) {
      out[ga * R + gb] = red[e];
      out[gb * R + ga] = red[e];
    }
  }
}

template <int T>
int launch_gram_staged(const double *U, const double *scale, int64_t n, int R, double *part, int &grid,
                       cudaStream_t st) {
  const int smem = (int)gram_staged_smem<T>();
  static int per_sm = 0;
  if (!per_sm) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(gram_mma_staged_kernel<T>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    RCP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gram_mma_staged_kernel<T>, 256,
                                                               smem));
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t slabs = (n + kGsRows - 1) / kGsRows;
  int g = per_sm * sm_count();
  if (g > grid) g = grid;   // the partial buffer holds gram_grid(n) matrices
  if (slabs < g) g = (int)slabs;
  grid = g < 1 ? 1 : g;
  gram_mma_staged_kernel<T><<<grid, 256, smem, st>>>(U, scale, n, R, part);
  return RCP_OK;
}

}  // namespace

extern "C" {

size_t rcp_gram_ws_bytes(int64_t n, int R) {
  return (size_t)gram_grid(n) * R * R * sizeof(double);
}

int rcp_gram(const double *d_U, const double *d_scale, int64_t n, int R, double *d_G,
             void *d_ws, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || n < 0 || !d_G || (n > 0 && (!d_U || !d_ws)))
    return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (n == 0) {
    RCP_CUDA_TRY(cudaMemsetAsync(d_G, 0, sizeof(double) * R * R, st));
    return RCP_OK;
  }
  int grid = gram_grid(n);
  const size_t smem = gram_smem(R);
  static bool attr = false;
  if (!attr) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(gram_partial_kernel<1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RCP_CUDA_TRY(cudaFuncSetAttribute(gram_partial_kernel<2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RCP_CUDA_TRY(cudaFuncSetAttribute(gram_partial_kernel<3>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const int al = ((uintptr_t)d_U & 15) == 0 ? 1 : 0;
  const int nT = (R + 3) / 4, npairs = nT * (nT + 1) / 2;
  double *part = (double *)d_ws;
  if (R <= 64) {   // fp64 tensor cores
    switch ((R + 7) / 8) {
      case 1: gram_mma_kernel<1><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      case 2: gram_mma_kernel<2><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      case 3: gram_mma_kernel<3><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      case 4: gram_mma_kernel<4><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      case 5: gram_mma_kernel<5><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      case 6: gram_mma_kernel<6><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      case 7: gram_mma_kernel<7><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
      default: gram_mma_kernel<8><<<grid, 256, 0, st>>>(d_U, d_scale, n, R, part); break;
    }
  } else if (getenv_flag("RCP_GRAM_SPLIT") == 0 && getenv_flag("RCP_GRAM_FFMA") == 0) {
    // 64 < R <= 128: fp64 tensor cores over shared-memory staged slabs
    int rc = RCP_OK;
    switch ((R + 7) / 8) {
      case 9: rc = launch_gram_staged<9>(d_U, d_scale, n, R, part, grid, st); break;
      case 10: rc = launch_gram_staged<10>(d_U, d_scale, n, R, part, grid, st); break;
      case 11: rc = launch_gram_staged<11>(d_U, d_scale, n, R, part, grid, st); break;
      case 12: rc = launch_gram_staged<12>(d_U, d_scale, n, R, part, grid, st); break;
      case 13: rc = launch_gram_staged<13>(d_U, d_scale, n, R, part, grid, st); break;
      case 14: rc = launch_gram_staged<14>(d_U, d_scale, n, R, part, grid, st); break;
      case 15: rc = launch_gram_staged<15>(d_U, d_scale, n, R, part, grid, st); break;
      default: rc = launch_gram_staged<16>(d_U, d_scale, n, R, part, grid, st); break;
    }
    if (rc) return rc;
  } else if (R <= 96 && getenv_flag("RCP_GRAM_FFMA") == 0) {
    // 64 < R <= 96: fp64 tensor cores with the tile pairs split over warp groups (C4 R=75 on
    // 4.8M rows: 3.15 ms vs 4.03 ms FFMA; above 96 the G=8 split is load-bound and the FFMA
    // kernel wins -- R=128: 18.5 vs 13.2 ms; profiles/r02_gram_r64.json)
    int rc = RCP_OK;
    switch ((R + 7) / 8) {
      case 9: rc = launch_gram_split<9, 4>(d_U, d_scale, n, R, part, grid, st); break;
      case 10: rc = launch_gram_split<10, 4>(d_U, d_scale, n, R, part, grid, st); break;
      case 11: rc = launch_gram_split<11, 4>(d_U, d_scale, n, R, part, grid, st); break;
      default: rc = launch_gram_split<12, 4>(d_U, d_scale, n, R, part, grid, st); break;
    }
    if (rc) return rc;
  } else if (npairs <= kGramThreads)
    gram_partial_kernel<1><<<grid, kGramThreads, smem, st>>>(d_U, d_scale, n, R, al, part);
  else if (npairs <= 2 * kGramThreads)
    gram_partial_kernel<2><<<grid, kGramThreads, smem, st>>>(d_U, d_scale, n, R, al, part);
  else
    gram_partial_kernel<3><<<grid, kGramThreads, smem, st>>>(d_U, d_scale, n, R, al, part);
  RCP_LAUNCH_CHECK("gram_partial");
  int64_t len = (int64_t)R * R;
  sum_partials_kernel<<<(unsigned)ceil_div(len, 32), 256, 0, st>>>((double *)d_ws, grid, len,
                                                                     d_G);
  RCP_LAUNCH_CHECK("gram_reduce");
  return RCP_OK;
}

int rcp_pinv(const double *d_in, int n_chain, int skip, int R, double rel_cutoff,
             double *d_chain_out, double *d_out, int *d_status, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || !d_in || !d_out) return RCP_ERR_ARG;
  // A, Jacobi scratch, pivot row/column buffers (see pinv_kernel's layout)
  const size_t smem =
      sizeof(double) * ((size_t)R * (R + 1) + 40 + (R + 1) + 3 * (R / 2 + 2) + 2 + 4 * R + 2) + 64;
  static bool attr = false;
  if (!attr) {
    RCP_CUDA_TRY(cudaFuncSetAttribute(pinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
    attr = true;
  }
  pinv_kernel<<<1, kPinvThreads, smem, RCP_STREAM(stream)>>>(d_in, n_chain, skip, R, rel_cutoff,
                                                            d_chain_out, d_out, d_status);
  RCP_LAUNCH_CHECK("pinv");
  return RCP_OK;
}

size_t rcp_update_ws_bytes(int64_t n, int R) {
  (void)n;
  return (size_t)4 * sm_count() * R * sizeof(double);
}

int rcp_update(const double *d_M, int64_t n, int R, const double *d_B, double *d_U_out,
               double *d_colsq, void *d_ws, int *d_status, void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || n < 0 || !d_B || !d_colsq || (n > 0 && (!d_M || !d_U_out)))
    return RCP_ERR_ARG;
  cudaStream_t st = RCP_STREAM(stream);
  if (n == 0) {
    RCP_CUDA_TRY(cudaMemsetAsync(d_colsq, 0, sizeof(double) * R, st));
    return RCP_OK;
  }
  const int nw = kUpdThreads / 32;
  double *part = (double *)d_ws;
  {   // fp64 tensor cores (every R <= RCP_MAX_RANK)
    static bool attr_mma = false;
    if (!attr_mma) {
#define RCP_UPD_ATTR(K)                                                                  \
  RCP_CUDA_TRY(cudaFuncSetAttribute(update_mma_kernel<K>,                                \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
      RCP_UPD_ATTR(2); RCP_UPD_ATTR(4); RCP_UPD_ATTR(6); RCP_UPD_ATTR(8);
      RCP_UPD_ATTR(10); RCP_UPD_ATTR(12); RCP_UPD_ATTR(14); RCP_UPD_ATTR(16);
      RCP_UPD_ATTR(18); RCP_UPD_ATTR(20); RCP_UPD_ATTR(22); RCP_UPD_ATTR(24);
      RCP_UPD_ATTR(26); RCP_UPD_ATTR(28); RCP_UPD_ATTR(30); RCP_UPD_ATTR(32);
#undef RCP_UPD_ATTR
      attr_mma = true;
    }
    const int Rn = (R + 7) & ~7;
    const int ks = Rn / 4;
    int64_t tiles = ceil_div(n, (int64_t)8);
    int g = (int)std::min<int64_t>(ceil_div(tiles, (int64_t)nw), 4LL * sm_count());
#ifndef RCP_UPD_NBUF
#define RCP_UPD_NBUF 2
#endif
#ifndef RCP_UPD_SMEM_KB
#define RCP_UPD_SMEM_KB 110   // two CTAs per SM
#endif
    int nbuf = RCP_UPD_NBUF;
    auto upd_smem = [&](int nb) {
      return sizeof(double) * ((size_t)Rn * (Rn + 4) + (size_t)nw * nb * 8 * (Rn + 4));
    };
    while (nbuf > 1 && upd_smem(nbuf) > RCP_UPD_SMEM_KB * 1024) --nbuf;
    const size_t sm2 = upd_smem(nbuf);
    switch (ks) {
      case 2: update_mma_kernel<2><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 4: update_mma_kernel<4><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 6: update_mma_kernel<6><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 8: update_mma_kernel<8><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 10: update_mma_kernel<10><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 12: update_mma_kernel<12><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 14: update_mma_kernel<14><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 16: update_mma_kernel<16><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 18: update_mma_kernel<18><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 20: update_mma_kernel<20><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 22: update_mma_kernel<22><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 24: update_mma_kernel<24><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 26: update_mma_kernel<26><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 28: update_mma_kernel<28><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      case 30: update_mma_kernel<30><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
      default: update_mma_kernel<32><<<g, kUpdThreads, sm2, st>>>(d_M, n, R, d_B, d_U_out, part, d_status, nbuf); break;
    }
    RCP_LAUNCH_CHECK("update_mma");
    sum_partials_kernel<<<(unsigned)ceil_div(R, 32), 256, 0, st>>>(part, g, R, d_colsq);
    RCP_LAUNCH_CHECK("update_colsq");
  }
  return RCP_OK;
}

int rcp_renormalize(double *d_U, int64_t n, int R, const double *d_colsq, double *d_sigma,
                    void *stream) {
  if (R < 1 || R > RCP_MAX_RANK || n < 0 || !d_colsq) return RCP_ERR_ARG;
  int64_t tot = n * R;
  int64_t blocks = ceil_div(tot > 0 ? tot : 1, 256);
  if (blocks > 8LL * sm_count()) blocks = 8LL * sm_count();
  renorm_kernel<<<(unsigned)blocks, 256, sizeof(double) * R, RCP_STREAM(stream)>>>(d_U, n, R,
                                                                                  d_colsq, d_sigma);
  RCP_LAUNCH_CHECK("renormalize");
  return RCP_OK;
}

int rcp_weights(const double *d_pmp, int N, int64_t J, double *d_prob, double *d_w,
                int *d_status, void *stream) {
  if (N < 1 || J < 0 || (J > 0 && (!d_pmp || !d_w))) return RCP_ERR_ARG;
  if (J == 0) return RCP_OK;
  weights_kernel<<<(unsigned)ceil_div(J, 256), 256, 0, RCP_STREAM(stream)>>>(d_pmp, N, J, d_prob,
                                                                             d_w, d_status);
  RCP_LAUNCH_CHECK("weights");
  return RCP_OK;
}

int rcp_ordered_sum(const double *d_parts, int nparts, int64_t len, double *d_out, void *stream) {
  if (nparts < 1 || len < 0) return RCP_ERR_ARG;
  if (len == 0) return RCP_OK;
  if (!d_parts || !d_out) return RCP_ERR_ARG;
  int64_t blocks = ceil_div(len, 256);
  if (blocks > 8LL * sm_count()) blocks = 8LL * sm_count();
  ordered_sum_kernel<<<(unsigned)blocks, 256, 0, RCP_STREAM(stream)>>>(d_parts, nparts, len, d_out);
  RCP_LAUNCH_CHECK("ordered_sum");
  return RCP_OK;
}

int rcp_hadamard_rows(double *d_H, const double *d_urow, int64_t J, int R, int init_ones,
                      void *stream) {
  if (J < 0 || R < 1) return RCP_ERR_ARG;
  int64_t tot = J * R;
  if (tot == 0) return RCP_OK;
  int64_t blocks = ceil_div(tot, 256);
  if (blocks > 8LL * sm_count()) blocks = 8LL * sm_count();
  hadamard_rows_kernel<<<(unsigned)blocks, 256, 0, RCP_STREAM(stream)>>>(d_H, d_urow, tot,
                                                                         init_ones);
  RCP_LAUNCH_CHECK("hadamard_rows");
  return RCP_OK;
}

}  // extern "C"
