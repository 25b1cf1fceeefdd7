// Random-stream contract of the reference (ref rng.py:26-32): numpy SeedSequence key
// derivation, Philox4x64-10 draws, Generator.random() and Generator.permutation().
#include <stdio.h>

#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace rcp {

static thread_local std::string g_err;

void set_error(const char *msg) { g_err = msg ? msg : ""; }

static unsigned long long g_launches = 0;

int check_launch(const char *what) {
  ++g_launches;  // every kernel launch site calls this once
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return RCP_ERR_CUDA;
  }
  return RCP_OK;
}

// ---------------------------------------------------------------- numpy SeedSequence
namespace seedseq {
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kPool = 4;

inline uint32_t hashmix(uint32_t v, uint32_t &h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> 16;
  return v;
}
inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}
// Python-int -> little-endian uint32 words (0 -> [0]).
inline void int_words(uint64_t x, std::vector<uint32_t> &out) {
  if (x == 0) {
    out.push_back(0);
    return;
  }
  while (x) {
    out.push_back((uint32_t)(x & 0xffffffffu));
    x >>= 32;
  }
}
}  // namespace seedseq

}  // namespace rcp

using namespace rcp;

extern "C" {

const char *rcp_version(void) { return "randcp_b200 0.1.0 (sm_100a)"; }
const char *rcp_last_error(void) { return rcp::g_err.c_str(); }
int64_t rcp_launch_count(void) { return (int64_t)rcp::g_launches; }

int rcp_device_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int rcp_stream_key(uint64_t seed, uint64_t purpose, const uint64_t *h_ctx, int n_ctx,
                   uint64_t *h_key_out) {
  using namespace rcp::seedseq;
  if (!h_key_out || n_ctx < 0 || (n_ctx > 0 && !h_ctx)) return RCP_ERR_ARG;
  std::vector<uint32_t> run, spawn;
  int_words(seed, run);
  int_words(purpose, spawn);
  for (int i = 0; i < n_ctx; ++i) int_words(h_ctx[i], spawn);
  if (!spawn.empty() && (int)run.size() < kPool) run.resize(kPool, 0u);
  std::vector<uint32_t> ent(run);
  ent.insert(ent.end(), spawn.begin(), spawn.end());
  uint32_t pool[kPool];
  uint32_t h = kInitA;
  for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u, h);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], h));
  for (size_t s = kPool; s < ent.size(); ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hashmix(ent[s], h));
  uint32_t hb = kInitB;
  uint32_t w[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i % kPool];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  h_key_out[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  h_key_out[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
  return RCP_OK;
}

int rcp_uniform_host(const uint64_t *h_key, int64_t first, int64_t n, double *h_out) {
  if (!h_key || (n > 0 && !h_out) || first < 0 || n < 0) return RCP_ERR_ARG;
  for (int64_t i = 0; i < n; ++i)
    h_out[i] = u64_to_unit(philox_word(h_key[0], h_key[1], (uint64_t)(first + i)));
  return RCP_OK;
}

int rcp_permutation_host(const uint64_t *h_key, int64_t n, int64_t *h_out) {
  if (!h_key || n < 0 || (n > 0 && !h_out)) return RCP_ERR_ARG;
  for (int64_t i = 0; i < n; ++i) h_out[i] = i;
  // Buffered Philox stream: 4 words per block; uint32 draws split a word low half first.
  uint64_t k0 = h_key[0], k1 = h_key[1];
  uint64_t block = 0;
  U64x4 buf;
  int pos = 4;
  bool have32 = false;
  uint32_t hold32 = 0;
  auto next64 = [&]() -> uint64_t {
    if (pos >= 4) {
      U64x4 c;
      c.v[0] = ++block;
      c.v[1] = c.v[2] = c.v[3] = 0;
      buf = philox4x64_10(c, k0, k1);
      pos = 0;
    }
    return buf.v[pos++];
  };
  auto next32 = [&]() -> uint32_t {
    if (have32) {
      have32 = false;
      return hold32;
    }
    uint64_t x = next64();
    have32 = true;
    hold32 = (uint32_t)(x >> 32);
    return (uint32_t)(x & 0xffffffffu);
  };
  for (int64_t i = n - 1; i >= 1; --i) {
    uint64_t mx = (uint64_t)i, mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t j;
    if (mx <= 0xffffffffull) {
      while ((j = (next32() & mask)) > mx) {
      }
    } else {
      while ((j = (next64() & mask)) > mx) {
      }
    }
    int64_t t = h_out[i];
    h_out[i] = h_out[j];
    h_out[j] = t;
  }
  return RCP_OK;
}

// Several permutations at once on native threads: one foreign call (the caller's
// interpreter lock is released once) instead of one call per stream.
int rcp_permutations_host(const uint64_t *h_keys, int count, int64_t n, int64_t *const *h_outs,
                          int threads) {
  if (count < 0 || n < 0 || (count > 0 && (!h_keys || !h_outs))) return RCP_ERR_ARG;
  for (int c = 0; c < count; ++c)
    if (n > 0 && !h_outs[c]) return RCP_ERR_ARG;
  if (threads < 1) threads = 1;
  if (threads > count) threads = count;
  if (threads <= 1) {
    for (int c = 0; c < count; ++c) rcp_permutation_host(h_keys + 2 * c, n, h_outs[c]);
    return RCP_OK;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([=]() {
      for (int c = t; c < count; c += threads) rcp_permutation_host(h_keys + 2 * c, n, h_outs[c]);
    });
  for (auto &th : pool) th.join();
  return RCP_OK;
}

}  // extern "C"

__global__ void uniform_kernel(uint64_t k0, uint64_t k1, int64_t first, int64_t n, double *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = u64_to_unit(philox_word(k0, k1, (uint64_t)(first + i)));
}

extern "C" int rcp_uniform(uint64_t key0, uint64_t key1, int64_t first, int64_t n,
                           double *d_out, void *stream) {
  if (n < 0 || first < 0) return RCP_ERR_ARG;
  if (n == 0) return RCP_OK;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  uniform_kernel<<<(unsigned)blocks, 256, 0, RCP_STREAM(stream)>>>(key0, key1, first, n, d_out);
  RCP_LAUNCH_CHECK("rcp_uniform");
  return RCP_OK;
}
