// Keyed-stream kernels: raw Philox words, numpy-exact bounded integers, and
// per-gid initial membrane potentials (sm/construction.py:361-365).
#include <cstring>
#include "draw_host.cuh"

using namespace smx;

namespace {

__global__ void words_kernel(Key key, uint64_t w0, uint64_t n, uint64_t* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox_word(key, w0 + i);
}

__global__ void fill_i64_kernel(int64_t* out, uint64_t n, int64_t v) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

struct RawSink {
  int64_t lo;
  int64_t* out;
  __device__ __forceinline__ void operator()(uint64_t j, uint32_t v) const { out[j] = lo + (int64_t)v; }
  template <bool ALL>
  __device__ __forceinline__ void batch(uint64_t j0, uint32_t stride, const uint32_t* v, uint32_t ok,
                                        uint32_t* keys) const {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      keys[u] = 0;
      if ((ok >> u) & 1u) out[j0 + (uint64_t)u * stride] = lo + (int64_t)v[u];
    }
  }
};

// Append the decimal form of x (may be negative) to buf at *len.
__device__ __forceinline__ void put_int(uint8_t* buf, uint32_t* len, long long x) {
  char tmp[24];
  int n = 0;
  unsigned long long u = x < 0 ? (unsigned long long)(-(x + 1)) + 1ULL : (unsigned long long)x;
  do { tmp[n++] = (char)('0' + (u % 10)); u /= 10; } while (u);
  if (x < 0) buf[(*len)++] = '-';
  while (n) buf[(*len)++] = (uint8_t)tmp[--n];
}

struct KeyedIdSpec {
  uint8_t prefix[96];
  uint32_t prefix_len;
  uint8_t suffix[16];
  uint32_t suffix_len;
};

// Philox key of RngStream(seed, (..., int_id)) whose canonical bytes are
// prefix + decimal(int_id) + suffix (sm/core.py:99-126).
__device__ __forceinline__ Key keyed_id(const KeyedIdSpec& s, long long id) {
  uint8_t msg[128];
  uint32_t len = 0;
  for (uint32_t i = 0; i < s.prefix_len; ++i) msg[len++] = s.prefix[i];
  put_int(msg, &len, id);
  for (uint32_t i = 0; i < s.suffix_len; ++i) msg[len++] = s.suffix[i];
  for (uint32_t i = len; i < 128; ++i) msg[i] = 0;
  uint64_t m[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    uint64_t w = 0;
#pragma unroll
    for (int b = 7; b >= 0; --b) w = (w << 8) | msg[i * 8 + b];
    m[i] = w;
  }
  return blake2b_128(m, len);
}

// v[i] = mu + sd * z(stream("init-v", gid[i])) -- numpy normal(mu, sd) from a
// fresh stream: the first ziggurat sample of word 0 onward.
__global__ void init_v_kernel(KeyedIdSpec spec, const int64_t* gids, uint64_t n, double mu, double sd,
                              double* v) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  SeqStream s;
  s.init(keyed_id(spec, (long long)gids[i]), 0);
  const double z = zig_standard_normal(s);
  v[i] = __dadd_rn(mu, __dmul_rn(sd, z));
}

__global__ void stream_keys_kernel(KeyedIdSpec spec, const int64_t* ids, uint64_t n, uint64_t* keys) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Key k = keyed_id(spec, (long long)ids[i]);
  keys[2 * i] = k.k0;
  keys[2 * i + 1] = k.k1;
}

int make_spec(const uint8_t* prefix, uint32_t plen, const uint8_t* suffix, uint32_t slen, KeyedIdSpec* s) {
  if (plen > sizeof(s->prefix) || slen > sizeof(s->suffix) || plen + slen + 21 > 127) {
    smx_set_error("stream id too long for the single-block blake2b kernel");
    return -1;
  }
  memset(s, 0, sizeof(*s));
  memcpy(s->prefix, prefix, plen);
  memcpy(s->suffix, suffix, slen);
  s->prefix_len = plen;
  s->suffix_len = slen;
  return 0;
}

}  // namespace

extern "C" int smx_philox_words(uint64_t k0, uint64_t k1, uint64_t w0, uint64_t n, uint64_t* out,
                                void* stream) {
  if (n == 0) return 0;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  smx_count_launch(); words_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(Key{k0, k1}, w0, n, out);
  SMX_LAUNCH_CHECK();
  return 0;
}

// numpy Generator.integers(lo, lo+ex, size=n) from u32 cursor `u32_cursor`;
// returns the cursor after the draws in *cursor_out.
extern "C" int smx_integers(uint64_t k0, uint64_t k1, uint64_t u32_cursor, int64_t lo, uint64_t ex,
                            uint64_t n, int64_t* out, uint64_t* cursor_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (ex == 1) {  // numpy: a one-value range consumes no draws
    if (n) {
      smx_count_launch(); fill_i64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, lo);
      SMX_LAUNCH_CHECK();
    }
    *cursor_out = u32_cursor;
    return 0;
  }
  DrawResult res;
  const int rc = run_draw(Key{k0, k1}, u32_cursor, ex, n, RawSink{lo, out}, st, &res);
  *cursor_out = res.cursor;
  return rc;
}

extern "C" int smx_init_v(const uint8_t* prefix, uint32_t plen, const uint8_t* suffix, uint32_t slen,
                          const int64_t* gids, uint64_t n, double mu, double sd, double* v_out,
                          void* stream) {
  if (n == 0) return 0;
  KeyedIdSpec s;
  if (int rc = make_spec(prefix, plen, suffix, slen, &s)) return rc;
  smx_count_launch(); init_v_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(s, gids, n, mu, sd, v_out);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_stream_keys(const uint8_t* prefix, uint32_t plen, const uint8_t* suffix,
                               uint32_t slen, const int64_t* ids, uint64_t n, uint64_t* keys_out,
                               void* stream) {
  if (n == 0) return 0;
  KeyedIdSpec s;
  if (int rc = make_spec(prefix, plen, suffix, slen, &s)) return rc;
  smx_count_launch(); stream_keys_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(s, ids, n, keys_out);
  SMX_LAUNCH_CHECK();
  return 0;
}
