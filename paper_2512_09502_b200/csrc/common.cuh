// Shared device helpers for the spikemesh-b200 kernels (sm_100a).
//
// Random arithmetic restates numpy 2.3.5's Philox4x64-10 bit generator and
// its consumers exactly (the reference draws every random number through
// numpy.random.Generator(Philox), sm/core.py:119-141):
//   word w of a stream      = Philox4x64_10(ctr = w/4 + 1, key)[w % 4]
//   u32 position u          = low half of word u/2 if u even, else high half
//   next_double(word)       = (word >> 11) * 2^-53
//   integers(lo, lo+ex)     = 32-bit Lemire; a u32 draw v is accepted iff
//                             (v*ex mod 2^32) >= (2^32-ex) % ex, value = v*ex >> 32
// Floating-point arithmetic that must match numpy bit-for-bit is written
// with explicit round-to-nearest intrinsics (no FMA contraction).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define SMX_PHILOX_M0 0xD2E7470EE14C6C93ULL
#define SMX_PHILOX_M1 0xCA5A826395121157ULL
#define SMX_PHILOX_W0 0x9E3779B97F4A7C15ULL
#define SMX_PHILOX_W1 0xBB67AE8584CAA73BULL

// Packed record payload: target row (24 bits) | syn class (8 bits).
#define SMX_ROW_BITS 24
#define SMX_ROW_MASK 0x00FFFFFFu
// Pending-record keys with this bit set are temporary keys resolved through
// the per-rank key LUT at sort time (remote-call records whose image ids are
// assigned after generation).
#define SMX_TMP_KEY 0x80000000u

namespace smx {

struct Key {
  uint64_t k0, k1;
};

__device__ __forceinline__ void philox4x64_10(uint64_t block, Key key, uint64_t out[4]) {
  uint64_t c0 = block, c1 = 0, c2 = 0, c3 = 0;
  uint64_t k0 = key.k0, k1 = key.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += SMX_PHILOX_W0; k1 += SMX_PHILOX_W1; }
    const uint64_t hi0 = __umul64hi(SMX_PHILOX_M0, c0), lo0 = SMX_PHILOX_M0 * c0;
    const uint64_t hi1 = __umul64hi(SMX_PHILOX_M1, c2), lo1 = SMX_PHILOX_M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__device__ __forceinline__ uint64_t philox_word(Key key, uint64_t w) {
  uint64_t b[4];
  philox4x64_10((w >> 2) + 1, key, b);
  return b[w & 3];
}

__device__ __forceinline__ double u53(uint64_t w) {
  return __dmul_rn((double)(w >> 11), 1.0 / 9007199254740992.0);
}

struct Lemire {
  uint32_t ex;         // range size, 2 <= ex <= 2^32-1; ex==0 encodes 2^32
  uint32_t threshold;  // (2^32 - ex) % ex
  __device__ __forceinline__ bool accept(uint32_t v, uint32_t& out) const {
    if (ex == 0) { out = v; return true; }
    const uint64_t m = (uint64_t)v * (uint64_t)ex;
    out = (uint32_t)(m >> 32);
    return (uint32_t)m >= threshold;
  }
};

// A sequential stream cursor on the device (one thread), mirroring numpy's
// Philox state: 64-bit word position plus the buffered high half.
struct SeqStream {
  Key key;
  uint64_t word;   // next 64-bit word index
  uint64_t buf[4];
  uint64_t bufblk; // block index held in buf (0 = none)
  __device__ __forceinline__ void init(Key k, uint64_t w) { key = k; word = w; bufblk = 0; }
  __device__ __forceinline__ uint64_t next64() {
    const uint64_t blk = (word >> 2) + 1;
    if (blk != bufblk) { philox4x64_10(blk, key, buf); bufblk = blk; }
    return buf[(word++) & 3];
  }
  __device__ __forceinline__ double next_double() { return u53(next64()); }
};

// ---------------------------------------------------------------------------
// Ziggurat standard normal (numpy random_standard_normal).  The tail value
// uses glibc's log1p restated bit for bit (below); the wedge's exp only
// enters a comparison, which could only differ when both sides lie within
// one ulp of each other.
// ---------------------------------------------------------------------------
}  // namespace smx

#include "ziggurat_tables.cuh"

namespace smx {

// log1p(x) for x in (-1, 0] exactly as the x86-64 glibc (2.39) that numpy's
// npy_log1p calls on an FMA-capable host: libm's ifunc picks the FMA build of
// sysdeps/ieee754/dbl-64/s_log1p.c, transcribed here operation for operation
// from that build (contractions included).  CUDA's log1p is faithfully rounded
// but differs from glibc's in the last bit often enough to change ziggurat
// tail values (tests/test_gpu_rng.py::test_normal_slow_paths_at_scale); this
// one was checked against glibc on 2e8 arguments -u, u = k 2^-53 (0 mismatches).
__device__ __forceinline__ double glibc_log1p_neg(double x) {
  const uint32_t hx = (uint32_t)((uint64_t)__double_as_longlong(x) >> 32);
  if ((hx & 0x7fffffffu) < 0x3e200000u) {  // |x| < 2^-29
    if ((hx & 0x7fffffffu) < 0x3c900000u) return x;
    return __fma_rn(-__dmul_rn(x, x), 0.5, x);
  }
  const double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
  int k;
  double f, hfsq, c = 0.0;
  uint32_t hu;
  if (hx + 0x402d413cu <= 0x402d413cu) {  // x <= -0.2929: k != 0
    double u = __dadd_rn(x, 1.0);
    hu = (uint32_t)((uint64_t)__double_as_longlong(u) >> 32);
    k = (int)(hu >> 20) - 1023;
    c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
    c = __ddiv_rn(c, u);
    hu &= 0xfffffu;
    const uint64_t lo = (uint64_t)__double_as_longlong(u) & 0xffffffffull;
    if (hu > 0x6a09du) {
      k += 1;
      u = __longlong_as_double((long long)(((uint64_t)(hu | 0x3fe00000u) << 32) | lo));
      hu = (0x100000u - hu) >> 2;
    } else {
      u = __longlong_as_double((long long)(((uint64_t)(hu | 0x3ff00000u) << 32) | lo));
    }
    f = __dsub_rn(u, 1.0);
    hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
    if (hu == 0) {
      const double dk = (double)k;
      if (f == 0.0) return __fma_rn(dk, LN2_HI, __fma_rn(dk, LN2_LO, c));
      const double R = __dmul_rn(__fma_rn(-f, 6.66666666666666629659e-01, 1.0), hfsq);
      return __fma_rn(dk, LN2_HI, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, LN2_LO, c)), f));
    }
  } else {
    k = 0;
    f = x;
    hfsq = __dmul_rn(__dmul_rn(x, 0.5), x);
  }
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double R2 = __fma_rn(z, 2.857142874366239149e-01, 3.999999999940941908e-01);
  const double R3 = __fma_rn(z, 1.818357216161805012e-01, 2.222219843214978396e-01);
  const double R4 = __fma_rn(z, 1.479819860511658591e-01, 1.531383769920937332e-01);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  const double R =
      __fma_rn(z6, R4, __fma_rn(z4, R3, __fma_rn(z, 6.666666666666735130e-01, __dmul_rn(z2, R2))));
  const double t = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  const double dk = (double)k;
  const double a = __dadd_rn(__fma_rn(dk, LN2_LO, c), t);
  return __fma_rn(dk, LN2_HI, -__dsub_rn(__dsub_rn(hfsq, a), f));
}

// The ziggurat's first word alone: true (and x) when it is accepted there --
// the 98.5% fast path, one word consumed (zig_standard_normal's first step).
__device__ __forceinline__ bool zig_first(uint64_t r, double& x) {
  const int idx = (int)(r & 0xff);
  r >>= 8;
  const int sign = (int)(r & 1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  x = __dmul_rn((double)rabs, __longlong_as_double((long long)ZIG_WI_DOUBLE_BITS[idx]));
  if (sign) x = -x;
  return rabs < ZIG_KI_DOUBLE_BITS[idx];
}

__device__ __forceinline__ double zig_standard_normal(SeqStream& s) {
  for (;;) {
    uint64_t r = s.next64();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, __longlong_as_double((long long)ZIG_WI_DOUBLE_BITS[idx]));
    if (sign) x = -x;
    if (rabs < ZIG_KI_DOUBLE_BITS[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-ZIG_NOR_INV_R, glibc_log1p_neg(-s.next_double()));
        const double yy = -glibc_log1p_neg(-s.next_double());
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 1) ? -__dadd_rn(ZIG_NOR_R, xx) : __dadd_rn(ZIG_NOR_R, xx);
      }
    } else {
      const double f0 = __longlong_as_double((long long)ZIG_FI_DOUBLE_BITS[idx - 1]);
      const double f1 = __longlong_as_double((long long)ZIG_FI_DOUBLE_BITS[idx]);
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(f0, f1), s.next_double()), f1);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    }
  }
}

// ---------------------------------------------------------------------------
// BLAKE2b-128 of a short message (< 128 bytes, one block), used to derive the
// per-neuron ("init-v", gid) Philox keys on the device (sm/core.py:119-126).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

__device__ __constant__ uint64_t BLAKE2B_IV[8] = {
    0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL, 0xa54ff53a5f1d36f1ULL,
    0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL, 0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};

__device__ __constant__ uint8_t BLAKE2B_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

// msg: little-endian message words (16 x u64, zero padded), len in bytes.
__device__ inline Key blake2b_128(const uint64_t m[16], uint32_t len) {
  uint64_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = BLAKE2B_IV[i];
  h[0] ^= 0x01010000ULL ^ 16ULL;  // digest 16, key 0, fanout 1, depth 1
  uint64_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[i + 8] = BLAKE2B_IV[i]; }
  v[12] ^= (uint64_t)len;
  v[14] = ~v[14];  // final block
#define SMX_G(a, b, c, d, x, y)            \
  a = a + b + x; d = rotr64(d ^ a, 32);    \
  c = c + d;     b = rotr64(b ^ c, 24);    \
  a = a + b + y; d = rotr64(d ^ a, 16);    \
  c = c + d;     b = rotr64(b ^ c, 63);
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = BLAKE2B_SIGMA[r];
    SMX_G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
    SMX_G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
    SMX_G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
    SMX_G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
    SMX_G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
    SMX_G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
    SMX_G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
    SMX_G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
  }
#undef SMX_G
  Key k;
  k.k0 = h[0] ^ v[0] ^ v[8];
  k.k1 = h[1] ^ v[1] ^ v[9];
  return k;
}

// Division of u32 by an invariant divisor without the (slow, software) integer
// divide: Granlund-Montgomery round-up multiplier, exact for every n < 2^32.
struct FastDiv {
  uint32_t d, m;
  int l;
  __host__ __device__ static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d ? d : 1;
    int l = 0;
    while ((1ULL << l) < f.d) ++l;
    f.l = l;
    f.m = (uint32_t)(((1ULL << 32) * ((1ULL << l) - f.d)) / f.d + 1);
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (l == 0) return n;
    const uint32_t t = __umulhi(m, n);
    return (t + ((n - t) >> 1)) >> (l - 1);
  }
};

// TMA 1-D bulk copies (cp.async.bulk) with mbarrier completion --------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy; bytes and both addresses multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p; SMX_WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra SMX_WAIT_%=; }" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Warp/block scan helpers -----------------------------------------------------
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Exclusive block scan of one value per thread; returns exclusive prefix and
// writes the block total.  `ws` needs blockDim.x/32 entries of scratch.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* ws, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t inc = warp_incl_scan(x);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < nw ? ws[lane] : 0;
    t = warp_incl_scan(t);
    if (lane < nw) ws[lane] = t;
  }
  __syncthreads();
  total = ws[nw - 1];
  const uint32_t base = warp ? ws[warp - 1] : 0;
  __syncthreads();
  return base + inc - x;
}

}  // namespace smx

// Error reporting and the kernel-launch counter shared by every translation
// unit (defined in capi.cu).
extern "C" void smx_set_error(const char* fmt, ...);
extern "C" void smx_count_launch(void);
// pinned-staged host -> device copy (capi.cu): never blocks the host
int smx_h2d_async(void* dst, const void* src, size_t bytes, cudaStream_t st);
// long persistent kernel in flight (capi.cu): smx_long_kernel_mark records
// its end; smx_grid_cap(grid, cap) returns min(grid, cap) while it runs
void smx_long_kernel_mark(cudaStream_t st);
// draw chaining (capi.cu, smx_draw_chain): taken once by the next run_draw
void smx_take_draw_chain(const uint64_t** u0_dev, uint64_t** cursor_dev);
int smx_chain_passthrough(const uint64_t* u0_dev, uint64_t u0, uint64_t* cursor_dev, cudaStream_t st);
// Scope of one chainable entry point: whatever path it returns by, a chain
// setting it did not take does not leak into the next call.
struct DrawChainScope {
  ~DrawChainScope() {
    const uint64_t* a;
    uint64_t* b;
    smx_take_draw_chain(&a, &b);
  }
};
int smx_grid_cap(int grid, int concurrent_cap);
int smx_pass_a_free_slots();   // fused.cu: CTA slots pass A leaves free
extern "C" int* smx_device_error_word(void);
// Kernel attributes (dynamic SMEM limits) are per device: launchers keep one
// bit per device in a static mask and set the attribute the first time they
// launch on each device.
inline unsigned long long smx_device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}
#define SMX_CUDA_CHECK(expr)                                                       \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      smx_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return -3;                                                                   \
    }                                                                              \
  } while (0)
#define SMX_LAUNCH_CHECK()                                                         \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      smx_set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return -3;                                                                   \
    }                                                                              \
  } while (0)
