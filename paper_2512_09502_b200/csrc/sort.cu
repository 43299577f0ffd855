// Stable LSD radix sort of (u32 key, u32 value) records by source node --
// the device form of ConnectionStore.finalize (sm/core.py:299-324):
// "concatenate batches in call order, stable argsort by source, first_index
// via add.at + cumsum".  Records arrive in pending (call, draw) order, so one
// stable sort by final source over that order reproduces the reference's
// table order exactly.
//
// Per 8-bit digit pass (reduce-then-scan):
//   upsweep   per-CTA digit histogram of a contiguous segment
//   scan      exclusive scan over (digit, CTA) -> each CTA's base per digit
//   downsweep CTA walks its segment in 4096-record tiles; warp-striped loads,
//             __match_any_sync ranking (stable), SMEM staging in digit order,
//             coalesced scatter of each digit run.
// Pass 1 resolves temporary keys through the LUT (remote-call records whose
// image ids were assigned after generation).  The last pass writes only
// values and accumulates per-source record counts (one atomic per run of
// equal keys: within a last-pass tile the lower digits are already sorted,
// so equal keys are adjacent in the staging buffer).
#include <algorithm>
#include "common.cuh"

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_IPT = 16;                       // items per thread per tile
constexpr int RS_TILE = RS_THREADS * RS_IPT;     // 4096
constexpr int RS_BINS = 256;

struct SortPass {
  const uint32_t* keys_in;
  const uint32_t* vals_in;  // null: value = record index (first pass only)
  uint32_t* keys_out;       // null on the last pass
  uint32_t* vals_out;
  uint64_t n;
  uint64_t seg;             // records per CTA (multiple of RS_TILE)
  int shift;
  int first;
  int last;
  const uint32_t* lut;      // temporary-key LUT (first pass)
  uint32_t* counts;         // per-key counts (last pass)
  const uint32_t* hist_scan;  // [RS_BINS * G] exclusive offsets
};

__device__ __forceinline__ uint32_t resolve(uint32_t k, const uint32_t* lut) {
  return (k & SMX_TMP_KEY) ? lut[k & ~SMX_TMP_KEY] : k;
}

__global__ void __launch_bounds__(RS_THREADS) upsweep_kernel(SortPass p, uint32_t* hist) {
  __shared__ uint32_t h[RS_BINS];
  for (int i = threadIdx.x; i < RS_BINS; i += RS_THREADS) h[i] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * p.seg;
  const uint64_t hi = lo + p.seg < p.n ? lo + p.seg : p.n;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += RS_THREADS) {
    uint32_t k = p.keys_in[i];
    if (p.first) k = resolve(k, p.lut);
    atomicAdd(&h[(k >> p.shift) & 0xff], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RS_BINS; d += RS_THREADS) hist[(uint64_t)d * gridDim.x + blockIdx.x] = h[d];
}

// Single-CTA exclusive scan of n u32 (n = RS_BINS * G, fits in u32 totals).
__global__ void scan_small_kernel(const uint32_t* in, uint32_t* out, int n) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const uint32_t x = i < n ? in[i] : 0;
    uint32_t tot;
    const uint32_t ex = smx::block_excl_scan(x, ws, tot);
    if (i < n) out[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RS_THREADS) downsweep_kernel(SortPass p) {
  __shared__ uint32_t wcnt[RS_WARPS][RS_BINS];
  __shared__ uint32_t run_base[RS_BINS];
  __shared__ uint32_t tstart[RS_BINS];
  __shared__ uint32_t skey[RS_TILE];
  __shared__ uint32_t sval[RS_TILE];
  __shared__ uint32_t ws[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1;
  for (int d = tid; d < RS_BINS; d += RS_THREADS) run_base[d] = p.hist_scan[(uint64_t)d * gridDim.x + blockIdx.x];
  const uint64_t lo = (uint64_t)blockIdx.x * p.seg;
  const uint64_t hi = lo + p.seg < p.n ? lo + p.seg : p.n;
  for (uint64_t t0 = lo; t0 < hi; t0 += RS_TILE) {
    for (int d = tid; d < RS_WARPS * RS_BINS; d += RS_THREADS) (&wcnt[0][0])[d] = 0;
    __syncthreads();
    uint32_t key[RS_IPT], val[RS_IPT], rank[RS_IPT];
    // warp-striped: warp w owns [t0 + w*512, +512), batch i = 32 consecutive records
#pragma unroll
    for (int i = 0; i < RS_IPT; ++i) {
      const uint64_t idx = t0 + (uint64_t)warp * (32 * RS_IPT) + i * 32 + lane;
      const bool valid = idx < hi;
      uint32_t k = 0, v = 0;
      if (valid) {
        k = p.keys_in[idx];
        if (p.first) k = resolve(k, p.lut);
        v = p.vals_in ? p.vals_in[idx] : (uint32_t)idx;
      }
      key[i] = k;
      val[i] = v;
      const uint32_t d = (k >> p.shift) & 0xff;
      const uint32_t tag = valid ? d : 0x100u + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, tag);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (valid && lane == leader) {
        old = wcnt[warp][d];
        wcnt[warp][d] = old + __popc(peers);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      rank[i] = valid ? old + __popc(peers & lt_mask) : 0xffffffffu;
    }
    __syncthreads();
    // per digit: warp prefixes (in place) and tile totals
    uint32_t total = 0;
    if (tid < RS_BINS) {
      for (int w = 0; w < RS_WARPS; ++w) {
        const uint32_t c = wcnt[w][tid];
        wcnt[w][tid] = total;
        total += c;
      }
    }
    uint32_t tsum;
    const uint32_t ts = smx::block_excl_scan(tid < RS_BINS ? total : 0, ws, tsum);
    if (tid < RS_BINS) tstart[tid] = ts;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RS_IPT; ++i) {
      if (rank[i] != 0xffffffffu) {
        const uint32_t d = (key[i] >> p.shift) & 0xff;
        const uint32_t pos = tstart[d] + wcnt[warp][d] + rank[i];
        skey[pos] = key[i];
        sval[pos] = val[i];
      }
    }
    __syncthreads();
    for (uint32_t q = tid; q < tsum; q += RS_THREADS) {
      const uint32_t k = skey[q];
      const uint32_t d = (k >> p.shift) & 0xff;
      const uint64_t g = (uint64_t)run_base[d] + (q - tstart[d]);
      p.vals_out[g] = sval[q];
      if (!p.last) {
        p.keys_out[g] = k;
      } else if (q == 0 || skey[q - 1] != k) {
        uint32_t e = q + 1;
        while (e < tsum && skey[e] == k) ++e;
        atomicAdd(&p.counts[k], e - q);
      }
    }
    __syncthreads();
    if (tid < RS_BINS) {
      uint32_t c = 0;
      // tile count of digit tid = next tstart - tstart
      const uint32_t nxt = tid + 1 < RS_BINS ? tstart[tid + 1] : tsum;
      c = nxt - tstart[tid];
      run_base[tid] += c;
    }
    __syncthreads();
  }
}

// --- large exclusive scan: counts (u32, n) -> offsets (i64, n+1) -------------
constexpr int SC_THREADS = 1024;
constexpr int SC_ITEMS = 8;

__global__ void scan_reduce_kernel(const uint32_t* in, uint64_t n, uint64_t* part) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * SC_THREADS * SC_ITEMS;
  unsigned long long acc = 0;
  for (int i = 0; i < SC_ITEMS; ++i) {
    const uint64_t idx = base + (uint64_t)i * SC_THREADS + threadIdx.x;
    if (idx < n) acc += in[idx];
  }
  atomicAdd(&s, acc);
  __syncthreads();
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void scan_parts_kernel(uint64_t* part, int np) {
  // single thread: np is small (n / 8192)
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    uint64_t c = 0;
    for (int i = 0; i < np; ++i) {
      const uint64_t x = part[i];
      part[i] = c;
      c += x;
    }
    part[np] = c;
  }
}

__global__ void scan_apply_kernel(const uint32_t* in, uint64_t n, const uint64_t* part, int64_t* out) {
  __shared__ uint32_t ws[32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = part[blockIdx.x];
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * SC_THREADS * SC_ITEMS;
  for (int i = 0; i < SC_ITEMS; ++i) {
    const uint64_t idx = base + (uint64_t)i * SC_THREADS + threadIdx.x;
    const uint32_t x = idx < n ? in[idx] : 0;
    uint32_t tot;
    const uint32_t ex = smx::block_excl_scan(x, ws, tot);
    if (idx < n) out[idx] = (int64_t)(carry + ex);
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (int64_t)carry;
}

}  // namespace

// first_index[0..n] = exclusive scan of counts[0..n-1]; first_index[n] = total.
extern "C" int smx_counts_to_offsets(const uint32_t* counts, uint64_t n, int64_t* first_index, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t per = (uint64_t)SC_THREADS * SC_ITEMS;
  const int nb = (int)((n + per - 1) / per) + (n == 0 ? 1 : 0);
  uint64_t* part = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&part, sizeof(uint64_t) * (nb + 1), st));
  smx_count_launch(); scan_reduce_kernel<<<nb, SC_THREADS, 0, st>>>(counts, n, part);
  smx_count_launch(); scan_parts_kernel<<<1, 32, 0, st>>>(part, nb);
  smx_count_launch(); scan_apply_kernel<<<nb, SC_THREADS, 0, st>>>(counts, n, part, first_index);
  SMX_LAUNCH_CHECK();
  cudaFreeAsync(part, st);
  return 0;
}

// Stable sort of n records by key (key_bits significant bits after LUT
// resolution).  keys_a/vals_a hold the pending records; with index_values the
// initial value of record i is i (vals_a is then only scratch).  keys_b/vals_b
// are scratch of n entries.  The sorted values land in vals_a or vals_b;
// *out_in_b tells which.  counts[0..n_keys) receive per-key record counts.
extern "C" int smx_sort_records(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b,
                                uint64_t n, int key_bits, int index_values, const uint32_t* lut,
                                uint32_t* counts, uint64_t n_keys, int* out_in_b, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  SMX_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * n_keys, st));
  *out_in_b = 0;
  if (n == 0) return 0;
  if (n >= (1ULL << 32)) {
    smx_set_error("smx_sort_records: %llu records exceed the 32-bit record index", (unsigned long long)n);
    return -1;
  }
  const int passes = key_bits <= 8 ? 1 : (key_bits + 7) / 8;
  int G = (int)std::min<uint64_t>((n + RS_TILE - 1) / RS_TILE, 148 * 4);
  if (G < 1) G = 1;
  const uint64_t seg = ((n + G - 1) / G + RS_TILE - 1) / RS_TILE * RS_TILE;
  G = (int)((n + seg - 1) / seg);
  uint32_t *hist = nullptr, *hscan = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&hist, sizeof(uint32_t) * RS_BINS * G, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&hscan, sizeof(uint32_t) * RS_BINS * G, st));
  for (int pass = 0; pass < passes; ++pass) {
    const bool from_a = (pass & 1) == 0;
    SortPass p;
    p.keys_in = from_a ? keys_a : keys_b;
    p.vals_in = (pass == 0 && index_values) ? nullptr : (from_a ? vals_a : vals_b);
    p.first = pass == 0;
    p.last = pass == passes - 1;
    p.shift = 8 * pass;
    p.n = n;
    p.seg = seg;
    p.lut = lut;
    p.counts = counts;
    p.hist_scan = hscan;
    p.keys_out = p.last ? nullptr : (from_a ? keys_b : keys_a);
    p.vals_out = from_a ? vals_b : vals_a;
    smx_count_launch(); upsweep_kernel<<<G, RS_THREADS, 0, st>>>(p, hist);
    smx_count_launch(); scan_small_kernel<<<1, 1024, 0, st>>>(hist, hscan, RS_BINS * G);
    smx_count_launch(); downsweep_kernel<<<G, RS_THREADS, 0, st>>>(p);
    SMX_LAUNCH_CHECK();
    *out_in_b = from_a ? 1 : 0;
  }
  cudaFreeAsync(hist, st);
  cudaFreeAsync(hscan, st);
  return 0;
}
