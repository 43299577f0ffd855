// Stable LSD radix sort of (u32 key, u32 value) records by source node --
// the device form of ConnectionStore.finalize (sm/core.py:299-324):
// "concatenate batches in call order, stable argsort by source, first_index
// via add.at + cumsum".  Records arrive in pending (call, draw) order, so one
// stable sort by final source over that order reproduces the reference's
// table order exactly.
//
// ceil(key_bits / 11) passes of equal digit width (<= 11 bits), each a
// reduce-then-scan:
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
#include <cstdlib>
#include "common.cuh"

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_IPT = 16;                       // items per thread per tile
constexpr int RS_TILE = RS_THREADS * RS_IPT;     // 4096
constexpr int RS_MAX_BITS = 11;

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
  const uint32_t* hist_scan;  // [BINS * G] exclusive offsets
  unsigned long long* timing; // optional per-phase cycle counters (tuning)
};

__device__ __forceinline__ uint32_t resolve(uint32_t k, const uint32_t* lut) {
  return (k & SMX_TMP_KEY) ? lut[k & ~SMX_TMP_KEY] : k;
}

template <int BITS>
__global__ void __launch_bounds__(RS_THREADS) upsweep_kernel(SortPass p, uint32_t* hist) {
  constexpr int BINS = 1 << BITS;
  __shared__ uint32_t h[BINS];
  for (int i = threadIdx.x; i < BINS; i += RS_THREADS) h[i] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * p.seg;
  const uint64_t hi = lo + p.seg < p.n ? lo + p.seg : p.n;
  const uint32_t mask = BINS - 1;
  // 4-wide vector loads (segments are multiples of 4096 records)
  const uint4* k4 = reinterpret_cast<const uint4*>(p.keys_in);
  for (uint64_t i = lo / 4 + threadIdx.x; i < (hi + 3) / 4; i += RS_THREADS) {
    const uint4 q = k4[i];
    const uint32_t kk[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i * 4 + j >= hi) break;
      uint32_t k = kk[j];
      if (p.first) k = resolve(k, p.lut);
      atomicAdd(&h[(k >> p.shift) & mask], 1u);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) hist[(uint64_t)d * gridDim.x + blockIdx.x] = h[d];
}

// Single-CTA exclusive scan of n u32 (n = BINS * G, totals fit in u32).
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

// Stable scatter of one segment per CTA by the digit (key >> shift) & (2^BITS-1).
// Input tiles are double-buffered in shared memory by TMA 1-D bulk copies
// (cp.async.bulk + mbarrier): tile i+1 streams in while tile i is ranked and
// scattered, so the warps never wait on DRAM for their inputs.
template <int BITS>
__global__ void __launch_bounds__(RS_THREADS, 2) downsweep_kernel(SortPass p) {
  constexpr int BINS = 1 << BITS;
  constexpr int DPT = BINS >= RS_THREADS ? BINS / RS_THREADS : 1;  // digits per thread
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* inbuf = reinterpret_cast<uint32_t*>(smem);                      // [2][2][RS_TILE] keys, vals
  uint32_t* skey = inbuf + 4 * RS_TILE;                                     // [RS_TILE]
  uint32_t* sval = skey + RS_TILE;                                          // [RS_TILE]
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(sval + RS_TILE);             // [RS_WARPS][BINS]
  uint32_t* run_base = reinterpret_cast<uint32_t*>(wcnt + RS_WARPS * BINS);  // [BINS]
  uint32_t* tstart = run_base + BINS;                                       // [BINS + 1]
  __shared__ uint32_t ws[32];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1;
  const uint32_t mask = BINS - 1;
  for (int d = tid; d < BINS; d += RS_THREADS) run_base[d] = p.hist_scan[(uint64_t)d * gridDim.x + blockIdx.x];
  const uint64_t lo = (uint64_t)blockIdx.x * p.seg;
  const uint64_t hi = lo + p.seg < p.n ? lo + p.seg : p.n;
  const bool has_vals = p.vals_in != nullptr;
  if (tid == 0) {
    smx::mbar_init(&bar[0], 1);
    smx::mbar_init(&bar[1], 1);
    smx::fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint64_t t0, int b) {  // thread 0: full tiles only
    const uint32_t bytes = RS_TILE * 4;
    smx::mbar_expect_tx(&bar[b], has_vals ? 2 * bytes : bytes);
    smx::bulk_g2s(inbuf + (2 * b) * RS_TILE, p.keys_in + t0, bytes, &bar[b]);
    if (has_vals) smx::bulk_g2s(inbuf + (2 * b + 1) * RS_TILE, p.vals_in + t0, bytes, &bar[b]);
  };
  uint32_t phase[2] = {0, 0};
  if (tid == 0 && lo + RS_TILE <= hi) issue(lo, 0);
  long long tm = clock64();
#define TMARK(i)                                                     \
  if (p.timing && tid == 0) {                                        \
    const long long t_ = clock64();                                  \
    atomicAdd(p.timing + (i), (unsigned long long)(t_ - tm));        \
    tm = t_;                                                         \
  }
  int b = 0;
  for (uint64_t t0 = lo; t0 < hi; t0 += RS_TILE, b ^= 1) {
    const bool full = t0 + RS_TILE <= hi;
    uint32_t* kin = inbuf + (2 * b) * RS_TILE;
    uint32_t* vin = kin + RS_TILE;
    // prefetch the next tile into the other buffer (consumed two iterations ago)
    if (tid == 0 && t0 + 2 * RS_TILE <= hi) {
      smx::fence_proxy_async();
      issue(t0 + RS_TILE, b ^ 1);
    }
    TMARK(5);
    if (full) {
      smx::mbar_wait(&bar[b], phase[b]);
      phase[b] ^= 1;
    } else {  // partial last tile: plain loads
      for (uint32_t q = tid; q < RS_TILE; q += RS_THREADS) {
        const uint64_t idx = t0 + q;
        kin[q] = idx < hi ? p.keys_in[idx] : 0u;
        if (has_vals) vin[q] = idx < hi ? p.vals_in[idx] : 0u;
      }
    }
    for (int d = tid; d < RS_WARPS * BINS / 2; d += RS_THREADS) reinterpret_cast<uint32_t*>(wcnt)[d] = 0;
    __syncthreads();
    TMARK(0);
    uint32_t rank2[RS_IPT / 2];  // two 16-bit ranks per register; 0xffff = invalid
    const uint32_t wofs = warp * (32 * RS_IPT) + lane;
#pragma unroll
    for (int i = 0; i < RS_IPT; ++i) {
      const uint32_t q = wofs + i * 32;
      const bool valid = t0 + q < hi;
      uint32_t k = kin[q];
      if (p.first) {
        k = resolve(k, p.lut);
        kin[q] = k;  // later phases reread the resolved key
      }
      const uint32_t d = (k >> p.shift) & mask;
      // warp-level multisplit: lanes with the same digit, one ballot per bit
      // (cheaper than MATCH.ANY on sm_100)
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < BITS; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      if (!valid) peers = 1u << lane;
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (valid && lane == leader) {
        old = wcnt[warp * BINS + d];
        wcnt[warp * BINS + d] = (uint16_t)(old + __popc(peers));
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      const uint32_t r = valid ? old + __popc(peers & lt_mask) : 0xffffu;
      if (i & 1) rank2[i >> 1] |= r << 16; else rank2[i >> 1] = r;
    }
    __syncthreads();
    TMARK(1);
    // digits [tid*DPT, tid*DPT+DPT): warp prefixes in place, tile totals, block scan
    uint32_t tot_d[DPT];
    uint32_t mysum = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      uint32_t t = 0;
      if (d < BINS) {
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
          const uint32_t c = wcnt[w * BINS + d];
          wcnt[w * BINS + d] = (uint16_t)t;
          t += c;
        }
      }
      tot_d[j] = t;
      mysum += t;
    }
    uint32_t tsum;
    uint32_t run = smx::block_excl_scan(mysum, ws, tsum);
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      if (d < BINS) tstart[d] = run;
      run += tot_d[j];
    }
    if (tid == 0) tstart[BINS] = tsum;
    __syncthreads();
    TMARK(2);
#pragma unroll
    for (int i = 0; i < RS_IPT; ++i) {
      const uint32_t r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
      if (r != 0xffffu) {
        const uint32_t q = wofs + i * 32;
        const uint32_t k = kin[q];
        const uint32_t d = (k >> p.shift) & mask;
        const uint32_t pos = tstart[d] + wcnt[warp * BINS + d] + r;
        skey[pos] = k;
        sval[pos] = has_vals ? vin[q] : (uint32_t)(t0 + q);
      }
    }
    __syncthreads();
    TMARK(3);
    for (uint32_t q0 = 0; q0 < tsum; q0 += RS_THREADS) {
      const uint32_t q = q0 + tid;
      const bool ok = q < tsum;
      const uint32_t k = ok ? skey[q] : 0xffffffffu;
      if (ok) {
        const uint32_t d = (k >> p.shift) & mask;
        const uint64_t g = (uint64_t)run_base[d] + (q - tstart[d]);
        p.vals_out[g] = sval[q];
        if (!p.last) p.keys_out[g] = k;
      }
      if (p.last) {
        // per-source counts: equal keys are adjacent in the staging buffer,
        // so one warp-aggregated atomic per distinct key per warp
        const uint32_t peers = __match_any_sync(0xffffffffu, k);
        if (ok && lane == __ffs(peers) - 1) atomicAdd(&p.counts[k], (uint32_t)__popc(peers));
      }
    }
    __syncthreads();
    TMARK(4);
    for (int d = tid; d < BINS; d += RS_THREADS) run_base[d] += tstart[d + 1] - tstart[d];
    __syncthreads();
  }
}

template <int BITS>
size_t downsweep_smem() {
  return (size_t)6 * RS_TILE * 4 + (size_t)RS_WARPS * (1 << BITS) * 2 + (size_t)(2 * (1 << BITS) + 1) * 4;
}

template <int BITS>
int run_pass(const SortPass& p, int G, uint32_t* hist, uint32_t* hscan, cudaStream_t st) {
  const size_t smem = downsweep_smem<BITS>();
  static bool configured = false;
  if (!configured) {
    SMX_CUDA_CHECK(cudaFuncSetAttribute(downsweep_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    configured = true;
  }
  smx_count_launch(); upsweep_kernel<BITS><<<G, RS_THREADS, 0, st>>>(p, hist);
  smx_count_launch(); scan_small_kernel<<<1, 1024, 0, st>>>(hist, hscan, (1 << BITS) * G);
  smx_count_launch(); downsweep_kernel<BITS><<<G, RS_THREADS, smem, st>>>(p);
  SMX_LAUNCH_CHECK();
  return 0;
}

int run_pass_bits(int bits, const SortPass& p, int G, uint32_t* hist, uint32_t* hscan, cudaStream_t st) {
  switch (bits) {
    case 1: case 2: case 3: case 4: case 5: case 6: case 7:
    case 8: return run_pass<8>(p, G, hist, hscan, st);
    case 9: return run_pass<9>(p, G, hist, hscan, st);
    case 10: return run_pass<10>(p, G, hist, hscan, st);
    default: return run_pass<11>(p, G, hist, hscan, st);
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

static unsigned long long* g_sort_timing = nullptr;
// Tuning aid: per-phase cycle counters of the downsweep (thread 0 of every
// CTA; phases: zero, rank, scan, stage, write, wait).  Pass null to disable.
extern "C" void smx_sort_timing(unsigned long long* counters) { g_sort_timing = counters; }

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
// resolution) in ceil(key_bits / 11) passes of equal digit width.
// keys_a/vals_a hold the pending records; with index_values the initial
// value of record i is i (vals_a is then only scratch).  keys_b/vals_b are
// scratch of n entries.  The sorted values land in vals_a or vals_b;
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
  if (key_bits < 1) key_bits = 1;
  static const int max_bits = getenv("SMX_SORT_MAX_BITS") ? atoi(getenv("SMX_SORT_MAX_BITS")) : RS_MAX_BITS;
  static const int grid_cap = getenv("SMX_SORT_GRID") ? atoi(getenv("SMX_SORT_GRID")) : 148 * 2;
  const int passes = (key_bits + max_bits - 1) / max_bits;
  const int bits = (key_bits + passes - 1) / passes;
  int G = (int)std::min<uint64_t>((n + RS_TILE - 1) / RS_TILE, grid_cap);
  if (G < 1) G = 1;
  const uint64_t seg = ((n + G - 1) / G + RS_TILE - 1) / RS_TILE * RS_TILE;
  G = (int)((n + seg - 1) / seg);
  uint32_t *hist = nullptr, *hscan = nullptr;
  const size_t hn = (size_t)(1 << std::max(bits, 8)) * G;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&hist, sizeof(uint32_t) * hn, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&hscan, sizeof(uint32_t) * hn, st));
  for (int pass = 0; pass < passes; ++pass) {
    const bool from_a = (pass & 1) == 0;
    SortPass p;
    p.keys_in = from_a ? keys_a : keys_b;
    p.vals_in = (pass == 0 && index_values) ? nullptr : (from_a ? vals_a : vals_b);
    p.first = pass == 0;
    p.last = pass == passes - 1;
    p.shift = bits * pass;
    p.n = n;
    p.seg = seg;
    p.lut = lut;
    p.counts = counts;
    p.hist_scan = hscan;
    p.timing = g_sort_timing;
    p.keys_out = p.last ? nullptr : (from_a ? keys_b : keys_a);
    p.vals_out = from_a ? vals_b : vals_a;
    if (int rc = run_pass_bits(bits, p, G, hist, hscan, st)) return rc;
    *out_in_b = from_a ? 1 : 0;
  }
  cudaFreeAsync(hist, st);
  cudaFreeAsync(hscan, st);
  return 0;
}
