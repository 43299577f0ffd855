// Fused construction path: connectivity generation fused into the first pass
// of the stable LSD sort (SURVEY §7 hard part 3).
//
// The reference realises a fixed-in-degree call as `integers(0, total, K*N)`
// target-major draws (sm/construction.py:391-406, 640-703), appends the
// records in call order and finally sorts them stably by source
// (ConnectionStore.finalize, sm/core.py:299-324).  A stable LSD radix sort
// of the records over their (call, draw) order reproduces that table, and its
// first pass only needs each record's low key digit -- which the draw itself
// produces.  So instead of writing (key, payload) records and re-reading them:
//
//   pass A (fused_gen_kernel, one launch per call, at prepare time)
//     draws a tile of 8192 raw u32 positions once (Philox4x64-10 + Lemire),
//     maps accepted values to final source keys, ranks the tile's records
//     stably by the low key digit (ballot multisplit), finds each digit's
//     position across tiles with a decoupled look-back (tiles taken in order
//     from a ticket) and writes one packed u32 per record into that digit's
//     region:  rec = (key >> lo_bits) << pbits | compact payload, the compact
//     payload being the target row and a per-rank class index.
//     Regions are sized from the exact digit probabilities of the call's
//     source-value -> key map (expectation + 8 sigma); an overflow sets a flag
//     and the engine rebuilds the rank through the general path.
//   pass B (smx_fused_sort)
//     per 3840-record tile of a region: histogram of the high digit
//     (fb_hist), per-region / per-digit scans (per-key counts for
//     first_index fall out of the same sums), then a stable scatter by the
//     high digit that writes the final payload (row | global class << 24)
//     (fb_scatter, TMA tile loads, coalesced digit runs).
//
// Record bytes: pass A writes 4 B, pass B reads 4 B twice and writes 4 B
// (16 B/synapse against 51 B for generate-then-sort with 8-byte records).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>
#include "common.cuh"

using namespace smx;

namespace {

// ------------------------------------------------------------------ pass A
// 256 threads x 32 positions, 3 CTAs per SM (measured: pass A 10.3 -> 9.0 ms
// on C3 against 512 x 16 x 2; 256 x 32 x 2 and x 4 were slower)
#ifndef SMX_FG_THREADS
#define SMX_FG_THREADS 256
#endif
#ifndef SMX_FG_IPT
#define SMX_FG_IPT 32
#endif
constexpr int FG_THREADS = SMX_FG_THREADS;
constexpr int FG_WARPS = FG_THREADS / 32;
constexpr int FG_IPT = SMX_FG_IPT;               // raw positions per thread per tile (multiple of 8)
constexpr int FG_TILE = FG_THREADS * FG_IPT;     // 8192 raw u32 positions per tile
constexpr int FG_XS = FG_TILE + FG_TILE / 32;    // padded transpose buffer
constexpr uint32_t FG_NOKEY = 0xFFFFFFFFu;       // rejected draw / outside the window
constexpr uint32_t FG_SENTINEL = 0xFFFFFFFFu;    // accepted draw past the call's last record
constexpr uint32_t ST_A = 1u << 30, ST_P = 2u << 30, ST_VAL = (1u << 30) - 1;
constexpr int FG_MAXP = 8;
#ifndef SMX_FG_MIN_BLOCKS
#define SMX_FG_MIN_BLOCKS 3
#endif
static_assert(FG_IPT == 8 || FG_IPT == 16 || FG_IPT == 32, "padded transpose: a thread's run never crosses a pad word");
#ifndef SMX_FG_LB_WIN
#define SMX_FG_LB_WIN 4   // look-back descriptors read per step
#endif
#ifndef SMX_FG_LB_SLEEP
#define SMX_FG_LB_SLEEP 64   // ns a look-back step backs off when its predecessor is still drawing
#endif
#ifndef SMX_FG_FREE_SMS
#define SMX_FG_FREE_SMS 8
#endif

struct FusedGen {
  Key key;
  Lemire lm;
  uint64_t n_raw;     // raw u32 positions of the window (from stream position 0)
  uint64_t n_out;     // records of the call
  uint32_t np;        // key pieces (key mode 3)
  uint32_t pstart[FG_MAXP], pdelta[FG_MAXP];
  const uint32_t* key_tab;  // key mode 1: key = key_tab[value]
  uint32_t kdiv;      // k_in: target index = j / kdiv
  FastDiv kd;
  const uint32_t* pay;   // payload of each target index (row | class << 24, smx_pay_table)
  uint32_t cls_field;    // this call's class index << its row bits (the record's payload field)
  int pbits;          // bits below the high key digit in a record
  uint32_t* region;
  const uint64_t* rstart;   // [B] first slot of each digit region
  const uint64_t* rcap;     // [B] capacity of each region (records)
  const uint64_t* fill_in;  // [B] records already in the region (earlier calls)
  uint64_t* fill_out;       // [B] after this call (written by the last tile)
  uint32_t* status;         // [n_tiles][B] look-back descriptors
  uint32_t* ticket;
  uint64_t* total;          // accepted draws in the window (last tile)
  int* overflow;
  uint32_t free_sms;        // SMs 148 - free_sms .. 147 left empty (0: all SMs work)
};

// SMs pass A leaves to concurrent work (replays of later calls), per process
// (smx_set_pass_a_free_sms; SMX_FG_FREE_SMS by default).
static int g_fg_free_sms = SMX_FG_FREE_SMS;

// KM 1: key table; 3: piecewise-affine pieces; 4: a single piece (key = v + delta)
template <int KM>
__device__ __forceinline__ uint32_t fg_key(const FusedGen& g, uint32_t v) {
  if (KM == 1) return __ldg(g.key_tab + v);
  if (KM == 4) return v + g.pdelta[0];
  if (KM == 5) return v + (v >= g.pstart[1] ? g.pdelta[1] : g.pdelta[0]);   // two pieces
  if (KM == 6) {  // up to four pieces (padding starts never reached: ex < 2^32)
    uint32_t off = g.pdelta[0];
    off = v >= g.pstart[1] ? g.pdelta[1] : off;
    off = v >= g.pstart[2] ? g.pdelta[2] : off;
    off = v >= g.pstart[3] ? g.pdelta[3] : off;
    return v + off;
  }
  uint32_t off = g.pdelta[0];
#pragma unroll
  for (int s = 1; s < FG_MAXP; ++s)
    if (s < (int)g.np && v >= g.pstart[s]) off = g.pdelta[s];
  return v + off;
}

__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) { return *(const volatile uint32_t*)p; }
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) { *(volatile uint32_t*)p = v; }

// Stable rank of one item per lane among the warp's items with the same
// digit (ballot multisplit, as in sort.cu) against the warp's SMEM counters.
#ifndef SMX_MATCH_RANK
#define SMX_MATCH_RANK 0   // 1: __match_any_sync instead of one ballot per digit bit (A/B)
#endif
template <int LB>
__device__ __forceinline__ uint32_t fg_rank(uint32_t d, bool valid, uint32_t vm, uint16_t* mycnt, int lane,
                                            uint32_t lt) {
  uint32_t peers = vm;
  if (SMX_MATCH_RANK) {
    peers = __match_any_sync(0xffffffffu, valid ? d : 0xffffffffu) & vm;
  } else {
#pragma unroll
  for (int b = 0; b < LB; ++b) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bal;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 bal, p, 0xffffffff;\n\t"
        "@!p not.b32 bal, bal;\n\t"
        "and.b32 %0, %0, bal;\n\t}"
        : "+r"(peers) : "r"(d), "r"(1u << b));
  }
  }
  if (!valid) peers = 1u << lane;
  const int leader = __ffs(peers) - 1;
  uint32_t old = 0;
  if (valid && lane == leader) {
    old = mycnt[d];
    mycnt[d] = (uint16_t)(old + __popc(peers));
  }
  old = __shfl_sync(0xffffffffu, old, leader);
  return valid ? old + __popc(peers & lt) : 0xffffu;
}

#ifdef SMX_FG_LBSTAT   // tuning aid: look-back statistics of digit 0 (tiles, steps, descriptors, waits)
__device__ unsigned long long g_fg_lbstat[4];
#endif

// WIDE: region slots may exceed 2^31 (64-bit staging offsets)
template <int KM, int LB, bool WIDE>
__global__ void __launch_bounds__(FG_THREADS, SMX_FG_MIN_BLOCKS)
    fused_gen_kernel(const __grid_constant__ FusedGen g, uint32_t n_tiles) {
  constexpr int B = 1 << LB;
  constexpr uint32_t DM = B - 1;
  constexpr int BC = B < 2 ? 2 : B;  // counter row length (even: zeroed as u32 words)
  extern __shared__ __align__(16) uint8_t fg_smem[];
  uint32_t* xs = reinterpret_cast<uint32_t*>(fg_smem);               // [FG_XS] keys, then staged records
  uint64_t* delta = reinterpret_cast<uint64_t*>(xs + FG_XS);         // [B]
  uint32_t* hist = reinterpret_cast<uint32_t*>(delta + B);           // [B] tile digit counts
  uint16_t* sd = reinterpret_cast<uint16_t*>(hist + B);              // [FG_TILE] digit of each staged record
  uint16_t* wcnt = sd + FG_TILE;                                     // [FG_WARPS][BC]
  __shared__ uint32_t ws[32];
  __shared__ uint32_t wacc[FG_WARPS];
  __shared__ unsigned long long wred[FG_WARPS];
  __shared__ uint32_t s_t;
  __shared__ unsigned long long s_tq;     // target index of the tile's first draw (64-bit: per-record payloads)
  __shared__ uint32_t s_tr, s_lim;        // remainder of the tile's first draw, records left
  __shared__ uint32_t s_cp[2];            // k_in >= tile: the (at most two) targets of the tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1;
  uint16_t* mycnt = wcnt + warp * BC;
  if (g.free_sms > 0) {  // CTAs placed on the reserved SMs leave at once (tiles go by ticket)
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid >= 148u - g.free_sms) return;
  }
  for (;;) {
    if (tid == 0) s_t = atomicAdd(g.ticket, 1u);
    for (int d = tid; d < B; d += FG_THREADS) hist[d] = 0;
    __syncthreads();
    const uint32_t t = s_t;
    if (t >= n_tiles) break;
    // 1. draw the thread's 16 consecutive raw positions (two Philox blocks);
    //    padded layout (one word per 32): conflict-free both ways
    const uint64_t p0 = (uint64_t)t * FG_TILE + (uint64_t)tid * FG_IPT;
    const bool full = (uint64_t)(t + 1) * FG_TILE <= g.n_raw;
    const uint32_t lim = full ? FG_IPT : (g.n_raw > p0 ? (g.n_raw - p0 < FG_IPT ? (uint32_t)(g.n_raw - p0) : (uint32_t)FG_IPT) : 0u);
    uint32_t* xw = xs + tid * FG_IPT + (tid * FG_IPT) / 32;
#pragma unroll
    for (int q = 0; q < FG_IPT / 8; ++q) {
      uint64_t w[4];
      philox4x64_10(p0 / 8 + q + 1, g.key, w);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t v = (i & 1) ? (uint32_t)(w[i >> 1] >> 32) : (uint32_t)w[i >> 1];
        uint32_t out;
        const bool ok = g.lm.accept(v, out) && (full || (uint32_t)(8 * q + i) < lim);
        xw[8 * q + i] = ok ? fg_key<KM>(g, out) : FG_NOKEY;
      }
    }
    __syncthreads();
    // 2. raw order, warp-striped: item i of lane l is warp position 32 i + l
    uint32_t k[FG_IPT];
    const uint32_t* xr = xs + warp * (33 * FG_IPT) + lane;
#pragma unroll
    for (int i = 0; i < FG_IPT; ++i) k[i] = xr[33 * i];
    // the tile's digit counts first, published before the (longer) ranking
    // so that successors' look-backs rarely wait on this tile
#pragma unroll
    for (int i = 0; i < FG_IPT; ++i) {
      if (LB == 0) {
        const uint32_t vm = __ballot_sync(0xffffffffu, k[i] != FG_NOKEY);
        if (lane == 0 && vm) atomicAdd(hist, (uint32_t)__popc(vm));
      } else if (k[i] != FG_NOKEY) {
        atomicAdd(hist + (k[i] & DM), 1u);
      }
    }
    for (int j = lane; j < BC / 2; j += 32) reinterpret_cast<uint32_t*>(mycnt)[j] = 0;
    __syncthreads();
    // digits per thread (blocked: thread tid owns digits tid * DPTA ..)
    constexpr int DPTA = (B + FG_THREADS - 1) / FG_THREADS;
    uint32_t c[DPTA];
#pragma unroll
    for (int j = 0; j < DPTA; ++j) {
      const int d = tid * DPTA + j;
      c[j] = d < B ? hist[d] : 0u;
      if (d < B) st_vol(g.status + (size_t)t * B + d, (t == 0 ? ST_P : ST_A) | c[j]);
    }
    uint32_t rank2[FG_IPT / 2];
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < FG_IPT; ++i) {
      const bool valid = k[i] != FG_NOKEY;
      const uint32_t vm = __ballot_sync(0xffffffffu, valid);
      const uint32_t ar = run + __popc(vm & lt);
      run += __popc(vm);
      const uint32_t r = LB == 0 ? (valid ? ar : 0xffffu) : fg_rank<LB>(k[i] & DM, valid, vm, mycnt, lane, lt);
      if (i & 1) rank2[i >> 1] |= r << 16;
      else rank2[i >> 1] = r;
    }
    if (lane == 0) {
      wacc[warp] = run;
      if (LB == 0) mycnt[0] = (uint16_t)run;
    }
    __syncthreads();  // counters complete; xs is free
    // 3. per digit: tile start, per-warp bases
    uint32_t tot, csum = 0;
#pragma unroll
    for (int j = 0; j < DPTA; ++j) csum += c[j];
    uint32_t ts[DPTA];
    ts[0] = block_excl_scan(csum, ws, tot);
#pragma unroll
    for (int j = 1; j < DPTA; ++j) ts[j] = ts[j - 1] + c[j - 1];
#pragma unroll
    for (int j = 0; j < DPTA; ++j) {  // wcnt[w][d] = staging position of warp w's first record of digit d
      const int d = tid * DPTA + j;
      if (d >= B) break;
      uint32_t acc = ts[j];
#pragma unroll
      for (int w = 0; w < FG_WARPS; ++w) {
        const uint32_t x = wcnt[w * BC + d];
        wcnt[w * BC + d] = (uint16_t)acc;
        acc += x;
      }
    }
    // 4. look-back: records of each digit in earlier tiles of the call
    uint64_t excl_sum = 0;
#pragma unroll
    for (int j = 0; j < DPTA; ++j) {
      const int d = tid * DPTA + j;
      if (d >= B) break;
      uint64_t excl = 0;
      if (t > 0) {
        // walk back SMX_FG_LB_WIN descriptors per step (independent loads):
        // a tile usually finds an inclusive prefix ~18 tiles back
        uint32_t e = 0;
        for (int64_t i = (int64_t)t - 1;;) {
          uint32_t w[SMX_FG_LB_WIN];
#pragma unroll
          for (int u = 0; u < SMX_FG_LB_WIN; ++u)
            w[u] = i - u >= 0 ? ld_vol(g.status + (size_t)(i - u) * B + d) : ST_P;
          int used = 0;
          bool done = false;
#pragma unroll
          for (int u = 0; u < SMX_FG_LB_WIN; ++u) {
            if (done || used < u || w[u] == 0) continue;  // stop at a predecessor still drawing
            e += w[u] & ST_VAL;
            used = u + 1;
            done = (w[u] & ST_P) != 0;
          }
#ifdef SMX_FG_LBSTAT
          if (tid == 0) {
            atomicAdd(&g_fg_lbstat[1], 1ull);
            atomicAdd(&g_fg_lbstat[2], (unsigned long long)used);
            if (used == 0) atomicAdd(&g_fg_lbstat[3], 1ull);
          }
#endif
          if (done) break;
          if (used == 0) __nanosleep(SMX_FG_LB_SLEEP);  // predecessor still drawing: leave the issue slots to others
          i -= used;
        }
#ifdef SMX_FG_LBSTAT
        if (tid == 0) atomicAdd(&g_fg_lbstat[0], 1ull);
#endif
        excl = e;
        st_vol(g.status + (size_t)t * B + d, ST_P | (e + c[j]));
      }
      excl_sum += excl;
      const uint64_t filled = g.fill_in[d] + excl;
      if (filled + c[j] > g.rcap[d]) {
        atomicExch(g.overflow, 1);
        delta[d] = ~0ull;
      } else {
        delta[d] = g.rstart[d] + filled - ts[j];
      }
      // clamped: an overflowing region is never read past its capacity
      if (t == n_tiles - 1) g.fill_out[d] = filled + c[j] < g.rcap[d] ? filled + c[j] : g.rcap[d];
    }
    // draw index of the tile's first accepted value = sum of the digit prefixes
    unsigned long long sx = excl_sum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
    if (lane == 0) wred[warp] = sx;
    __syncthreads();
    uint64_t jbase = 0, wbase = 0;
#pragma unroll
    for (int w = 0; w < FG_WARPS; ++w) {
      jbase += wred[w];
      if (w < warp) wbase += wacc[w];
    }
    if (tid == 0) {
      // draw j of the tile = jbase + a: target index tq + (tr + a) / k (32-bit
      // from here on); records past the call's end become sentinels
      const uint64_t tq = jbase / g.kdiv;
      s_tq = tq;
      s_tr = (uint32_t)(jbase - tq * g.kdiv);
      s_lim = jbase >= g.n_out ? 0u : (g.n_out - jbase > 0xffffffffull ? 0xffffffffu : (uint32_t)(g.n_out - jbase));
      if (g.kdiv >= FG_TILE) {
        const uint64_t n_tgt = (g.n_out + g.kdiv - 1) / g.kdiv;
        s_cp[0] = tq < n_tgt ? (__ldg(g.pay + tq) & 0xffffffu) | g.cls_field : 0u;
        s_cp[1] = tq + 1 < n_tgt ? (__ldg(g.pay + tq + 1) & 0xffffffu) | g.cls_field : 0u;
      }
      if (t == n_tiles - 1) *g.total = jbase + tot;
    }
    __syncthreads();
    // 5. records, staged in digit order (accept ranks recomputed: fewer live registers)
    const uint64_t tq = s_tq;
    const uint32_t tr = s_tr, left = s_lim;
    const bool bigk = g.kdiv >= FG_TILE;   // j / k_in takes two values in a tile
    const uint32_t cp0 = s_cp[0], cp1 = s_cp[1], kth = g.kdiv - tr;
    uint32_t aw = (uint32_t)wbase;
#pragma unroll
    for (int i = 0; i < FG_IPT; ++i) {
      const uint32_t vm = __ballot_sync(0xffffffffu, k[i] != FG_NOKEY);
      const uint32_t a = aw + __popc(vm & lt);
      aw += __popc(vm);
      const uint32_t r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
      if (r == 0xffffu) continue;
      const uint32_t d = LB ? (k[i] & DM) : 0u;
      const uint32_t cp = bigk ? (a >= kth ? cp1 : cp0)
                               : (__ldg(g.pay + tq + g.kd.div(tr + a)) & 0xffffffu) | g.cls_field;
      const uint32_t rec = a < left ? (((k[i] >> LB) << g.pbits) | cp) : FG_SENTINEL;
      const uint32_t pos = wcnt[warp * BC + d] + r;
      xs[pos] = rec;
      sd[pos] = (uint16_t)d;
    }
    __syncthreads();
    // 6. coalesced runs per digit
    if (WIDE) {
      for (uint32_t q = tid; q < tot; q += FG_THREADS) {
        const uint64_t base = delta[sd[q]];
        if (base != ~0ull) g.region[base + q] = xs[q];
      }
    } else {
      const uint32_t* d32 = reinterpret_cast<const uint32_t*>(delta);  // low words (little endian)
      for (uint32_t q = tid; q < tot; q += FG_THREADS) {
        const uint32_t base = d32[2 * sd[q]];
        if (base != 0xffffffffu) g.region[base + q] = xs[q];
      }
    }
    __syncthreads();
  }
}

template <int LB>
size_t fg_smem() {
  constexpr int B = 1 << LB;
  constexpr int BC = B < 2 ? 2 : B;
  return (size_t)FG_XS * 4 + (size_t)B * 12 + (size_t)FG_TILE * 2 + (size_t)FG_WARPS * BC * 2;
}

template <int KM, int LB, bool WIDE>
int fg_launch(const FusedGen& g, uint32_t n_tiles, cudaStream_t st) {
  const size_t smem = fg_smem<LB>();
  static unsigned long long configured = 0;   // one bit per device
  const unsigned long long dbit = smx_device_bit();
  if (!(configured & dbit)) {
    SMX_CUDA_CHECK(cudaFuncSetAttribute(fused_gen_kernel<KM, LB, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    configured |= dbit;
  }
  // persistent CTAs on 140 of the 148 SMs: the replays and small kernels of
  // the calls that follow (their host code waits on them) run beside pass A
  // instead of queueing behind it.  The grid fills every SM (the block
  // scheduler spreads CTAs round-robin, so a smaller grid would leave half
  // SMs, too small for a draw CTA); the CTAs that land on SMs 140..147 exit
  // at once, leaving those SMs empty
  const uint32_t grid = std::min<uint32_t>(n_tiles + g.free_sms * SMX_FG_MIN_BLOCKS, 148u * SMX_FG_MIN_BLOCKS);
  smx_count_launch();
  fused_gen_kernel<KM, LB, WIDE><<<grid, FG_THREADS, smem, st>>>(g, n_tiles);
  SMX_LAUNCH_CHECK();
  if (g.free_sms) smx_long_kernel_mark(st);
  return 0;
}

template <int KM, int LB>
int fg_wide(bool wide, const FusedGen& g, uint32_t n_tiles, cudaStream_t st) {
  return wide ? fg_launch<KM, LB, true>(g, n_tiles, st) : fg_launch<KM, LB, false>(g, n_tiles, st);
}

template <int KM>
int fg_dispatch(int lo_bits, bool wide, const FusedGen& g, uint32_t n_tiles, cudaStream_t st) {
  switch (lo_bits) {
    case 0: return fg_wide<KM, 0>(wide, g, n_tiles, st);
    case 1: return fg_wide<KM, 1>(wide, g, n_tiles, st);
    case 2: return fg_wide<KM, 2>(wide, g, n_tiles, st);
    case 3: return fg_wide<KM, 3>(wide, g, n_tiles, st);
    case 4: return fg_wide<KM, 4>(wide, g, n_tiles, st);
    case 5: return fg_wide<KM, 5>(wide, g, n_tiles, st);
    case 6: return fg_wide<KM, 6>(wide, g, n_tiles, st);
    case 7: return fg_wide<KM, 7>(wide, g, n_tiles, st);
    case 8: return fg_wide<KM, 8>(wide, g, n_tiles, st);
    case 9: return fg_wide<KM, 9>(wide, g, n_tiles, st);
    default: break;
  }
  smx_set_error("smx_fused_gen: low digit of %d bits (0..9 supported)", lo_bits);
  return -1;
}

// ------------------------------------------------------------------ pass B
#ifndef SMX_FB_THREADS
#define SMX_FB_THREADS 256   // with 30 records per thread and 3 CTAs per SM (measured best: 5.9 vs 6.6 ms on C3)
#endif
constexpr int FB_THREADS = SMX_FB_THREADS;
constexpr int FB_WARPS = FB_THREADS / 32;
#ifndef SMX_FB_IPT
#define SMX_FB_IPT 30
#endif
constexpr int FB_IPT = SMX_FB_IPT;
constexpr int FB_TILE = FB_THREADS * FB_IPT;   // 7680 records by default
constexpr int FB_TC = 256;                     // tiles per scan chunk (chunks never straddle regions)
constexpr int FB_MAX_CALLS = 512;              // calls (regions per low digit) one pass B takes

struct FusedSort {
  const uint64_t* rptr;       // [R] region base pointers, regions in (low digit, call) order
  const uint64_t* fill;       // [R] records per region
  const uint32_t* tile_first; // [R + 1] first tile of each region
  const uint32_t* chunk_first;// [R + 1] first scan chunk of each region
  uint32_t n_regions;
  uint32_t per_digit;         // regions per low digit (one per call)
  int pbits;                  // record = hi << pbits | class index << row bits | row
  int lo_bits;                // key = hi << lo_bits | region
  const uint32_t* cls_map;    // [256] class index -> global class id << 24
  uint32_t* counts;           // [n_keys] records per key
  uint64_t n_keys;
  uint32_t* out;              // final payload (sorted by key)
  int* err;
  uint8_t row_bits[FB_MAX_CALLS];  // per call: payload = class index << row_bits[call] | row
};

__device__ __forceinline__ uint32_t upper_region(const uint32_t* first, uint32_t n, uint32_t x) {
  // largest r with first[r] <= x  (first ascending, first[0] = 0)
  uint32_t lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(first + mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}

struct FbTile {
  const uint32_t* src;  // first record
  uint32_t region;
  uint32_t n;           // records in the tile
};

__device__ __forceinline__ FbTile fb_tile(const FusedSort& s, uint32_t T) {
  FbTile x;
  x.region = upper_region(s.tile_first, s.n_regions, T);
  const uint64_t local = (uint64_t)(T - __ldg(s.tile_first + x.region)) * FB_TILE;
  x.src = reinterpret_cast<const uint32_t*>(__ldg(s.rptr + x.region)) + local;
  const uint64_t f = __ldg(s.fill + x.region);
  x.n = f > local ? (f - local < (uint64_t)FB_TILE ? (uint32_t)(f - local) : (uint32_t)FB_TILE) : 0u;
  return x;
}

// Per-tile histogram of the high digit (sentinels skipped); one warp per
// tile, as many warps per CTA as their u32 histograms fit in 128 KB.
template <int BITS>
__host__ __device__ constexpr int fb_hist_warps() { return (128 * 1024) / (4 << BITS) < 32 ? (128 * 1024) / (4 << BITS) : 32; }

template <int BITS>
__global__ void __launch_bounds__(1024) fb_hist_kernel(const __grid_constant__ FusedSort s, uint16_t* tcnt,
                                                       uint32_t n_tiles) {
  constexpr int BINS = 1 << BITS;
  constexpr int HW = fb_hist_warps<BITS>();
  extern __shared__ uint32_t fbh[];  // [HW][BINS]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* wh = fbh + warp * BINS;
  for (uint32_t T = blockIdx.x * HW + warp; T < n_tiles; T += gridDim.x * HW) {
    for (int j = lane; j < BINS; j += 32) wh[j] = 0;
    __syncwarp();
    const FbTile x = fb_tile(s, T);
    const uint32_t* src = x.src;
    const uint32_t nq = x.n / 4;
    for (uint32_t i = lane; i < nq; i += 32) {
      const uint4 q = __ldcs(reinterpret_cast<const uint4*>(src) + i);
      const uint32_t r[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r[u] != FG_SENTINEL) atomicAdd(&wh[r[u] >> s.pbits], 1u);
    }
    for (uint32_t i = nq * 4 + lane; i < x.n; i += 32) {
      const uint32_t r = src[i];
      if (r != FG_SENTINEL) atomicAdd(&wh[r >> s.pbits], 1u);
    }
    __syncwarp();
    uint32_t* o = reinterpret_cast<uint32_t*>(tcnt + (size_t)T * BINS);
    for (int j = lane; j < BINS / 2; j += 32) o[j] = wh[2 * j] | (wh[2 * j + 1] << 16);
    __syncwarp();
  }
}

// csum[chunk][d] = sum of the chunk's tile counts
template <int BITS>
__global__ void __launch_bounds__(256) fb_chunk_sum_kernel(const __grid_constant__ FusedSort s, const uint16_t* tcnt,
                                                           uint32_t* csum) {
  constexpr int BINS = 1 << BITS;
  const uint32_t C = blockIdx.x;
  const uint32_t r = upper_region(s.chunk_first, s.n_regions, C);
  const uint32_t t0 = s.tile_first[r] + (C - s.chunk_first[r]) * FB_TC;
  const uint32_t t1 = min(s.tile_first[r + 1], t0 + FB_TC);
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t acc = 0;
#pragma unroll 8
    for (uint32_t t = t0; t < t1; ++t) acc += tcnt[(size_t)t * BINS + d];
    csum[(size_t)C * BINS + d] = acc;
  }
}

// rsum[r][d] = records of digit d in region r (sum over the region's
// chunks); per-key counts (key = d << lo_bits | r) are these sums.
template <int BITS>
__global__ void __launch_bounds__(256) fb_region_sum_kernel(const __grid_constant__ FusedSort s, const uint32_t* csum,
                                                            uint32_t* rsum) {
  constexpr int BINS = 1 << BITS;
  const uint32_t r = blockIdx.x;
  const uint32_t c0 = s.chunk_first[r], c1 = s.chunk_first[r + 1];
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t acc = 0;
    for (uint32_t C = c0; C < c1; ++C) acc += csum[(size_t)C * BINS + d];
    rsum[(size_t)r * BINS + d] = acc;
    const uint64_t key = ((uint64_t)d << s.lo_bits) | (r / s.per_digit);
    if (acc) {
      if (key < s.n_keys) atomicAdd(s.counts + key, acc);  // one region per call of the digit
      else atomicExch(s.err, 6);
    }
  }
}

// The per-digit exclusive scan over the regions runs in three steps over
// groups of FB_RG consecutive regions: group sums, one CTA scanning the
// groups (and the 64-bit digit bases), then each group's regions.
constexpr uint32_t FB_RG = 64;

template <int BITS>
__global__ void __launch_bounds__(256) fb_group_sum_kernel(const __grid_constant__ FusedSort s, const uint32_t* rsum,
                                                           uint32_t* gsum) {
  constexpr int BINS = 1 << BITS;
  const uint32_t g = blockIdx.x;
  const uint32_t r0 = g * FB_RG, r1 = min(s.n_regions, r0 + FB_RG);
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint64_t acc = 0;
    for (uint32_t r = r0; r < r1; ++r) acc += rsum[(size_t)r * BINS + d];
    if (acc > 0xffffffffull) atomicExch(s.err, 7);  // within-digit offsets are 32-bit
    gsum[(size_t)g * BINS + d] = (uint32_t)acc;
  }
}

template <int BITS>
__global__ void __launch_bounds__(256) fb_group_apply_kernel(const __grid_constant__ FusedSort s, uint32_t* rsum,
                                                             const uint32_t* gbase) {
  constexpr int BINS = 1 << BITS;
  const uint32_t g = blockIdx.x;
  const uint32_t r0 = g * FB_RG, r1 = min(s.n_regions, r0 + FB_RG);
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t run = gbase[(size_t)g * BINS + d];
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t x = rsum[(size_t)r * BINS + d];
      rsum[(size_t)r * BINS + d] = run;
      run += x;
    }
  }
}

// One CTA: per digit, exclusive scan over the region groups (in place: gsum
// -> group base within the digit) and the 64-bit digit bases.
template <int BITS>
__global__ void __launch_bounds__(1024) fb_region_scan_kernel(const __grid_constant__ FusedSort s, uint32_t* gsum,
                                                              uint32_t n_groups, uint64_t* dbase) {
  constexpr int BINS = 1 << BITS;
  constexpr int DPT = (BINS + 1023) / 1024;
  __shared__ unsigned long long ws[32];
  uint64_t tot[DPT];
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = j * 1024 + threadIdx.x;
    uint64_t run = 0;
    if (d < BINS) {
#pragma unroll 8
      for (uint32_t g = 0; g < n_groups; ++g) {
        const uint32_t x = gsum[(size_t)g * BINS + d];
        gsum[(size_t)g * BINS + d] = (uint32_t)run;
        run += x;
      }
      if (run > 0xffffffffull) atomicExch(s.err, 7);  // within-digit offsets are 32-bit
    }
    tot[j] = run;
  }
  uint64_t mine = 0;
#pragma unroll
  for (int j = 0; j < DPT; ++j) mine += tot[j];
  // digit order is j * 1024 + tid: scan thread-major within each j slice
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t carry = 0;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    uint64_t inc = tot[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint64_t v = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      ws[lane] = v;
    }
    __syncthreads();
    const int d = j * 1024 + threadIdx.x;
    if (d < BINS) dbase[d] = carry + (warp ? ws[warp - 1] : 0) + inc - tot[j];
    carry += ws[31];
    __syncthreads();
  }
  (void)mine;
}

// csum[C][d] = position of chunk C's first record of digit d within the digit
template <int BITS>
__global__ void __launch_bounds__(256) fb_chunk_base_kernel(const __grid_constant__ FusedSort s, uint32_t* csum,
                                                            const uint32_t* rbase) {
  constexpr int BINS = 1 << BITS;
  const uint32_t r = blockIdx.x;
  const uint32_t c0 = s.chunk_first[r], c1 = s.chunk_first[r + 1];
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t run = rbase[(size_t)r * BINS + d];
    for (uint32_t C = c0; C < c1; ++C) {
      const uint32_t x = csum[(size_t)C * BINS + d];
      csum[(size_t)C * BINS + d] = run;
      run += x;
    }
  }
}

// off[tile][d] = within-digit position of the tile's first record of digit d
template <int BITS>
__global__ void __launch_bounds__(256) fb_tile_offsets_kernel(const __grid_constant__ FusedSort s, const uint16_t* tcnt,
                                                              const uint32_t* csum, uint32_t* off) {
  constexpr int BINS = 1 << BITS;
  const uint32_t C = blockIdx.x;
  const uint32_t r = upper_region(s.chunk_first, s.n_regions, C);
  const uint32_t t0 = s.tile_first[r] + (C - s.chunk_first[r]) * FB_TC;
  const uint32_t t1 = min(s.tile_first[r + 1], t0 + FB_TC);
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t run = csum[(size_t)C * BINS + d];
    for (uint32_t t = t0; t < t1; ++t) {
      off[(size_t)t * BINS + d] = run;
      run += tcnt[(size_t)t * BINS + d];
    }
  }
}

// Stable scatter by the high digit; tiles in global (region, tile) order from
// a ticket so the tiles in flight write neighbouring parts of every digit's
// output (partial sectors complete in L2).  Writes the final payload.
#ifndef SMX_FB_CTAS
#define SMX_FB_CTAS (FB_THREADS >= 512 ? 2 : 3)
#endif
template <int BITS, bool WIDE>
__global__ void __launch_bounds__(FB_THREADS, BITS >= 12 ? 1 : SMX_FB_CTAS) fb_scatter_kernel(const __grid_constant__ FusedSort s,
                                                                   const uint32_t* off, const uint64_t* dbase,
                                                                   uint32_t n_tiles, uint32_t* tile_ctr) {
  constexpr int BINS = 1 << BITS;
  constexpr int DPT = BINS >= FB_THREADS ? BINS / FB_THREADS : 1;   // digits per thread
  constexpr uint32_t mask = BINS - 1;
  extern __shared__ __align__(128) uint8_t fbs[];
  uint32_t* irec = reinterpret_cast<uint32_t*>(fbs);              // [FB_TILE] TMA target, then staged payloads
  uint16_t* sdig = reinterpret_cast<uint16_t*>(irec + FB_TILE);   // [FB_TILE] staged digits
  uint32_t* ioff = reinterpret_cast<uint32_t*>(sdig + FB_TILE);   // [BINS] TMA target
  uint64_t* delta = reinterpret_cast<uint64_t*>(ioff + BINS);     // [BINS]
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(delta + BINS);     // [FB_WARPS][BINS]
  __shared__ uint32_t ws[32];
  __shared__ uint32_t ticket[2];
  __shared__ FbTile tinfo[2];
  __shared__ uint32_t cmap[256];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1;
  for (int i = tid; i < 256; i += FB_THREADS) cmap[i] = s.cls_map[i];
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // thread 0 takes the tickets: the tile's (region, slots) for everyone, then
  // its TMA -- the offset row and, for full tiles, the records
  auto take = [&](int sl) {
    const uint32_t T = atomicAdd(tile_ctr, 1u);
    ticket[sl] = T;
    if (T < n_tiles) tinfo[sl] = fb_tile(s, T);
  };
  auto issue = [&](uint32_t T, const FbTile& x) {
    const bool full = x.n == FB_TILE;
    mbar_expect_tx(&bar, BINS * 4 + (full ? FB_TILE * 4 : 0));
    bulk_g2s(ioff, off + (size_t)T * BINS, BINS * 4, &bar);
    if (full) bulk_g2s(irec, x.src, FB_TILE * 4, &bar);
  };
  if (tid == 0) {
    take(0);
    if (ticket[0] < n_tiles) issue(ticket[0], tinfo[0]);
  }
  __syncthreads();
  uint16_t* mycnt = wcnt + warp * BINS;
  const uint32_t wofs = warp * (32 * FB_IPT) + lane;
  uint32_t phase = 0;
  int slot = 0;
  for (uint32_t T = ticket[0]; T < n_tiles; T = ticket[slot ^= 1]) {
    const FbTile x = tinfo[slot];
    const bool full = x.n == FB_TILE;
    // the tile's call (regions are in (low digit, call) order) fixes its row / class split
    const int rbits = s.row_bits[x.region % s.per_digit];
    const uint32_t rmask = (1u << rbits) - 1;
    const uint32_t cmask = (1u << (s.pbits - rbits < 8 ? s.pbits - rbits : 8)) - 1;
    mbar_wait(&bar, phase);
    phase ^= 1;
    uint32_t rec[FB_IPT];
#pragma unroll
    for (int i = 0; i < FB_IPT; ++i) {
      const uint32_t q = wofs + i * 32;
      rec[i] = full ? irec[q] : (q < x.n ? x.src[q] : FG_SENTINEL);
    }
    {
      uint32_t* w32 = reinterpret_cast<uint32_t*>(mycnt);
#pragma unroll
      for (int j = lane; j < BINS / 2; j += 32) w32[j] = 0;
      __syncwarp();
    }
    uint32_t rank2[(FB_IPT + 1) / 2];
#pragma unroll
    for (int i = 0; i < FB_IPT; ++i) {
      const bool valid = rec[i] != FG_SENTINEL;
      const uint32_t vm = __ballot_sync(0xffffffffu, valid);
      const uint32_t r = fg_rank<BITS>((rec[i] >> s.pbits) & mask, valid, vm, mycnt, lane, lt);
      if (i & 1) rank2[i >> 1] |= r << 16; else rank2[i >> 1] = r;
    }
    __syncthreads();  // 1: counters complete, records in registers
    if (tid == 0) take(slot ^ 1);
    uint32_t tot[DPT];
    uint32_t mysum = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < FB_WARPS; ++w) t += d < BINS ? wcnt[w * BINS + d] : 0u;
      tot[j] = t;
      mysum += t;
    }
    uint32_t tsum;
    uint32_t run = block_excl_scan(mysum, ws, tsum);
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      if (d >= BINS) break;
      uint32_t t = run;
#pragma unroll
      for (int w = 0; w < FB_WARPS; ++w) {
        const uint32_t c = wcnt[w * BINS + d];
        wcnt[w * BINS + d] = (uint16_t)t;
        t += c;
      }
      delta[d] = dbase[d] + ioff[d] - run;
      run += tot[j];
    }
    __syncthreads();  // 2: offsets ready; offset row and record buffer free
    const uint32_t nxt = ticket[slot ^ 1];
    // stage the final payloads in digit order (the record buffer is reused)
#pragma unroll
    for (int i = 0; i < FB_IPT; ++i) {
      const uint32_t r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
      if (r != 0xffffu) {
        const uint32_t d = (rec[i] >> s.pbits) & mask;
        const uint32_t pos = mycnt[d] + r;
        irec[pos] = (rec[i] & rmask) | cmap[(rec[i] >> rbits) & cmask];
        sdig[pos] = (uint16_t)d;
      }
    }
    __syncthreads();  // 3: staged
    if (WIDE) {
      for (uint32_t q = tid; q < tsum; q += FB_THREADS) s.out[delta[sdig[q]] + q] = irec[q];
    } else {
      const uint32_t* d32 = reinterpret_cast<const uint32_t*>(delta);
      for (uint32_t q = tid; q < tsum; q += FB_THREADS) s.out[d32[2 * sdig[q]] + q] = irec[q];
    }
    __syncthreads();  // 4: staging read: buffers may be refilled
    if (tid == 0 && nxt < n_tiles) {
      fence_proxy_async();
      issue(nxt, tinfo[slot ^ 1]);
    }
  }
}

template <int BITS>
int fb_run(const FusedSort& s, uint32_t n_tiles, uint32_t n_chunks, bool wide, cudaStream_t st) {
  constexpr int BINS = 1 << BITS;
  uint16_t* tcnt = nullptr;
  uint32_t *off = nullptr, *csum = nullptr, *ctr = nullptr, *rsum = nullptr, *gsum = nullptr;
  const uint32_t n_groups = (s.n_regions + FB_RG - 1) / FB_RG;
  uint64_t* dbase = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&tcnt, sizeof(uint16_t) * (size_t)n_tiles * BINS, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&off, sizeof(uint32_t) * (size_t)n_tiles * BINS, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&csum, sizeof(uint32_t) * (size_t)std::max<uint32_t>(n_chunks, 1) * BINS, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&dbase, sizeof(uint64_t) * BINS, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&rsum, sizeof(uint32_t) * (size_t)s.n_regions * BINS, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&ctr, sizeof(uint32_t), st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&gsum, sizeof(uint32_t) * (size_t)n_groups * BINS, st));
  SMX_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
  constexpr int HW = fb_hist_warps<BITS>();
  const size_t h_smem = (size_t)HW * BINS * 4;
  const size_t s_smem = (size_t)FB_TILE * 6 + (size_t)BINS * 12 + (size_t)FB_WARPS * BINS * 2;
  static unsigned long long configured = 0;   // one bit per device
  const unsigned long long dbit = smx_device_bit();
  if (!(configured & dbit)) {
    SMX_CUDA_CHECK(cudaFuncSetAttribute(fb_hist_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h_smem));
    SMX_CUDA_CHECK(cudaFuncSetAttribute(fb_scatter_kernel<BITS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)s_smem));
    SMX_CUDA_CHECK(cudaFuncSetAttribute(fb_scatter_kernel<BITS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)s_smem));
    configured |= dbit;
  }
  const uint32_t hgrid = std::max<uint32_t>(1, std::min<uint32_t>((n_tiles + HW - 1) / HW, (148 - SMX_FG_FREE_SMS) * 2));
  smx_count_launch(); fb_hist_kernel<BITS><<<hgrid, 32 * HW, h_smem, st>>>(s, tcnt, n_tiles);
  if (n_chunks) {
    smx_count_launch(); fb_chunk_sum_kernel<BITS><<<n_chunks, 256, 0, st>>>(s, tcnt, csum);
  }
  smx_count_launch(); fb_region_sum_kernel<BITS><<<s.n_regions, 256, 0, st>>>(s, csum, rsum);
  smx_count_launch(); fb_group_sum_kernel<BITS><<<n_groups, 256, 0, st>>>(s, rsum, gsum);
  smx_count_launch(); fb_region_scan_kernel<BITS><<<1, 1024, 0, st>>>(s, gsum, n_groups, dbase);
  smx_count_launch(); fb_group_apply_kernel<BITS><<<n_groups, 256, 0, st>>>(s, rsum, gsum);
  smx_count_launch(); fb_chunk_base_kernel<BITS><<<s.n_regions, 256, 0, st>>>(s, csum, rsum);
  if (n_chunks) {
    smx_count_launch(); fb_tile_offsets_kernel<BITS><<<n_chunks, 256, 0, st>>>(s, tcnt, csum, off);
  }
  // like pass A, the scatter leaves SMX_FG_FREE_SMS SMs to the preparation
  // side stream (map compaction, routes), whose host code waits on it
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(n_tiles, (148u - SMX_FG_FREE_SMS) * SMX_FB_CTAS));
  smx_count_launch();
  if (wide) fb_scatter_kernel<BITS, true><<<grid, FB_THREADS, s_smem, st>>>(s, off, dbase, n_tiles, ctr);
  else fb_scatter_kernel<BITS, false><<<grid, FB_THREADS, s_smem, st>>>(s, off, dbase, n_tiles, ctr);
  SMX_LAUNCH_CHECK();
  cudaFreeAsync(tcnt, st);
  cudaFreeAsync(off, st);
  cudaFreeAsync(csum, st);
  cudaFreeAsync(dbase, st);
  cudaFreeAsync(rsum, st);
  cudaFreeAsync(ctr, st);
  cudaFreeAsync(gsum, st);
  return 0;
}

}  // namespace

// Pass A for one deferred fixed-indegree call (see the file comment): draws
// integers(0, ex, size=n_out) from the start of stream (k0, k1); record j
// has source key = pieces(value) (key_mode 3: key_tab is a HOST array
// {n, start[n], delta[n]}) or key_tab[value] (key_mode 1: device table) and
// target index j / kdiv.  rstart / rcap / fill_in / fill_out (device, 2^lo_bits
// entries) describe the digit regions; *total_out receives the accepted draws
// in the raw window (< n_out: the window was short, rebuild), *overflow is
// set when a region is too small.
extern "C" int smx_fused_gen(uint64_t k0, uint64_t k1, uint64_t ex, uint64_t n_out, int key_mode,
                             const uint32_t* key_tab, uint32_t kdiv, const uint32_t* pay_tab, uint32_t cls_field,
                             int lo_bits, int pbits,
                             uint32_t* region, uint64_t n_slots, const uint64_t* rstart, const uint64_t* rcap,
                             const uint64_t* fill_in, uint64_t* fill_out, uint64_t* total_out, int* overflow,
                             void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_out == 0) {
    SMX_CUDA_CHECK(cudaMemcpyAsync(fill_out, fill_in, sizeof(uint64_t) << lo_bits, cudaMemcpyDeviceToDevice, st));
    SMX_CUDA_CHECK(cudaMemsetAsync(total_out, 0, sizeof(uint64_t), st));
    return 0;
  }
  if (ex < 2 || ex > (1ULL << 32) || kdiv == 0 || lo_bits < 0 || lo_bits > 9 || (key_mode != 1 && key_mode != 3)) {
    smx_set_error("smx_fused_gen: unsupported call (ex %llu, k %u, lo_bits %d, key mode %d)",
                  (unsigned long long)ex, kdiv, lo_bits, key_mode);
    return -1;
  }
  FusedGen g{};
  g.free_sms = (uint32_t)g_fg_free_sms;
  g.key = Key{k0, k1};
  g.lm.ex = (uint32_t)(ex & 0xffffffffULL);
  g.lm.threshold = ex == (1ULL << 32) ? 0u : (uint32_t)(((1ULL << 32) - ex) % ex);
  const double prej = (double)g.lm.threshold / 4294967296.0;
  g.n_raw = n_out + (uint64_t)std::ceil(n_out * prej * 1.25 + 12.0 * std::sqrt(n_out * prej + 1.0) + 64.0);
  g.n_out = n_out;
  if (key_mode == 3) {
    const uint32_t np = key_tab ? key_tab[0] : 0;
    if (np < 1 || np > FG_MAXP) {
      smx_set_error("smx_fused_gen: %u key pieces (1..%d supported)", np, FG_MAXP);
      return -1;
    }
    g.np = np;
    for (uint32_t i = 0; i < FG_MAXP; ++i) {
      g.pstart[i] = i < np ? key_tab[1 + i] : 0xffffffffu;
      g.pdelta[i] = i < np ? key_tab[1 + np + i] : 0u;
    }
  } else {
    g.key_tab = key_tab;
  }
  g.kdiv = kdiv;
  g.kd = FastDiv::make(kdiv);
  g.pay = pay_tab;
  g.cls_field = cls_field;
  if ((uint64_t)kdiv + 2 * FG_TILE >= 0xffffffffull) {
    smx_set_error("smx_fused_gen: k_in %u too large", kdiv);
    return -1;
  }
  g.pbits = pbits;
  g.region = region;
  g.rstart = rstart;
  g.rcap = rcap;
  g.fill_in = fill_in;
  g.fill_out = fill_out;
  g.total = total_out;
  g.overflow = overflow;
  const uint64_t n_tiles = (g.n_raw + FG_TILE - 1) / FG_TILE;
  if (n_tiles >= 0xffffffffull) {
    smx_set_error("smx_fused_gen: %llu raw positions exceed the tile range", (unsigned long long)g.n_raw);
    return -1;
  }
  const size_t B = (size_t)1 << lo_bits;
  uint32_t* ws = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&ws, sizeof(uint32_t) * (n_tiles * B + 1), st));
  SMX_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(uint32_t) * (n_tiles * B + 1), st));
  g.status = ws;
  g.ticket = ws + n_tiles * B;
  const bool wide = n_slots >= 0x7fffffffull;  // 32-bit staging offsets below 2^31 slots
  // key modes by piece count: 4 (one), 5 (two), 6 (three or four), 3 (up to FG_MAXP)
  const int rc = key_mode == 1                  ? fg_dispatch<1>(lo_bits, wide, g, (uint32_t)n_tiles, st)
                 : g.np == 1                    ? fg_dispatch<4>(lo_bits, wide, g, (uint32_t)n_tiles, st)
                 : g.np == 2                    ? fg_dispatch<5>(lo_bits, wide, g, (uint32_t)n_tiles, st)
                 : g.np <= 4 && ex < (1ull << 32) ? fg_dispatch<6>(lo_bits, wide, g, (uint32_t)n_tiles, st)
                                                : fg_dispatch<3>(lo_bits, wide, g, (uint32_t)n_tiles, st);
  cudaFreeAsync(ws, st);
  return rc;
}

#ifdef SMX_FG_LBSTAT
extern "C" int smx_fg_lbstat(unsigned long long* out, int reset) {
  SMX_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_fg_lbstat, sizeof(unsigned long long) * 4));
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    SMX_CUDA_CHECK(cudaMemcpyToSymbol(g_fg_lbstat, z, sizeof(z)));
  }
  return 0;
}
#endif

// CTA slots (two per free SM) a kernel launched beside pass A can count on.
int smx_pass_a_free_slots() { return g_fg_free_sms * SMX_FG_MIN_BLOCKS; }

// SMs pass A leaves free for concurrent work (0..16; default SMX_FG_FREE_SMS).
// A single-rank construction has nothing to run beside pass A: 0.
extern "C" int smx_set_pass_a_free_sms(int n) {
  if (n < 0 || n > 16) {
    smx_set_error("smx_set_pass_a_free_sms: %d outside 0..16", n);
    return -1;
  }
  g_fg_free_sms = n;
  return 0;
}

// Pass B: stable sort of the digit regions by the high digit.  Region
// r = digit * per_digit + call holds fill[r] records at rptr[r] (device
// arrays; every call wrote its own regions in pass A); rcap_host (host, the
// regions' capacities) fixes the tile layout.  Writes out[] (payloads sorted
// by key = hi << lo_bits | digit) and counts[key] (zeroed first).  err
// receives 6 for a key >= n_keys, 7 when a digit holds >= 2^32 records.
extern "C" int smx_fused_sort(const uint64_t* rptr, const uint64_t* fill, const uint64_t* rcap_host, int per_digit,
                              int lo_bits, int hi_bits, int pbits, const uint8_t* row_bits_host,
                              const uint32_t* cls_map, uint32_t* counts, uint64_t n_keys, uint64_t n_records,
                              uint32_t* out, int* err, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  SMX_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * n_keys, st));
  if (hi_bits < 8 || hi_bits > 12) {
    smx_set_error("smx_fused_sort: high digit of %d bits (8..12 supported)", hi_bits);
    return -1;
  }
  if (per_digit < 1) {
    smx_set_error("smx_fused_sort: no regions");
    return -1;
  }
  const uint32_t R = (uint32_t)per_digit << lo_bits;
  std::vector<uint32_t> firsts(2 * (R + 1));
  uint32_t* tile_first = firsts.data();
  uint32_t* chunk_first = firsts.data() + R + 1;
  uint64_t nt = 0, nc = 0;
  for (uint32_t r = 0; r < R; ++r) {
    tile_first[r] = (uint32_t)nt;
    chunk_first[r] = (uint32_t)nc;
    const uint64_t t = (rcap_host[r] + FB_TILE - 1) / FB_TILE;
    nt += t;
    nc += (t + FB_TC - 1) / FB_TC;
  }
  tile_first[R] = (uint32_t)nt;
  chunk_first[R] = (uint32_t)nc;
  if (nt >= 0xffffffffull) {
    smx_set_error("smx_fused_sort: too many tiles");
    return -1;
  }
  uint32_t* dfirst = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&dfirst, sizeof(uint32_t) * firsts.size(), st));
  if (smx_h2d_async(dfirst, firsts.data(), sizeof(uint32_t) * firsts.size(), st)) return -3;
  FusedSort s{};
  s.rptr = rptr;
  s.fill = fill;
  s.tile_first = dfirst;
  s.chunk_first = dfirst + R + 1;
  s.n_regions = R;
  s.per_digit = (uint32_t)per_digit;
  s.pbits = pbits;
  s.lo_bits = lo_bits;
  s.cls_map = cls_map;
  if (per_digit > FB_MAX_CALLS) {
    smx_set_error("smx_fused_sort: more than %d calls", FB_MAX_CALLS);
    return -1;
  }
  for (int c = 0; c < per_digit; ++c) {
    if (row_bits_host[c] < 1 || row_bits_host[c] > pbits) {
      smx_set_error("smx_fused_sort: call %d: %d row bits of %d payload bits", c, (int)row_bits_host[c], pbits);
      return -1;
    }
    s.row_bits[c] = row_bits_host[c];
  }
  const bool wide = n_records >= 0xffffffffull;
  s.counts = counts;
  s.n_keys = n_keys;
  s.out = out;
  s.err = err;
  int rc = 0;
  switch (hi_bits) {
    case 8: rc = fb_run<8>(s, (uint32_t)nt, (uint32_t)nc, wide, st); break;
    case 9: rc = fb_run<9>(s, (uint32_t)nt, (uint32_t)nc, wide, st); break;
    case 10: rc = fb_run<10>(s, (uint32_t)nt, (uint32_t)nc, wide, st); break;
    case 11: rc = fb_run<11>(s, (uint32_t)nt, (uint32_t)nc, wide, st); break;
    default: rc = fb_run<12>(s, (uint32_t)nt, (uint32_t)nc, wide, st); break;   // 1 CTA/SM (221 KB SMEM)
  }
  cudaFreeAsync(dfirst, st);
  return rc;
}
