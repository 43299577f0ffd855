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

constexpr int DS_THREADS = 256;
constexpr int DS_WARPS = DS_THREADS / 32;
constexpr int DS_IPT = 15;                        // items per thread per tile
constexpr int DS_TILE = DS_THREADS * DS_IPT;      // 3840 records (15 KB of keys)
constexpr int RS_MAX_BITS = 11;
constexpr int US_THREADS = 1024;
constexpr int CNT_BINS = 12288;                   // last-pass key-count bins in SMEM (48 KB)

__host__ __device__ constexpr int ds_ctas_per_sm(int bits) { return bits <= 9 ? 3 : 2; }

struct SortPass {
  const uint32_t* keys_in;  // SoA input keys (first pass)
  const uint32_t* vals_in;  // null: value = record index (first pass only)
  const uint2* recs_in;     // later passes: (key, value) records
  uint2* recs_out;          // all but the last pass: (key, value) records
  uint32_t* vals_out;       // last pass: values only
  uint64_t n;
  uint64_t seg;             // records per CTA (multiple of DS_TILE)
  int shift;
  int first;
  int last;
  const uint32_t* lut;      // temporary-key LUT (first pass)
  uint32_t* counts;         // per-key counts (filled by the last pass's upsweep)
  uint64_t n_keys;
  const uint32_t* hist_scan;  // [BINS * G] exclusive offsets
  uint32_t* tmp_flag;         // first pass: set by tile_hist when a temporary key occurs
};

__device__ __forceinline__ uint32_t resolve(uint32_t k, const uint32_t* lut) {
  return (k & SMX_TMP_KEY) ? lut[k & ~SMX_TMP_KEY] : k;
}

__device__ __forceinline__ uint32_t key_at(const SortPass& p, uint64_t i) {
  return p.recs_in ? p.recs_in[i].x : p.keys_in[i];
}

__device__ __forceinline__ void count_key(const SortPass& p, uint32_t key, uint32_t c) {
  if (key < p.n_keys) atomicAdd(&p.counts[key], c);  // out-of-range keys show up in the total check
}

// Per-tile digit histograms tcnt[tile][BINS] (u16), one warp per tile with a
// warp-private SMEM histogram; a CTA covers a contiguous run of tiles.  The
// last pass also produces the per-key record counts (-> first_index): its
// input is sorted by the lower key bits (all earlier passes), so the CTA's
// run covers a short range [lo_v, hi_v] of lower values and (lower - lo_v,
// digit) indexes a small SMEM table -- one shared atomic per record, flushed
// with one global atomic per non-empty bin.  Degenerate ranges fall back to
// one global atomic per record.
constexpr int TH_WARPS = US_THREADS / 32;
// warps that histogram tiles (their u32 histograms fit in 160 KB of SMEM)
__host__ __device__ constexpr int th_hist_warps(int bits) {
  return (160 * 1024) / (4 << bits) < TH_WARPS ? (160 * 1024) / (4 << bits) : TH_WARPS;
}

template <int BITS>
__global__ void __launch_bounds__(US_THREADS, 2) tile_hist_kernel(SortPass p, uint16_t* tcnt, uint32_t n_tiles,
                                                               uint32_t tiles_per_cta) {
  constexpr int BINS = 1 << BITS;
  constexpr int HW = th_hist_warps(BITS);
  extern __shared__ uint32_t th[];  // [HW][BINS] warp histograms, then count bins
  uint32_t* cnt = th + HW * BINS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tile0 = blockIdx.x * tiles_per_cta;
  const uint32_t tile1 = min(n_tiles, tile0 + tiles_per_cta);
  const uint64_t lo = (uint64_t)tile0 * DS_TILE;
  const uint64_t hi = min(p.n, (uint64_t)tile1 * DS_TILE);
  const uint32_t mask = BINS - 1;
  const uint32_t lm = (1u << p.shift) - 1;
  int mode = 0;  // 0 digits only, 1 key bins in SMEM, 2 key counts by global atomics
  uint32_t lo_v = 0, span = 1;
  if (p.last && p.counts && lo < hi) {
    if (p.shift == 0) {
      mode = 1;
    } else {
      lo_v = key_at(p, lo) & lm;
      const uint32_t hi_v = key_at(p, hi - 1) & lm;
      span = hi_v - lo_v + 1;
      mode = (hi_v >= lo_v && (uint64_t)span * BINS <= CNT_BINS) ? 1 : 2;
    }
    const uint32_t nb = mode == 1 ? span * BINS : 0;
    for (uint32_t i = threadIdx.x; i < nb; i += US_THREADS) cnt[i] = 0;
  }
  __syncthreads();
  uint32_t* wh = th + warp * BINS;
  bool saw_tmp = false;
  for (uint32_t t = tile0 + warp; warp < HW && t < tile1; t += HW) {
    for (int j = lane; j < BINS; j += 32) wh[j] = 0;
    __syncwarp();
    const uint64_t a = (uint64_t)t * DS_TILE, b = min(p.n, a + DS_TILE);
    const uint32_t nq = (uint32_t)((b - a) / 4);
    auto add_key = [&](uint32_t k) {
      if (p.first && p.lut && (k & SMX_TMP_KEY)) {
        saw_tmp = true;
        k = p.lut[k & ~SMX_TMP_KEY];
      }
      const uint32_t d = (k >> p.shift) & mask;
      atomicAdd(&wh[d], 1u);
      if (mode == 1) atomicAdd(&cnt[((k & lm) - lo_v) * BINS + d], 1u);
      else if (mode == 2) count_key(p, k, 1u);
    };
    if (b - a == DS_TILE) {
      // full tile: three 4-key groups per lane loaded before any is counted
      constexpr int PER = DS_TILE / 4 / 32;  // 30 groups of four keys per lane
      constexpr int G = 3;
      static_assert(PER % G == 0, "group count");
#pragma unroll 1
      for (int g0 = 0; g0 < PER; g0 += G) {
        uint32_t kk[G][4];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const uint32_t i = lane + (uint32_t)(g0 + u) * 32;
          if (p.recs_in) {
            const uint4* r4 = reinterpret_cast<const uint4*>(p.recs_in + a) + 2 * i;
            const uint4 q0 = __ldcs(r4), q1 = __ldcs(r4 + 1);
            kk[u][0] = q0.x; kk[u][1] = q0.z; kk[u][2] = q1.x; kk[u][3] = q1.z;
          } else {
            const uint4 q = __ldcs(reinterpret_cast<const uint4*>(p.keys_in + a) + i);
            kk[u][0] = q.x; kk[u][1] = q.y; kk[u][2] = q.z; kk[u][3] = q.w;
          }
        }
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int j = 0; j < 4; ++j) add_key(kk[u][j]);
      }
    }
    for (uint32_t i = lane; b - a != DS_TILE && i < nq + 1; i += 32) {
      uint32_t kk[4];
      int m = 4;
      if (i < nq) {
        if (p.recs_in) {  // four (key, value) records: two 16-byte loads
          const uint4* r4 = reinterpret_cast<const uint4*>(p.recs_in + a) + 2 * i;
          const uint4 q0 = r4[0], q1 = r4[1];
          kk[0] = q0.x; kk[1] = q0.z; kk[2] = q1.x; kk[3] = q1.z;
        } else {
          const uint4 q = reinterpret_cast<const uint4*>(p.keys_in + a)[i];
          kk[0] = q.x; kk[1] = q.y; kk[2] = q.z; kk[3] = q.w;
        }
      } else {  // ragged tail of the last tile
        m = (int)((b - a) - 4 * (uint64_t)nq);
#pragma unroll
        for (int j = 0; j < 4; ++j) kk[j] = j < m ? key_at(p, a + 4 * nq + j) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= m) break;
        add_key(kk[j]);
      }
    }
    __syncwarp();
    uint32_t* out = reinterpret_cast<uint32_t*>(tcnt + (size_t)t * BINS);
    for (int j = lane; j < BINS / 2; j += 32) out[j] = wh[2 * j] | (wh[2 * j + 1] << 16);
    __syncwarp();
  }
  if (p.tmp_flag && __any_sync(0xffffffffu, saw_tmp) && lane == 0) atomicOr(p.tmp_flag, 1u);
  if (mode == 1) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < span * BINS; i += US_THREADS) {
      const uint32_t c = cnt[i];
      if (c) count_key(p, (lo_v + i / BINS) | ((i % BINS) << p.shift), c);
    }
  }
}

// Column sums of tcnt over chunks of TC tiles: csum[chunk][d].
constexpr int TC = 256;
template <int BITS>
__global__ void __launch_bounds__(256) chunk_sum_kernel(const uint16_t* tcnt, uint32_t n_tiles, uint32_t* csum) {
  constexpr int BINS = 1 << BITS;
  const uint32_t c = blockIdx.x;
  const uint32_t t0 = c * TC, t1 = min(n_tiles, t0 + TC);
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t s = 0;
#pragma unroll 8
    for (uint32_t t = t0; t < t1; ++t) s += tcnt[(size_t)t * BINS + d];
    csum[(size_t)c * BINS + d] = s;
  }
}

// Single CTA: per digit, exclusive scan over chunks, offset by the digit's
// global base (exclusive scan of the digit totals).  In place on csum.
template <int BITS>
__global__ void __launch_bounds__(1024) chunk_scan_kernel(uint32_t* csum, uint32_t n_chunks) {
  constexpr int BINS = 1 << BITS;
  constexpr int DPT = (BINS + 1023) / 1024;
  __shared__ uint32_t ws[32];
  uint32_t tot[DPT];
  uint32_t mysum = 0;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = threadIdx.x * DPT + j;
    uint32_t s = 0;
    if (d < BINS) {
#pragma unroll 8
      for (uint32_t c = 0; c < n_chunks; ++c) s += csum[(size_t)c * BINS + d];
    }
    tot[j] = s;
    mysum += s;
  }
  uint32_t total;
  uint32_t base = smx::block_excl_scan(mysum, ws, total);
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = threadIdx.x * DPT + j;
    if (d < BINS) {
      uint32_t run = base;
      for (uint32_t c = 0; c < n_chunks; ++c) {
        const uint32_t x = csum[(size_t)c * BINS + d];
        csum[(size_t)c * BINS + d] = run;
        run += x;
      }
    }
    base += tot[j];
  }
}

// off[tile][d] = global output position of the tile's first record of digit d.
template <int BITS>
__global__ void __launch_bounds__(256) tile_offsets_kernel(const uint16_t* tcnt, const uint32_t* cbase,
                                                           uint32_t n_tiles, uint32_t* off) {
  constexpr int BINS = 1 << BITS;
  const uint32_t c = blockIdx.x;
  const uint32_t t0 = c * TC, t1 = min(n_tiles, t0 + TC);
  for (int d = threadIdx.x; d < BINS; d += 256) {
    uint32_t run = cbase[(size_t)c * BINS + d];
    for (uint32_t t = t0; t < t1; ++t) {
      off[(size_t)t * BINS + d] = run;
      run += tcnt[(size_t)t * BINS + d];
    }
  }
}

// Stable scatter by the digit (key >> shift) & (2^BITS-1).  CTAs take tiles
// in global order from an atomic ticket (one tile ahead, for the TMA
// prefetch): the tiles in flight are neighbours, so every digit's output
// grows at one frontier and a sector split between two tiles is completed
// while it is still in L2.  (Contiguous per-CTA segments left G frontiers per
// digit, and even a static interleave drifts by many tiles; both paid a DRAM
// read-modify-write per partial sector -- 2x the traffic of the pass.)  The
// tile's global digit offsets are precomputed (tile_hist -> chunk scans), so
// no tile waits on another.
// Per 3840-record tile:
//   load    the tile arrived in SMEM by TMA (cp.async.bulk + mbarrier) with
//           its offset row; each thread takes its 15 keys/values into
//           registers, so the buffer is free again and the next tile's TMA is
//           issued right after barrier 1
//   rank    warp-private u16 digit counters + ballot multisplit (stable)
//   scan    tile offsets; delta[d] = off[tile][d] - tile offset of d
//   stage   records to SMEM in digit order
//   write   coalesced runs: g = delta[d] + q
// Stable ranks of a warp's DS_IPT x 32 items (item i of lane l is the
// (i*32 + l)-th of the warp) within the warp's digit counters; invalid items
// (partial last tile) get 0xffff.  Packed two u16 per word.
template <int BITS, bool FULL>
__device__ __forceinline__ void rank_tile(const uint32_t (&k)[DS_IPT], uint32_t (&rank2)[(DS_IPT + 1) / 2],
                                          uint16_t* mycnt, int shift, uint64_t q0, uint64_t n, int lane) {
  constexpr uint32_t mask = (1u << BITS) - 1;
  const uint32_t lt_mask = (1u << lane) - 1;
#pragma unroll
  for (int i = 0; i < DS_IPT; ++i) {
    const bool valid = FULL || q0 + i * 32 < n;
    const uint32_t d = (k[i] >> shift) & mask;
    // warp multisplit: lanes holding the same digit, one ballot per bit.
    // Written in PTX so the bit tests become predicates (R2P) and the
    // complement is a predicated LOP3 -- about 3 instructions per bit.
    // (__match_any_sync measured 20% slower on B200 for 9-bit digits.)
    uint32_t peers = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
      asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bal;\n\t"
          "and.b32 t, %1, %2;\n\t"
          "setp.ne.u32 p, t, 0;\n\t"
          "vote.sync.ballot.b32 bal, p, 0xffffffff;\n\t"
          "@!p not.b32 bal, bal;\n\t"
          "and.b32 %0, %0, bal;\n\t}"
          : "+r"(peers) : "r"(d), "r"(1u << b));
    }
    if (!valid) peers = 1u << lane;
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = mycnt[d];
      mycnt[d] = (uint16_t)(old + __popc(peers));
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    const uint32_t r = valid ? old + __popc(peers & lt_mask) : 0xffffu;
    if (i & 1) rank2[i >> 1] |= r << 16; else rank2[i >> 1] = r;
  }
}

template <int BITS>
__global__ void __launch_bounds__(DS_THREADS, ds_ctas_per_sm(BITS)) downsweep_kernel(SortPass p, const uint32_t* off,
                                                                                    uint32_t n_tiles,
                                                                                    uint32_t* tile_ctr) {
  constexpr int BINS = 1 << BITS;
  constexpr int DPT = BINS / DS_THREADS;  // digits per thread (BITS >= 8)
  static_assert(DPT >= 1, "at least 8-bit digits");
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* ikey = reinterpret_cast<uint32_t*>(smem);  // [DS_TILE] TMA target
  uint32_t* ival = ikey + DS_TILE;                      // [DS_TILE] TMA target
  uint32_t* ioff = ival + DS_TILE;                      // [2][BINS] TMA target (offset rows)
  uint32_t* skey = ioff + 2 * BINS;                     // [DS_TILE] staging
  uint32_t* sval = skey + DS_TILE;                      // [DS_TILE] staging
  uint32_t* delta = sval + DS_TILE;                     // [BINS]
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(delta + BINS);  // [DS_WARPS][BINS]
  __shared__ uint32_t ws[32];
  __shared__ uint32_t ticket[2];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1;
  const uint32_t mask = BINS - 1;
  const bool has_vals = p.vals_in != nullptr || p.recs_in != nullptr;
  const bool any_tmp = p.first && p.lut && p.tmp_flag && *p.tmp_flag;  // temporary keys to resolve
  if (tid == 0) {
    smx::mbar_init(&bar, 1);
    smx::fence_mbar_init();
  }
  __syncthreads();
  // thread 0: TMA of tile t (keys, values if any, offset row into slot b)
  auto issue = [&](uint32_t t, int b) {
    const uint64_t t0 = (uint64_t)t * DS_TILE;
    const bool full = t0 + DS_TILE <= p.n;
    const uint32_t bytes = DS_TILE * 4;
    smx::mbar_expect_tx(&bar, BINS * 4 + (full ? (has_vals ? 2 * bytes : bytes) : 0));  // records: 2 * bytes
    smx::bulk_g2s(ioff + b * BINS, off + (size_t)t * BINS, BINS * 4, &bar);
    if (full) {
      if (p.recs_in) {
        smx::bulk_g2s(ikey, p.recs_in + t0, 2 * bytes, &bar);  // ikey|ival hold the records
      } else {
        smx::bulk_g2s(ikey, p.keys_in + t0, bytes, &bar);
        if (has_vals) smx::bulk_g2s(ival, p.vals_in + t0, bytes, &bar);
      }
    }
  };
  uint32_t phase = 0;
  if (tid == 0) {
    const uint32_t t = atomicAdd(tile_ctr, 1u);
    ticket[0] = t;
    if (t < n_tiles) issue(t, 0);
  }
  __syncthreads();
  const uint32_t wofs = warp * (32 * DS_IPT) + lane;
  uint16_t* mycnt = wcnt + warp * BINS;
  int slot = 0;
  for (uint32_t tile = ticket[0]; tile < n_tiles; tile = ticket[slot ^= 1]) {
    const uint64_t t0 = (uint64_t)tile * DS_TILE;
    const bool full = t0 + DS_TILE <= p.n;
    uint32_t k[DS_IPT], v[DS_IPT];
    smx::mbar_wait(&bar, phase);
    phase ^= 1;
    if (full) {
      if (p.recs_in) {
        const uint2* rin = reinterpret_cast<const uint2*>(ikey);
#pragma unroll
        for (int i = 0; i < DS_IPT; ++i) {
          const uint2 r = rin[wofs + i * 32];
          k[i] = r.x;
          v[i] = r.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < DS_IPT; ++i) {
          const uint32_t q = wofs + i * 32;
          k[i] = ikey[q];
          v[i] = has_vals ? ival[q] : (uint32_t)(t0 + q);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < DS_IPT; ++i) {
        const uint64_t idx = t0 + wofs + i * 32;
        const bool ok = idx < p.n;
        if (p.recs_in) {
          const uint2 r = ok ? p.recs_in[idx] : make_uint2(0u, 0u);
          k[i] = r.x;
          v[i] = r.y;
        } else {
          k[i] = ok ? p.keys_in[idx] : 0u;
          v[i] = ok ? (p.vals_in ? p.vals_in[idx] : (uint32_t)idx) : 0u;
        }
      }
    }
    if (any_tmp) {
#pragma unroll
      for (int i = 0; i < DS_IPT; ++i) k[i] = resolve(k[i], p.lut);
    }
    {
      uint32_t* w32 = reinterpret_cast<uint32_t*>(mycnt);
#pragma unroll
      for (int j = lane; j < BINS / 2; j += 32) w32[j] = 0;
      __syncwarp();
    }
    uint32_t rank2[(DS_IPT + 1) / 2];
    if (full) rank_tile<BITS, true>(k, rank2, mycnt, p.shift, 0, 0, lane);
    else rank_tile<BITS, false>(k, rank2, mycnt, p.shift, t0 + wofs, p.n, lane);
    __syncthreads();  // 1: counters complete, TMA buffers of this tile consumed
    if (tid == 0) {  // next ticket: tiles are taken in global order
      const uint32_t t = atomicAdd(tile_ctr, 1u);
      ticket[slot ^ 1] = t;
      if (t < n_tiles) {
        smx::fence_proxy_async();
        issue(t, slot ^ 1);
      }
    }
    uint32_t tot[DPT];
    uint32_t mysum = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < DS_WARPS; ++w) t += wcnt[w * BINS + d];
      tot[j] = t;
      mysum += t;
    }
    uint32_t tsum;
    uint32_t run = smx::block_excl_scan(mysum, ws, tsum);
    const uint32_t* orow = ioff + slot * BINS;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      uint32_t t = run;
#pragma unroll
      for (int w = 0; w < DS_WARPS; ++w) {
        const uint32_t c = wcnt[w * BINS + d];
        wcnt[w * BINS + d] = (uint16_t)t;
        t += c;
      }
      delta[d] = orow[d] - run;
      run += tot[j];
    }
    __syncthreads();  // 2: offsets ready
#pragma unroll
    for (int i = 0; i < DS_IPT; ++i) {
      const uint32_t r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
      if (r != 0xffffu) {
        const uint32_t d = (k[i] >> p.shift) & mask;
        const uint32_t pos = mycnt[d] + r;
        skey[pos] = k[i];
        sval[pos] = v[i];
      }
    }
    __syncthreads();  // 3: tile staged in digit order
    for (uint32_t q = tid; q < tsum; q += DS_THREADS) {
      const uint32_t kk = skey[q];
      const uint32_t g = delta[(kk >> p.shift) & mask] + q;
      if (p.last) p.vals_out[g] = sval[q];
      else p.recs_out[g] = make_uint2(kk, sval[q]);  // one 8-byte store per record
    }
  }
}

// Downsweep with the staging aliased onto the TMA input buffer and a
// single-buffered offset row: 30 + 2*BINS*4 + 16*BINS bytes of SMEM (38 KB at
// 8 bits, 48 KB at 10) instead of 60 + ..., so more CTAs per SM.  The next
// tile's input is fetched after the write phase (the other CTAs of the SM
// cover the load); its offset row right after the scan.
//   LAST:  (key, value) records in, values out (staging: values + u16 digits)
//   !LAST: SoA keys/values, index values or records in; records out
//          (staging: keys + values)
#ifndef SMX_DS_ALIAS_CTAS
#define SMX_DS_ALIAS_CTAS 3
#endif
constexpr int ds_last_ctas_per_sm(int bits) { return bits <= 9 ? SMX_DS_ALIAS_CTAS : bits <= 10 ? 3 : 2; }

template <int BITS, bool LAST>
__global__ void __launch_bounds__(DS_THREADS, ds_last_ctas_per_sm(BITS)) downsweep_last_kernel(
    SortPass p, const uint32_t* off, uint32_t n_tiles, uint32_t* tile_ctr) {
  constexpr int BINS = 1 << BITS;
  constexpr int DPT = BINS / DS_THREADS;
  extern __shared__ __align__(128) uint8_t smem[];
  uint2* irec = reinterpret_cast<uint2*>(smem);                           // [DS_TILE] TMA target (records)
  uint32_t* ikey = reinterpret_cast<uint32_t*>(smem);                     // [DS_TILE] TMA target (SoA keys)
  uint32_t* ival = ikey + DS_TILE;                                        // [DS_TILE] TMA target (SoA values)
  uint32_t* sval = reinterpret_cast<uint32_t*>(smem);                     // LAST staging, aliases the input
  uint16_t* sdig = reinterpret_cast<uint16_t*>(sval + DS_TILE);           // LAST staging digits
  uint32_t* skey = ikey;                                                  // !LAST staging keys
  uint32_t* svl2 = ival;                                                  // !LAST staging values
  uint32_t* ioff = reinterpret_cast<uint32_t*>(smem + (size_t)DS_TILE * 8);  // [BINS] TMA target
  uint32_t* delta = ioff + BINS;                                          // [BINS]
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(delta + BINS);             // [DS_WARPS][BINS]
  __shared__ uint32_t ws[32];
  __shared__ uint32_t ticket[2];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t mask = BINS - 1;
  const bool soa_vals = !p.recs_in && p.vals_in;
  const bool any_tmp = !LAST && p.first && p.lut && p.tmp_flag && *p.tmp_flag;
  const uint32_t in_bytes = (p.recs_in || soa_vals) ? DS_TILE * 8 : DS_TILE * 4;
  if (tid == 0) {
    smx::mbar_init(&bar, 1);
    smx::fence_mbar_init();
  }
  __syncthreads();
  auto full_tile = [&](uint32_t t) { return (uint64_t)t * DS_TILE + DS_TILE <= p.n; };
  auto load_input = [&](uint32_t t) {  // thread 0, after expect_tx
    const uint64_t t0 = (uint64_t)t * DS_TILE;
    if (p.recs_in) {
      smx::bulk_g2s(irec, p.recs_in + t0, DS_TILE * 8, &bar);
    } else {
      smx::bulk_g2s(ikey, p.keys_in + t0, DS_TILE * 4, &bar);
      if (soa_vals) smx::bulk_g2s(ival, p.vals_in + t0, DS_TILE * 4, &bar);
    }
  };
  if (tid == 0) {
    const uint32_t t = atomicAdd(tile_ctr, 1u);
    ticket[0] = t;
    if (t < n_tiles) {
      smx::mbar_expect_tx(&bar, BINS * 4 + (full_tile(t) ? in_bytes : 0));
      smx::bulk_g2s(ioff, off + (size_t)t * BINS, BINS * 4, &bar);
      if (full_tile(t)) load_input(t);
    }
  }
  __syncthreads();
  const uint32_t wofs = warp * (32 * DS_IPT) + lane;
  uint16_t* mycnt = wcnt + warp * BINS;
  uint32_t phase = 0;
  int slot = 0;
  for (uint32_t tile = ticket[0]; tile < n_tiles; tile = ticket[slot ^= 1]) {
    const uint64_t t0 = (uint64_t)tile * DS_TILE;
    const bool full = full_tile(tile);
    uint32_t k[DS_IPT], v[DS_IPT];
    smx::mbar_wait(&bar, phase);
    phase ^= 1;
#pragma unroll
    for (int i = 0; i < DS_IPT; ++i) {
      const uint32_t q = wofs + i * 32;
      const uint64_t idx = t0 + q;
      if (p.recs_in) {
        uint2 r;
        if (full) r = irec[q];
        else r = idx < p.n ? p.recs_in[idx] : make_uint2(0u, 0u);
        k[i] = r.x;
        v[i] = r.y;
      } else if (full) {
        k[i] = ikey[q];
        v[i] = soa_vals ? ival[q] : (uint32_t)idx;
      } else {
        const bool ok = idx < p.n;
        k[i] = ok ? p.keys_in[idx] : 0u;
        v[i] = ok ? (soa_vals ? p.vals_in[idx] : (uint32_t)idx) : 0u;
      }
    }
    if (any_tmp) {
#pragma unroll
      for (int i = 0; i < DS_IPT; ++i) k[i] = resolve(k[i], p.lut);
    }
    {
      uint32_t* w32 = reinterpret_cast<uint32_t*>(mycnt);
#pragma unroll
      for (int j = lane; j < BINS / 2; j += 32) w32[j] = 0;
      __syncwarp();
    }
    uint32_t rank2[(DS_IPT + 1) / 2];
    if (full) rank_tile<BITS, true>(k, rank2, mycnt, p.shift, 0, 0, lane);
    else rank_tile<BITS, false>(k, rank2, mycnt, p.shift, t0 + wofs, p.n, lane);
    __syncthreads();  // 1: counters complete, records in registers
    if (tid == 0) ticket[slot ^ 1] = atomicAdd(tile_ctr, 1u);
    uint32_t tot[DPT];
    uint32_t mysum = 0;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < DS_WARPS; ++w) t += wcnt[w * BINS + d];
      tot[j] = t;
      mysum += t;
    }
    uint32_t tsum;
    uint32_t run = smx::block_excl_scan(mysum, ws, tsum);
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const int d = tid * DPT + j;
      uint32_t t = run;
#pragma unroll
      for (int w = 0; w < DS_WARPS; ++w) {
        const uint32_t c = wcnt[w * BINS + d];
        wcnt[w * BINS + d] = (uint16_t)t;
        t += c;
      }
      delta[d] = ioff[d] - run;
      run += tot[j];
    }
    __syncthreads();  // 2: offsets ready; the offset row and the input buffer are free
    const uint32_t nxt = ticket[slot ^ 1];
    if (tid == 0 && nxt < n_tiles) {
      smx::fence_proxy_async();
      smx::mbar_expect_tx(&bar, BINS * 4 + (full_tile(nxt) ? in_bytes : 0));
      smx::bulk_g2s(ioff, off + (size_t)nxt * BINS, BINS * 4, &bar);
    }
#pragma unroll
    for (int i = 0; i < DS_IPT; ++i) {
      const uint32_t r = (rank2[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
      if (r != 0xffffu) {
        const uint32_t d = (k[i] >> p.shift) & mask;
        const uint32_t pos = mycnt[d] + r;
        if (LAST) {
          sval[pos] = v[i];
          sdig[pos] = (uint16_t)d;
        } else {
          skey[pos] = k[i];
          svl2[pos] = v[i];
        }
      }
    }
    __syncthreads();  // 3: tile staged in digit order
    if (LAST) {
      for (uint32_t q = tid; q < tsum; q += DS_THREADS) p.vals_out[delta[sdig[q]] + q] = sval[q];
    } else {
      for (uint32_t q = tid; q < tsum; q += DS_THREADS) {
        const uint32_t kk = skey[q];
        p.recs_out[delta[(kk >> p.shift) & mask] + q] = make_uint2(kk, svl2[q]);
      }
    }
    __syncthreads();  // 4: staging read: the input buffer may be refilled
    if (tid == 0 && nxt < n_tiles && full_tile(nxt)) {
      smx::fence_proxy_async();
      load_input(nxt);
    }
  }
}

template <int BITS>
size_t downsweep_last_smem() {
  return (size_t)DS_TILE * 8 + (size_t)2 * (1 << BITS) * 4 + (size_t)DS_WARPS * (1 << BITS) * 2;
}

template <int BITS>
size_t downsweep_smem() {
  return (size_t)4 * DS_TILE * 4 + (size_t)3 * (1 << BITS) * 4 + (size_t)DS_WARPS * (1 << BITS) * 2;
}

// One pass (histograms, offsets, scatter) with BITS-wide digits.
template <int BITS>
int run_pass(const SortPass& p, uint32_t n_tiles, uint16_t* tcnt, uint32_t* off, uint32_t* csum,
             uint32_t* tile_ctr, cudaStream_t st) {
  constexpr int BINS = 1 << BITS;
  const size_t smem = downsweep_smem<BITS>();
  const size_t smem_last = downsweep_last_smem<BITS>();
  const size_t th_smem = (size_t)4 * (th_hist_warps(BITS) * BINS + CNT_BINS);
  static unsigned long long configured = 0;   // one bit per device
  const unsigned long long dbit = smx_device_bit();
  if (!(configured & dbit)) {
    SMX_CUDA_CHECK(cudaFuncSetAttribute(downsweep_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    SMX_CUDA_CHECK(cudaFuncSetAttribute(downsweep_last_kernel<BITS, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_last));
    SMX_CUDA_CHECK(cudaFuncSetAttribute(downsweep_last_kernel<BITS, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_last));
    SMX_CUDA_CHECK(cudaFuncSetAttribute(tile_hist_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)th_smem));
    configured |= dbit;
  }
  const uint32_t n_chunks = (n_tiles + TC - 1) / TC;
  const uint32_t hg = std::min<uint32_t>(n_tiles, 148 * 2);
  const uint32_t tpc = (n_tiles + hg - 1) / hg;
  const uint32_t hgrid = (n_tiles + tpc - 1) / tpc;
  const uint32_t grid = std::min<uint32_t>(n_tiles, 148u * ds_ctas_per_sm(BITS));
  smx_count_launch(); tile_hist_kernel<BITS><<<hgrid, US_THREADS, th_smem, st>>>(p, tcnt, n_tiles, tpc);
  smx_count_launch(); chunk_sum_kernel<BITS><<<n_chunks, 256, 0, st>>>(tcnt, n_tiles, csum);
  smx_count_launch(); chunk_scan_kernel<BITS><<<1, 1024, 0, st>>>(csum, n_chunks);
  smx_count_launch(); tile_offsets_kernel<BITS><<<n_chunks, 256, 0, st>>>(tcnt, csum, n_tiles, off);
  // A/B switches: SMX_SORT_LAST=0 disables the aliased last pass; SMX_SORT_ALIAS=<min bits> uses the
  // aliased kernel for last passes from that width and SMX_SORT_ALIAS_MID=<min bits> for record-out passes.
  static const bool last_ok = !getenv("SMX_SORT_LAST") || atoi(getenv("SMX_SORT_LAST")) != 0;
  static const int alias_last = getenv("SMX_SORT_ALIAS") ? atoi(getenv("SMX_SORT_ALIAS")) : 10;
  static const int alias_mid = getenv("SMX_SORT_ALIAS_MID") ? atoi(getenv("SMX_SORT_ALIAS_MID")) : 99;
  const uint32_t g2 = std::min<uint32_t>(n_tiles, 148u * ds_last_ctas_per_sm(BITS));
  if (p.last && p.recs_in && BITS >= alias_last && last_ok) {
    smx_count_launch();
    downsweep_last_kernel<BITS, true><<<g2, DS_THREADS, smem_last, st>>>(p, off, n_tiles, tile_ctr);
  } else if (!p.last && BITS >= alias_mid) {
    smx_count_launch();
    downsweep_last_kernel<BITS, false><<<g2, DS_THREADS, smem_last, st>>>(p, off, n_tiles, tile_ctr);
  } else {
    smx_count_launch(); downsweep_kernel<BITS><<<grid, DS_THREADS, smem, st>>>(p, off, n_tiles, tile_ctr);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}

int run_pass_bits(int bits, const SortPass& p, uint32_t n_tiles, uint16_t* tcnt, uint32_t* off, uint32_t* csum,
                  uint32_t* tile_ctr, cudaStream_t st) {
  switch (bits) {
    case 8: return run_pass<8>(p, n_tiles, tcnt, off, csum, tile_ctr, st);
    case 9: return run_pass<9>(p, n_tiles, tcnt, off, csum, tile_ctr, st);
    case 10: return run_pass<10>(p, n_tiles, tcnt, off, csum, tile_ctr, st);
    default: return run_pass<11>(p, n_tiles, tcnt, off, csum, tile_ctr, st);
  }
}

// passes of pass_bits[0..passes) digit bits, least significant first
int run_sort(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b, uint64_t n,
             const int* pass_bits, int passes, int index_values, const uint32_t* lut, uint32_t* counts,
             uint64_t n_keys, int* out_in_b, cudaStream_t st) {
  int max_bits = 8;
  for (int i = 0; i < passes; ++i) max_bits = std::max(max_bits, pass_bits[i]);
  const uint32_t max_bins = 1u << max_bits;
  const uint32_t n_tiles = (uint32_t)((n + DS_TILE - 1) / DS_TILE);
  const uint32_t n_chunks = (n_tiles + TC - 1) / TC;
  uint16_t* tcnt = nullptr;
  uint32_t *off = nullptr, *csum = nullptr, *ctr = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&ctr, sizeof(uint32_t) * (passes + 1), st));
  SMX_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(uint32_t) * (passes + 1), st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&tcnt, sizeof(uint16_t) * n_tiles * max_bins, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&off, sizeof(uint32_t) * n_tiles * max_bins, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&csum, sizeof(uint32_t) * n_chunks * max_bins, st));
  // Intermediate passes move (key, value) records as one 8-byte item (AoS):
  // half the store instructions and twice the bytes per scattered run of the
  // SoA layout.  X lives in the scratch pair when keys_b | vals_b are
  // contiguous, Y (three or more passes) in keys_a | vals_a likewise.
  uint2* X = vals_b == keys_b + n ? reinterpret_cast<uint2*>(keys_b) : nullptr;
  uint2* Y = nullptr;
  uint2* own = nullptr;
  if (passes > 1 && !X) {
    SMX_CUDA_CHECK(cudaMallocAsync((void**)&own, sizeof(uint2) * n * (passes > 2 ? 2 : 1), st));
    X = own;
  }
  if (passes > 2) Y = own ? own + n : (vals_a == keys_a + n ? reinterpret_cast<uint2*>(keys_a) : nullptr);
  if (passes > 2 && !Y) {
    SMX_CUDA_CHECK(cudaMallocAsync((void**)&own, sizeof(uint2) * n, st));
    Y = own;
  }
  int shift = 0;
  for (int pass = 0; pass < passes; ++pass) {
    SortPass p{};
    const uint2* in = pass == 0 ? nullptr : (pass & 1 ? X : Y);
    if (pass == 0) {
      p.keys_in = keys_a;
      p.vals_in = index_values ? nullptr : vals_a;
    } else {
      p.recs_in = in;
    }
    p.first = pass == 0;
    p.last = pass == passes - 1;
    p.shift = shift;
    p.n = n;
    p.lut = lut;
    p.counts = counts;
    p.n_keys = n_keys;
    if (!p.last) {
      p.recs_out = pass & 1 ? Y : X;
    } else {
      // values land in whichever SoA value array does not overlap the input
      const bool in_b = pass == 0 || in == reinterpret_cast<const uint2*>(keys_b);
      p.vals_out = in_b ? (pass == 0 ? vals_b : vals_a) : vals_b;
      *out_in_b = p.vals_out == vals_b ? 1 : 0;
    }
    p.tmp_flag = ctr + passes;
    if (int rc = run_pass_bits(pass_bits[pass], p, n_tiles, tcnt, off, csum, ctr + pass, st)) return rc;
    shift += pass_bits[pass];
  }
  if (own) cudaFreeAsync(own, st);
  cudaFreeAsync(tcnt, st);
  cudaFreeAsync(off, st);
  cudaFreeAsync(csum, st);
  cudaFreeAsync(ctr, st);
  return 0;
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
  // digit plan: 9-bit lower passes (three CTAs per SM), the last pass takes
  // the rest up to 10 bits (values only, the cheapest scatter); an env cap
  // (tuning) forces equal passes of at most that many bits
  static const int cap = getenv("SMX_SORT_MAX_BITS") ? atoi(getenv("SMX_SORT_MAX_BITS")) : 0;
  int bits[8];
  int passes = 0;
  if (cap > 0) {
    const int np = (key_bits + cap - 1) / cap;
    for (int i = 0; i < np; ++i) bits[passes++] = std::max((key_bits + np - 1) / np, 8);
  } else if (key_bits <= 11) {
    bits[passes++] = std::max(key_bits, 8);
  } else if (key_bits == 20) {  // a 9 + 11 split measured slower than 10 + 10
    bits[passes++] = 10;
    bits[passes++] = 10;
  } else if (key_bits > 20 && key_bits <= 22) {
    bits[passes++] = key_bits - 11;
    bits[passes++] = 11;
  } else {
    int rest = key_bits;
    while (rest > 10) {
      bits[passes++] = 9;
      rest -= 9;
    }
    bits[passes++] = std::max(rest, 8);
  }
  return run_sort(keys_a, vals_a, keys_b, vals_b, n, bits, passes, index_values, lut, counts, n_keys, out_in_b, st);
}
