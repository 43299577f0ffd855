// Ordered Lemire draw engine: numpy `Generator.integers(lo, lo+ex, size=n)`
// on a Philox stream starting at an arbitrary u32 cursor, parallelised as
// "accept-mask + ordered compaction" (every raw u32 draw, first try or retry,
// is accepted by the same predicate, so the n-th accepted raw u32 is the
// n-th output value; verified against numpy in tests/test_oracle_rng.py).
//
// Default: one launch per draw call (draw_onepass_kernel, below): ticketed
// tiles, each drawn once, output bases by a decoupled look-back.
// A/B path (SMX_DRAW_ONEPASS=0), two launches per draw call:
//   count:  warp w counts accepts over its contiguous raw range (compute only)
//   write:  warp w regenerates its range, ranks accepts with a warp scan,
//           stages them in its own SMEM slice and hands (output index, value)
//           to a Sink functor with coalesced indices.  Warps never wait for
//           each other (no CTA barrier inside the loop).
// A tiny single-CTA scan between them turns per-warp counts into offsets.
#pragma once
#include "common.cuh"

namespace smx {

constexpr int DRAW_THREADS = 256;

struct DrawRange {
  Key key;
  uint64_t u0;       // first raw u32 position (replaced by *u0_dev when set)
  const uint64_t* u0_dev;  // device cursor written by an earlier draw of the same stream, or null
  uint64_t n_raw;     // raw positions covered by the launch
  uint64_t per_warp;  // raw positions per warp (multiple of 8)
  Lemire lm;
};

// Accept mask and values for the 8 u32 draws of Philox block `blk`,
// restricted to raw positions in [lo, hi).
__device__ __forceinline__ uint32_t block_accepts(const DrawRange& r, uint64_t blk, uint64_t lo,
                                                  uint64_t hi, uint32_t vals[8]) {
  uint64_t w[4];
  philox4x64_10(blk, r.key, w);
  const uint64_t p0 = (blk - 1) * 8;
  uint32_t mask = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t v = (i & 1) ? (uint32_t)(w[i >> 1] >> 32) : (uint32_t)w[i >> 1];
    uint32_t out;
    const bool ok = r.lm.accept(v, out);
    vals[i] = out;
    mask |= (ok ? 1u : 0u) << i;
  }
  if (p0 < lo || p0 + 8 > hi) {  // block straddles the range edge (rare)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (p0 + i < lo || p0 + i >= hi) mask &= ~(1u << i);
  }
  return mask;
}

constexpr int DRAW_WARPS = DRAW_THREADS / 32;

__device__ __forceinline__ void warp_range(const DrawRange& r, uint64_t& lo, uint64_t& hi) {
  const uint64_t gw = (uint64_t)blockIdx.x * DRAW_WARPS + (threadIdx.x >> 5);
  lo = r.u0 + gw * r.per_warp;
  const uint64_t end = r.u0 + r.n_raw;
  hi = lo + r.per_warp < end ? lo + r.per_warp : end;
}

#ifndef SMX_DRAW_COUNT_MB
#define SMX_DRAW_COUNT_MB 3
#endif
static __global__ void __launch_bounds__(DRAW_THREADS, SMX_DRAW_COUNT_MB) draw_count_kernel(DrawRange r, uint32_t* warp_counts) {
  uint64_t lo, hi;
  warp_range(r, lo, hi);
  uint32_t cnt = 0;
  if (lo < hi) {
    const uint64_t b0 = lo / 8 + 1, b1 = (hi - 1) / 8 + 1;
    for (uint64_t b = b0 + (threadIdx.x & 31); b <= b1; b += 32) {
      uint32_t v[8];
      cnt += __popc(block_accepts(r, b, lo, hi, v));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) warp_counts[(uint64_t)blockIdx.x * DRAW_WARPS + (threadIdx.x >> 5)] = cnt;
}

// Exclusive scan of per-warp counts (n <= some ten thousand) into 64-bit offsets;
// offsets[n] = total.
static __global__ void cta_offsets_kernel(const uint32_t* counts, int n, uint64_t* offsets) {
  __shared__ uint32_t ws[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const uint32_t x = i < n ? counts[i] : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(x, ws, tot);
    if (i < n) offsets[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[n] = carry;
}

// Sink contract: `template <bool ALL> void batch(uint64_t j0, uint32_t stride,
// const uint32_t v[8], uint32_t ok, uint32_t keys_out[8])` consumes values
// v[u] (bit u of ok set; ALL: every bit set)
// for output indices j0 + u*stride and reports the record keys it wrote;
// `void operator()(uint64_t j, uint32_t value)` consumes one item.
// Sinks must be idempotent: when a synchronous call's raw window turns out
// too short, run_draw widens it and launches again, so the same (j, value)
// can be handed over more than once (every sink here stores positionally or
// ORs marks; an accumulating sink would double-count).
// Optional used-value marking fused into the write pass: bit
// (tab ? tab[value] : value) of `bits` is set for every emitted draw; with
// from_key the bit comes from the sink's key instead: temporary keys mark
// (key & ~TMP) - tmp_base, direct (local) keys mark local_bit.  Small bitmaps
// are accumulated in shared memory and OR-ed out once per CTA; only first
// sightings pay an atomic.
struct DrawMark {
  uint32_t* bits;
  const uint32_t* tab;
  uint32_t nwords;  // bitmap size
  int in_smem;      // nwords fit the dynamic shared-memory bitmap
  int from_key;
  uint32_t tmp_base;
  uint32_t local_bit;
};

constexpr uint32_t DRAW_MARK_SMEM_WORDS = 12288;  // 48 KB
#ifndef SMX_DRAW_BPT
#define SMX_DRAW_BPT 1  // measured: 1 block per lane 4.94 ms, 2: 5.23 ms, 4: 7.69 ms (C3 generation)
#endif
constexpr int DRAW_BPT = SMX_DRAW_BPT;  // Philox blocks per lane per iteration

// MARK: 0 no marking, 1 bit from the sink's key, 2 bit from the value (via tab)
template <int MARK>
__device__ __forceinline__ uint32_t mark_bit(const DrawMark& mk, uint32_t key, uint32_t value) {
  if (MARK == 1) return (key & SMX_TMP_KEY) ? (key & ~SMX_TMP_KEY) - mk.tmp_base : mk.local_bit;
  return mk.tab ? __ldg(mk.tab + value) : value;
}

#ifndef SMX_DRAW_MIN_BLOCKS
#define SMX_DRAW_MIN_BLOCKS 3
#endif
template <class Sink, int MARK>
__global__ void __launch_bounds__(DRAW_THREADS, SMX_DRAW_MIN_BLOCKS) draw_write_kernel(DrawRange r, const uint64_t* warp_offsets,
                                                                  uint64_t n_out, Sink sink, uint64_t* cursor_out,
                                                                  DrawMark mk) {
  extern __shared__ uint32_t smark[];
  __shared__ uint32_t sv_all[DRAW_WARPS][32 * 8 * DRAW_BPT];  // a warp's accepted values of one iteration
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* sv = sv_all[warp];
  if (MARK && mk.in_smem) {
    for (uint32_t w = threadIdx.x; w < mk.nwords; w += blockDim.x) smark[w] = 0;
    __syncthreads();
  }
  uint64_t lo, hi;
  warp_range(r, lo, hi);
  uint64_t base = warp_offsets[(uint64_t)blockIdx.x * DRAW_WARPS + warp];
  bool saw_local = false;
  if (lo < hi && base < n_out) {
    const uint64_t b0 = lo / 8 + 1, b1 = (hi - 1) / 8 + 1;
    for (uint64_t bb = b0; bb <= b1 && base < n_out; bb += (uint64_t)DRAW_BPT * 32) {
      // lane l owns blocks bb + BPT*l .. +BPT-1: raw order = lane order
      uint32_t v[DRAW_BPT][8];
      uint32_t mask[DRAW_BPT];
      uint32_t cnt = 0;
#pragma unroll
      for (int q = 0; q < DRAW_BPT; ++q) {
        const uint64_t b = bb + (uint64_t)DRAW_BPT * lane + q;
        mask[q] = b <= b1 ? block_accepts(r, b, lo, hi, v[q]) : 0u;
        cnt += __popc(mask[q]);
      }
      const uint32_t inc = warp_incl_scan(cnt);
      const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
      uint32_t k = inc - cnt;
      if (cursor_out && base + tot >= n_out) {  // this iteration holds the last output
        const uint64_t want = n_out - 1 - base;   // its index within the iteration
        if (want >= k && want < inc) {
          uint32_t left = (uint32_t)(want - k);
#pragma unroll
          for (int q = 0; q < DRAW_BPT; ++q) {
            const uint32_t c = __popc(mask[q]);
            if (left < c && left != 0xffffffffu) {
              uint32_t m = mask[q];
              for (uint32_t z = 0; z < left; ++z) m &= m - 1;
              const uint64_t b = bb + (uint64_t)DRAW_BPT * lane + q;
              *cursor_out = (b - 1) * 8 + (__ffs(m) - 1) + 1;
              left = 0xffffffffu;
            } else if (left != 0xffffffffu) {
              left -= c;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < DRAW_BPT; ++q) {
        if (mask[q] == 0xffu) {  // no rejection in the block (the common case)
#pragma unroll
          for (int i = 0; i < 8; ++i) sv[k + i] = v[q][i];
          k += 8;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // static indexing keeps v[] in registers
            if ((mask[q] >> i) & 1u) sv[k++] = v[q][i];
          }
        }
      }
      __syncwarp();
      // coalesced hand-off: consecutive lanes own consecutive output indices;
      // a lane's items go over in batches of 8 so their gathers overlap
      const bool all = tot == 256 * DRAW_BPT && base + tot <= n_out;  // every slot valid
#pragma unroll
      for (int h = 0; h < DRAW_BPT; ++h) {
        if ((uint32_t)h * 256 >= tot) break;
        uint32_t vv[8], kk[8];
        uint32_t okm = 0xffu;
        if (all) {
#pragma unroll
          for (int u = 0; u < 8; ++u) vv[u] = sv[lane + (h * 8 + u) * 32];
          sink.template batch<true>(base + lane + (uint64_t)h * 256, 32, vv, okm, kk);
        } else {
          okm = 0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t q = lane + (h * 8 + u) * 32;
            const bool ok = q < tot && base + q < n_out;
            vv[u] = ok ? sv[q] : 0u;
            okm |= (ok ? 1u : 0u) << u;
          }
          sink.template batch<false>(base + lane + (uint64_t)h * 256, 32, vv, okm, kk);
        }
        if (MARK) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (!((okm >> u) & 1u)) continue;
            if (MARK == 1 && !(kk[u] & SMX_TMP_KEY)) {  // local key: one bit for all, set once below
              saw_local = true;
              continue;
            }
            const uint32_t bit = mark_bit<MARK>(mk, kk[u], vv[u]);
            if (bit == 0xffffffffu) continue;
            const uint32_t m = 1u << (bit & 31);
            uint32_t* w = mk.in_smem ? &smark[bit >> 5] : &mk.bits[bit >> 5];
            if (!(*(volatile uint32_t*)w & m)) atomicOr(w, m);
          }
        }
      }
      base += tot;
      __syncwarp();
    }
  }
  if (MARK == 1 && __any_sync(0xffffffffu, saw_local) && lane == 0 && mk.local_bit != 0xffffffffu) {
    const uint32_t b = mk.local_bit;
    atomicOr(mk.in_smem ? &smark[b >> 5] : &mk.bits[b >> 5], 1u << (b & 31));
  }
  if (MARK && mk.in_smem) {
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < mk.nwords; w += blockDim.x) {
      const uint32_t x = smark[w];
      if (x & ~__ldcg(&mk.bits[w])) atomicOr(&mk.bits[w], x);
    }
  }
}

// ---------------------------------------------------------------------------
// One-pass variant: the count pass and the offset scan fold into the write
// pass through a decoupled look-back over raw tiles of OP_TILE positions.
// A warp takes tile t from an atomic ticket (so every earlier tile belongs to
// a warp that is already running), draws it once into its SMEM slice,
// publishes the tile's accept count (flag A), walks back over the
// predecessors' descriptors until one carries an inclusive prefix (flag P),
// publishes its own inclusive prefix and hands the staged values to the sink
// exactly as draw_write_kernel does.  Philox runs once per raw position
// instead of twice.
#ifndef SMX_DRAW_TILE
#define SMX_DRAW_TILE 2048  // measured (C3 generation): 512 6.98 ms, 1024 4.53, 2048 3.88, 4096 5.27
#endif
constexpr int OP_TILE = SMX_DRAW_TILE;  // default raw positions per tile (multiple of 256)
#ifndef SMX_LOOKBACK_SLEEP_NS
#define SMX_LOOKBACK_SLEEP_NS 0  // back-off while a predecessor draws; 0 / 64 / 256 ns measured equal (3.87-3.90 ms)
#endif
constexpr uint64_t OP_FLAG_A = 1ull << 62, OP_FLAG_P = 2ull << 62, OP_VAL = (1ull << 62) - 1;

// Raw position (plus one) of the want-th accepted draw in [lo, hi); whole warp.
__device__ __forceinline__ uint64_t nth_accept_cursor(const DrawRange& r, uint64_t lo, uint64_t hi, uint32_t want) {
  const int lane = threadIdx.x & 31;
  const uint64_t b0 = lo / 8 + 1, b1 = (hi - 1) / 8 + 1;
  uint64_t cur = 0;
  for (uint64_t bb = b0; bb <= b1; bb += 32) {
    const uint64_t b = bb + lane;
    uint32_t v[8];
    const uint32_t mask = b <= b1 ? block_accepts(r, b, lo, hi, v) : 0u;
    const uint32_t cnt = __popc(mask);
    const uint32_t inc = warp_incl_scan(cnt);
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    const uint32_t k = inc - cnt;
    if (want < tot) {
      if (want >= k && want < inc) {
        uint32_t m = mask;
        for (uint32_t z = 0; z < want - k; ++z) m &= m - 1;
        cur = (b - 1) * 8 + (__ffs(m) - 1) + 1;
      }
      break;
    }
    want -= tot;
  }
  // the owning lane holds the answer; everyone else 0
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cur |= __shfl_xor_sync(0xffffffffu, cur, o);
  return cur;
}

template <class Sink, int MARK>
__global__ void __launch_bounds__(DRAW_THREADS, SMX_DRAW_MIN_BLOCKS)
    draw_onepass_kernel(DrawRange r_in, uint32_t tile, uint32_t n_tiles, uint64_t* desc, uint32_t* ticket,
                        uint64_t* total_out, uint64_t n_out, Sink sink, uint64_t* cursor_out, DrawMark mk) {
  DrawRange r = r_in;
  if (r_in.u0_dev) r.u0 = *r_in.u0_dev;   // chained draw: starts where the previous one ended
  extern __shared__ uint32_t op_smem[];  // [DRAW_WARPS][tile] accepted values, then the mark bitmap
  uint32_t* smark = op_smem + DRAW_WARPS * tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* sv = op_smem + warp * tile;
  if (MARK && mk.in_smem) {
    for (uint32_t w = threadIdx.x; w < mk.nwords; w += blockDim.x) smark[w] = 0;
    __syncthreads();
  }
  bool saw_local = false;
  const uint64_t end = r.u0 + r.n_raw;
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_tiles) break;
    const uint64_t lo = r.u0 + (uint64_t)t * tile;
    const uint64_t hi = lo + tile < end ? lo + tile : end;
    // draw the tile once, compacted into SMEM in raw order
    const uint64_t b0 = lo / 8 + 1, b1 = (hi - 1) / 8 + 1;
    uint32_t n_acc = 0;
    for (uint64_t bb = b0; bb <= b1; bb += 32) {
      const uint64_t b = bb + lane;
      uint32_t v[8];
      const uint32_t mask = b <= b1 ? block_accepts(r, b, lo, hi, v) : 0u;
      const uint32_t cnt = __popc(mask);
      const uint32_t inc = warp_incl_scan(cnt);
      uint32_t k = n_acc + inc - cnt;
      if (mask == 0xffu) {
#pragma unroll
        for (int i = 0; i < 8; ++i) sv[k + i] = v[i];
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if ((mask >> i) & 1u) sv[k++] = v[i];
      }
      n_acc += __shfl_sync(0xffffffffu, inc, 31);
    }
    // publish the aggregate, look back (32 predecessors per warp-wide read)
    // for the exclusive prefix
    uint64_t base = 0;
    volatile uint64_t* vd = desc;
    if (t == 0) {
      if (lane == 0) vd[0] = OP_FLAG_P | n_acc;
    } else {
      if (lane == 0) vd[t] = OP_FLAG_A | n_acc;
      for (int64_t j = (int64_t)t - 1;;) {
        const int64_t idx = j - lane;
        const uint64_t d = idx >= 0 ? vd[idx] : (OP_FLAG_P + 0);
        const uint32_t pm = __ballot_sync(0xffffffffu, (d & OP_FLAG_P) != 0);
        const uint32_t zm = __ballot_sync(0xffffffffu, d == 0);
        const int fp = pm ? __ffs(pm) - 1 : 31;  // nearest inclusive prefix (or the window)
        const uint32_t need = fp == 31 ? 0xffffffffu : ((2u << fp) - 1u);
        if (zm & need) {  // a tile in the window is still drawing
          __nanosleep(SMX_LOOKBACK_SLEEP_NS);
          continue;
        }
        uint64_t v = lane <= fp ? (d & OP_VAL) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        base += v;
        if (pm) break;
        j -= 32;
      }
      if (lane == 0) vd[t] = OP_FLAG_P | (base + n_acc);
    }
    if (lane == 0 && t == n_tiles - 1) *total_out = base + n_acc;
    __syncwarp();
    if (base >= n_out || n_acc == 0) continue;
    if (cursor_out && base + n_acc >= n_out) *cursor_out = nth_accept_cursor(r, lo, hi, (uint32_t)(n_out - 1 - base));
    // coalesced hand-off in batches of 256 (8 per lane, stride 32)
    for (uint32_t h0 = 0; h0 < n_acc; h0 += 256) {
      const uint64_t j0 = base + h0;
      if (j0 >= n_out) break;
      uint32_t vv[8], kk[8];
      uint32_t okm = 0xffu;
      if (h0 + 256 <= n_acc && j0 + 256 <= n_out) {
#pragma unroll
        for (int u = 0; u < 8; ++u) vv[u] = sv[h0 + lane + u * 32];
        sink.template batch<true>(j0 + lane, 32, vv, okm, kk);
      } else {
        okm = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t q = h0 + lane + u * 32;
          const bool ok = q < n_acc && base + q < n_out;
          vv[u] = ok ? sv[q] : 0u;
          okm |= (ok ? 1u : 0u) << u;
        }
        sink.template batch<false>(j0 + lane, 32, vv, okm, kk);
      }
      if (MARK) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (!((okm >> u) & 1u)) continue;
          if (MARK == 1 && !(kk[u] & SMX_TMP_KEY)) {
            saw_local = true;
            continue;
          }
          const uint32_t bit = mark_bit<MARK>(mk, kk[u], vv[u]);
          if (bit == 0xffffffffu) continue;
          const uint32_t m = 1u << (bit & 31);
          uint32_t* w = mk.in_smem ? &smark[bit >> 5] : &mk.bits[bit >> 5];
          if (!(*(volatile uint32_t*)w & m)) atomicOr(w, m);
        }
      }
    }
    __syncwarp();
  }
  if (MARK == 1 && __any_sync(0xffffffffu, saw_local) && lane == 0 && mk.local_bit != 0xffffffffu) {
    const uint32_t b = mk.local_bit;
    atomicOr(mk.in_smem ? &smark[b >> 5] : &mk.bits[b >> 5], 1u << (b & 31));
  }
  if (MARK && mk.in_smem) {
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < mk.nwords; w += blockDim.x) {
      const uint32_t x = smark[w];
      if (x & ~__ldcg(&mk.bits[w])) atomicOr(&mk.bits[w], x);
    }
  }
}

static __global__ void draw_window_check_kernel(const uint64_t* total, uint64_t n_out, int* err) {
  if (*total < n_out) atomicExch(err, 1);
}

// A one-value range (ex == 1) consumes no draws: every value is 0.
template <class Sink>
__global__ void draw_const_kernel(uint64_t n_out, Sink sink) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n_out) sink(j, 0u);
}

}  // namespace smx
