// Construction kernels: connection-rule generation into the pending record
// buffers, remote-source bitmaps and image assignment, the temporary-key LUT,
// and the preparation-time compactions (R/L, S, H/I) and routing tables
// (T/P, G/Q).
//
// Reference mapping (sm/construction.py):
//   _realize_pairs / _draw_source_positions (391-432)  -> gen_draw / gen_pairs
//   used_flags / extract_used (454-470)                -> mark_values
//   lookup_or_create_images + RemoteSourceMap.insert   -> assign_images
//     (473-486, 227-236): new images get ids M, M+1, ... in ascending order of
//     the new source values, per (group, source rank), source ranks ascending
//   remap_connection_sources (489-495)                 -> LUT resolved at sort
//   mirror_merge / roster update (295-306, 620-636)    -> bits_or
//   prepare: rosters, image_lookups, routes (710-807)  -> bits_compact,
//     gather_lookup, build_routes
//
// Remote-source maps are stored densely per (group, source rank): img_of[v]
// (int32, -1 = no image) over the source rank's node values plus a presence
// bitmap; the sorted (R, L) pair of the reference is the compaction of that
// bitmap.  Lookups are O(1) gathers instead of searchsorted.
#include <algorithm>
#include <cstdlib>
#include "draw_host.cuh"

using namespace smx;

namespace {

constexpr int T256 = 256;

inline unsigned nblk(uint64_t n, int t = T256) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t b) {
  const uint32_t m = 1u << (b & 31);
  uint32_t* w = bits + (b >> 5);
  if (!(__ldcg(w) & m)) atomicOr(w, m);
}

// --- key / payload tables ----------------------------------------------------

__global__ void pay_table_kernel(const int64_t* targets, uint64_t n, const int32_t* node2row,
                                 uint64_t n_nodes, uint32_t cls, uint32_t* pay, int* bad) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t t = targets[i];
  int32_t row = (t >= 0 && (uint64_t)t < n_nodes) ? node2row[t] : -1;
  if (row < 0 || row > (int32_t)SMX_ROW_MASK) { atomicExch(bad, 3); row = 0; }
  pay[i] = (uint32_t)row | (cls << SMX_ROW_BITS);
}

__global__ void key_table_kernel(const int64_t* sources, uint64_t n, uint32_t tmp_base, int tmp,
                                 uint32_t* key) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = tmp ? (SMX_TMP_KEY | (tmp_base + (uint32_t)i)) : (uint32_t)sources[i];
}

// Distributed fixed in-degree: flat population index f -> pending key and the
// bit (global value key gv = vbase[rank] + node) to mark in the call's
// used-value bitmap.  Local sources (rank == tgt_rank) get their node as the
// key directly; they are marked too (their presence bumps the local counter).
__global__ void dist_tables_kernel(const int32_t* src_rank, const int64_t* src_node, uint64_t total,
                                   const uint32_t* vbase, int tgt_rank, uint32_t lut_base,
                                   uint32_t* key, uint32_t* gv_out) {
  const uint64_t f = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= total) return;
  const int r = src_rank[f];
  const uint32_t node = (uint32_t)src_node[f];
  const uint32_t gv = vbase[r] + node;
  key[f] = (r == tgt_rank) ? node : (SMX_TMP_KEY | (lut_base + gv));
  gv_out[f] = gv;
}

// --- generation sinks ----------------------------------------------------------

enum { K_NONE = 0, K_FROM_VALUE = 1, K_FROM_J = 2, K_PIECES = 3 };

// Piecewise-affine key table: key(v) = v + delta[s] for start[s] <= v <
// start[s+1].  A source population made of one contiguous node range per
// rank (every reference model) is one piece per source rank, so the draw
// writes keys without gathering from a table (the gather from an L2-resident
// table was the generation kernel's longest dependency).
constexpr int MAX_KEY_PIECES = 8;
struct KeyPieces {
  uint32_t n;
  uint32_t start[MAX_KEY_PIECES];
  uint32_t delta[MAX_KEY_PIECES];
  __device__ __forceinline__ uint32_t key(uint32_t v) const {
    uint32_t off = delta[0];
    if (n > 1) {
#pragma unroll
      for (int s = 1; s < MAX_KEY_PIECES; ++s)
        if (s < (int)n && v >= start[s]) off = delta[s];
    }
    return v + off;
  }
};
enum { P_NONE = 0, P_FROM_VALUE = 1, P_FROM_J = 2 };

template <int KM, int PM>
struct GenSink {
  static constexpr bool kMark = true;
  KeyPieces kp;
  const uint32_t* key_tab;
  const uint32_t* pay_tab;
  uint32_t kdiv;
  FastDiv kd;  // j / kdiv for call-local record indices j < 2^32
  uint32_t* keys;        // pre-offset to the call's first record
  uint32_t* vals;
  __device__ __forceinline__ void operator()(uint64_t j, uint32_t v) const {
    if (KM == K_FROM_VALUE) {
      if (keys && key_tab) keys[j] = __ldg(key_tab + v);
    } else if (KM == K_PIECES) {
      if (keys) keys[j] = kp.key(v);
    } else if (KM == K_FROM_J) {
      keys[j] = key_tab[j / kdiv];
    }
    if (PM == P_FROM_J) vals[j] = pay_tab[j / kdiv];
    else if (PM == P_FROM_VALUE) vals[j] = pay_tab[v];
  }
  // 8 items at j0 + u*stride: all gathers issued before any store
  template <bool ALL>
  __device__ __forceinline__ void batch(uint64_t j0, uint32_t stride, const uint32_t* v, uint32_t okm,
                                        uint32_t* kk) const {
    uint32_t pp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t j = (uint32_t)j0 + u * stride;  // call-local index < 2^32
      const bool ok = ALL || ((okm >> u) & 1u);
      kk[u] = 0;
      pp[u] = 0;
      if (ok) {
        if (KM == K_FROM_VALUE && key_tab) kk[u] = __ldg(key_tab + v[u]);
        else if (KM == K_PIECES) kk[u] = kp.key(v[u]);
        else if (KM == K_FROM_J && key_tab) kk[u] = __ldg(key_tab + kd.div(j));
        if (PM == P_FROM_J) pp[u] = __ldg(pay_tab + kd.div(j));
        else if (PM == P_FROM_VALUE) pp[u] = __ldg(pay_tab + v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!ALL && !((okm >> u) & 1u)) continue;
      const uint64_t j = j0 + (uint64_t)u * stride;
      if (KM != K_NONE && keys) keys[j] = kk[u];
      if (PM != P_NONE) vals[j] = pp[u];
    }
  }
};

__global__ void mark_one_kernel(uint32_t* bits, const uint32_t* tab) {
  const uint32_t b = tab ? tab[0] : 0u;
  if (b != 0xffffffffu) atomicOr(&bits[b >> 5], 1u << (b & 31));
}

// uniform_int delays of a wide call: meta[j] = (lo + value) | port << 24
struct MetaSink {
  uint32_t lo;
  uint32_t port_bits;
  uint32_t* meta;
  __device__ __forceinline__ void operator()(uint64_t j, uint32_t v) const { meta[j] = (lo + v) | port_bits; }
  template <bool ALL>
  __device__ __forceinline__ void batch(uint64_t j0, uint32_t stride, const uint32_t* v, uint32_t ok,
                                        uint32_t* keys) const {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      keys[u] = 0;
      if ((ok >> u) & 1u) meta[j0 + (uint64_t)u * stride] = (lo + v[u]) | port_bits;
    }
  }
};

// --- autapse redraw loop (sm/construction.py:524-529) ------------------------
// flag[i] = record idx[i] is a self-connection (source node's row == target row)
__global__ void autapse_flags_kernel(const uint32_t* idx, uint32_t m, const uint32_t* keys, const uint32_t* rows,
                                     const int32_t* node2row, uint64_t n_nodes, uint32_t* flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t j = idx ? idx[i] : i;
  const uint32_t k = keys[j];
  const int32_t r = (uint64_t)k < n_nodes ? node2row[k] : -1;
  flag[i] = (r >= 0 && (uint32_t)r == (rows[j] & SMX_ROW_MASK)) ? 1u : 0u;
}

__global__ void autapse_compact_kernel(const uint32_t* idx, uint32_t m, const uint32_t* flag, const int64_t* excl,
                                       uint32_t* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m && flag[i]) out[excl[i]] = idx ? idx[i] : i;
}

__global__ void autapse_apply_kernel(const uint32_t* idx, uint32_t m, const int64_t* draws, const uint32_t* key_tab,
                                     uint32_t* keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) keys[idx[i]] = key_tab[draws[i]];
}

struct RawI64Sink {
  int64_t* out;
  __device__ __forceinline__ void operator()(uint64_t j, uint32_t v) const { out[j] = (int64_t)v; }
  template <bool ALL>
  __device__ __forceinline__ void batch(uint64_t j0, uint32_t stride, const uint32_t* v, uint32_t ok,
                                        uint32_t* keys) const {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      keys[u] = 0;
      if ((ok >> u) & 1u) out[j0 + (uint64_t)u * stride] = (int64_t)v[u];
    }
  }
};

// Deterministic-use rules: one_to_one / assigned (mode 0: record i = (i, i)),
// all_to_all (mode 1: record r = (r % n_src, r / n_src)).
__global__ void pairs_kernel(int mode, uint64_t n, uint64_t n_src, const uint32_t* key_tab,
                             const uint32_t* pay_tab, uint32_t* keys, uint32_t* vals) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint64_t s = r, t = r;
  if (mode == 1) { s = r % n_src; t = r / n_src; }
  keys[r] = key_tab[s];
  vals[r] = pay_tab[t];
}

// --- bitmaps and images ---------------------------------------------------------

// vbits[sources[p]] = 1 for every position p whose bit is set in pos_bits
// (pos_bits == null: every position).
__global__ void mark_values_kernel(const uint32_t* pos_bits, const int64_t* sources, uint64_t n,
                                   uint32_t* vbits) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (pos_bits && !((pos_bits[p >> 5] >> (p & 31)) & 1)) return;
  set_bit(vbits, (uint32_t)sources[p]);
}

struct Segment {          // one (group, source rank) map inside a call
  uint64_t word0;         // first word of the segment in the concatenated bitmap
  uint64_t nwords;
  uint32_t* present;      // the map's presence bitmap (nwords words)
  int32_t* img_of;        // the map's dense value -> image array
};

__device__ __forceinline__ int find_seg(const Segment* segs, int ns, uint64_t w) {
  int lo = 0, hi = ns - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].word0 <= w) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void new_counts_kernel(const uint32_t* vbits, uint64_t nwords, const Segment* segs, int ns,
                                  uint32_t* cnt) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  const int s = find_seg(segs, ns, w);
  const uint64_t lw = w - segs[s].word0;
  if (!segs[s].img_of || lw >= segs[s].nwords) { cnt[w] = 0; return; }
  cnt[w] = __popc(vbits[w] & ~segs[s].present[lw]);
}

__global__ void assign_kernel(const uint32_t* vbits, uint64_t nwords, const Segment* segs, int ns,
                              const int64_t* excl, int64_t m0) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  const int s = find_seg(segs, ns, w);
  const uint64_t lw = w - segs[s].word0;
  if (!segs[s].img_of || lw >= segs[s].nwords) return;
  uint32_t nb = vbits[w] & ~segs[s].present[lw];
  if (!nb) return;
  int64_t id = m0 + excl[w];
  segs[s].present[lw] |= nb;
  while (nb) {
    const int b = __ffs(nb) - 1;
    nb &= nb - 1;
    segs[s].img_of[lw * 32 + b] = (int32_t)(id++);
  }
}

__global__ void gather_lut_kernel(const int64_t* sources, uint64_t n, const int32_t* img_of,
                                  uint32_t* lut) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  lut[p] = (uint32_t)img_of[sources[p]];
}

__global__ void bits_or_kernel(uint32_t* dst, const uint32_t* src, uint64_t nwords) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nwords) {
    const uint32_t x = src[w];
    if (x) dst[w] |= x;
  }
}

__global__ void popc_kernel(const uint32_t* bits, uint64_t nwords, uint32_t* cnt) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nwords) cnt[w] = __popc(bits[w]);
}

// out[excl[w] + k] = value of the k-th set bit of word w (ascending).
__global__ void compact_kernel(const uint32_t* bits, uint64_t nwords, const int64_t* excl, int64_t* out,
                               const int32_t* img_of, int64_t* img_out) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  uint32_t x = bits[w];
  int64_t o = excl[w];
  while (x) {
    const int b = __ffs(x) - 1;
    x &= x - 1;
    const int64_t v = (int64_t)(w * 32 + b);
    out[o] = v;
    if (img_out) img_out[o] = img_of ? (int64_t)img_of[v] : -1;
    ++o;
  }
}

// Routing tables of one source rank (T/P or G/Q).  For node s, every table
// t (destination rank or group, ascending) whose bitmap holds s contributes
// (dest[t], rank of s in that bitmap).  Tables are given as bitmaps plus
// per-word exclusive prefix counts.
struct RouteTable {
  const uint32_t* bits;
  const int64_t* excl;
  uint64_t nwords;
  int32_t dest;
};

__global__ void route_count_kernel(const RouteTable* tabs, int nt, uint64_t n_nodes, uint32_t* cnt) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_nodes) return;
  uint32_t c = 0;
  for (int t = 0; t < nt; ++t) {
    const uint64_t w = s >> 5;
    if (w < tabs[t].nwords && ((tabs[t].bits[w] >> (s & 31)) & 1)) ++c;
  }
  cnt[s] = c;
}

__global__ void route_fill_kernel(const RouteTable* tabs, int nt, uint64_t n_nodes, const int64_t* first,
                                  int32_t* dest, uint32_t* pos) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_nodes) return;
  int64_t o = first[s];
  for (int t = 0; t < nt; ++t) {
    const uint64_t w = s >> 5;
    if (w >= tabs[t].nwords) continue;
    const uint32_t x = tabs[t].bits[w];
    if ((x >> (s & 31)) & 1) {
      dest[o] = tabs[t].dest;
      pos[o] = (uint32_t)(tabs[t].excl[w] + __popc(x & ((1u << (s & 31)) - 1)));
      ++o;
    }
  }
}

// Wide-mode (per-record weight/delay) helpers.
__global__ void fill_wide_const_kernel(double* w, uint32_t* meta, uint64_t n, double wv, uint32_t mv) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { w[i] = wv; meta[i] = mv; }
}

__global__ void promote_wide_kernel(const uint32_t* vals, uint64_t n, const double* cls_w,
                                    const uint32_t* cls_meta, uint32_t* rows, double* w, uint32_t* meta) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t v = vals[i];
  const uint32_t c = v >> SMX_ROW_BITS;
  rows[i] = v & SMX_ROW_MASK;
  w[i] = cls_w[c];
  meta[i] = cls_meta[c];
}

// Wide records packed into 16-byte structs, so the permutation's random
// reads touch one 32-byte sector per record instead of three.
struct WideRec {
  uint32_t row, meta;
  double w;
};

__global__ void pack_wide_kernel(uint64_t n, const uint32_t* rows_in, const double* w_in, const uint32_t* meta_in,
                                 WideRec* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  WideRec r;
  r.row = rows_in[i];
  r.meta = meta_in[i];
  r.w = w_in[i];
  out[i] = r;
}

__global__ void gather_packed_kernel(const uint32_t* idx, uint64_t n, const WideRec* in, uint32_t* rows, double* w,
                                     uint32_t* meta) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const WideRec r = in[idx[i]];
  rows[i] = r.row;
  w[i] = r.w;
  meta[i] = r.meta;
}

__global__ void gather_wide_kernel(const uint32_t* idx, uint64_t n, const uint32_t* rows_in,
                                   const double* w_in, const uint32_t* meta_in, uint32_t* rows,
                                   double* w, uint32_t* meta) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = idx[i];
  rows[i] = rows_in[j];
  w[i] = w_in[j];
  meta[i] = meta_in[j];
}

__global__ void max_meta_kernel(const uint32_t* meta, uint64_t n, uint32_t* out3) {
  uint32_t md = 0, mp = 0, mn = 0xffffffffu;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t m = meta[i];
    md = max(md, m & 0xffffffu);
    mn = min(mn, m & 0xffffffu);
    mp = max(mp, m >> 24);
  }
  for (int o = 16; o; o >>= 1) {
    md = max(md, __shfl_xor_sync(0xffffffffu, md, o));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mp = max(mp, __shfl_xor_sync(0xffffffffu, mp, o));
  }
  if ((threadIdx.x & 31) == 0) { atomicMax(out3, md); atomicMax(out3 + 1, mp); atomicMin(out3 + 2, mn); }
}

}  // namespace

extern "C" int smx_counts_to_offsets(const uint32_t* counts, uint64_t n, int64_t* first_index, void* stream);

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" int smx_pay_table(const int64_t* targets, uint64_t n, const int32_t* node2row, uint64_t n_nodes,
                             uint32_t cls, uint32_t* pay_tab, void* stream) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  // the engine checks on the host that targets are real neurons; a bad row
  // here is an internal error, reported through the device error word
  // (no synchronisation: a persistent pass-A kernel may hold every SM)
  int* bad = smx_device_error_word();
  if (!bad) {
    smx_set_error("smx_pay_table: no device error word");
    return -3;
  }
  smx_count_launch(); pay_table_kernel<<<nblk(n), T256, 0, st>>>(targets, n, node2row, n_nodes, cls, pay_tab, bad);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_key_table(const int64_t* sources, uint64_t n, uint32_t tmp_base, int tmp, uint32_t* key_tab,
                             void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); key_table_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(sources, n, tmp_base, tmp, key_tab);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_dist_tables(const int32_t* src_rank, const int64_t* src_node, uint64_t total,
                               const uint32_t* vbase, int tgt_rank, uint32_t lut_base, uint32_t* key_tab,
                               uint32_t* gv_tab, void* stream) {
  if (total == 0) return 0;
  smx_count_launch(); dist_tables_kernel<<<nblk(total), T256, 0, (cudaStream_t)stream>>>(src_rank, src_node, total, vbase, tgt_rank,
                                                                       lut_base, key_tab, gv_tab);
  SMX_LAUNCH_CHECK();
  return 0;
}

// One numpy integers(0, ex, size=n) draw on stream (k0,k1) from u32 cursor u0,
// routed into the pending record buffers by the rule's sink.
template <int KM, int PM>
static int gen_draw(uint64_t k0, uint64_t k1, uint64_t u0, uint64_t ex, uint64_t n, const uint32_t* key_tab,
                    const uint32_t* pay_tab, uint32_t kdiv, uint32_t* keys, uint32_t* vals, const DrawMark& mk0,
                    uint64_t* cursor_out, cudaStream_t st) {
  GenSink<KM, PM> s;
  s.kp.n = 0;
  if (KM == K_PIECES) {  // key_tab is a host array {n, start[n], delta[n]}
    const uint32_t np = key_tab ? key_tab[0] : 0;
    if (np < 1 || np > MAX_KEY_PIECES) {
      smx_set_error("smx_gen_draw: %u key pieces (1..%d supported)", np, MAX_KEY_PIECES);
      return -1;
    }
    s.kp.n = np;
    for (uint32_t i = 0; i < MAX_KEY_PIECES; ++i) {
      s.kp.start[i] = i < np ? key_tab[1 + i] : 0xffffffffu;
      s.kp.delta[i] = i < np ? key_tab[1 + np + i] : 0u;
    }
    key_tab = nullptr;
  }
  s.key_tab = key_tab;
  s.pay_tab = pay_tab;
  s.kdiv = kdiv ? kdiv : 1;
  s.kd = FastDiv::make(s.kdiv);
  s.keys = keys;
  s.vals = vals;
  DrawResult res;
  if (ex == 1) {  // numpy: a one-value range consumes nothing; every draw is 0
    if (n) {
      smx_count_launch(); draw_const_kernel<GenSink<KM, PM>><<<nblk(n), T256, 0, st>>>(n, s);
      if (mk0.bits) { smx_count_launch(); mark_one_kernel<<<1, 1, 0, st>>>(mk0.bits, mk0.tab); }
      SMX_LAUNCH_CHECK();
    }
    if (cursor_out) *cursor_out = u0;
    const uint64_t* u0_dev = nullptr;   // a chained call's cursor passes through
    uint64_t* cursor_dev = nullptr;
    smx_take_draw_chain(&u0_dev, &cursor_dev);
    return smx_chain_passthrough(u0_dev, u0, cursor_dev, st);
  }
  // no cursor wanted: the asynchronous path (no host synchronisation)
  res.cursor = u0;
  const int rc = run_draw(Key{k0, k1}, u0, ex, n, s, st, cursor_out ? &res : nullptr, mk0);
  if (cursor_out) *cursor_out = res.cursor;
  return rc;
}

extern "C" int smx_gen_draw(uint64_t k0, uint64_t k1, uint64_t u0, uint64_t ex, uint64_t n, int key_mode,
                            int pay_mode, const uint32_t* key_tab, const uint32_t* pay_tab, uint32_t kdiv,
                            uint32_t* keys, uint32_t* vals, uint32_t* used_bits, const uint32_t* used_tab,
                            uint32_t used_bits_words, int mark_from_key, uint32_t tmp_base, uint32_t local_bit,
                            uint64_t* cursor_out, void* stream) {
  DrawChainScope chain_scope;
  if (n >= (1ULL << 32)) {
    smx_set_error("smx_gen_draw: %llu records in one call exceed 2^32", (unsigned long long)n);
    return -1;
  }
  if (key_mode < K_NONE || key_mode > K_PIECES || pay_mode < P_NONE || pay_mode > P_FROM_J) {
    smx_set_error("smx_gen_draw: bad key/payload mode %d/%d", key_mode, pay_mode);
    return -1;
  }
  // used-value marking (flagged / remote sources): bitmap size from the table
  // range -- the caller sizes used_bits to cover every bit it can receive
  const DrawMark mk{used_bits, used_tab, used_bits_words, 0, mark_from_key, tmp_base, local_bit};
  cudaStream_t st = (cudaStream_t)stream;
#define SMX_GEN(KM, PM) \
  if (key_mode == KM && pay_mode == PM) \
    return gen_draw<KM, PM>(k0, k1, u0, ex, n, key_tab, pay_tab, kdiv, keys, vals, mk, cursor_out, st);
  SMX_GEN(K_NONE, P_NONE) SMX_GEN(K_NONE, P_FROM_VALUE) SMX_GEN(K_NONE, P_FROM_J)
  SMX_GEN(K_FROM_VALUE, P_NONE) SMX_GEN(K_FROM_VALUE, P_FROM_VALUE) SMX_GEN(K_FROM_VALUE, P_FROM_J)
  SMX_GEN(K_FROM_J, P_NONE) SMX_GEN(K_FROM_J, P_FROM_VALUE) SMX_GEN(K_FROM_J, P_FROM_J)
  SMX_GEN(K_PIECES, P_NONE) SMX_GEN(K_PIECES, P_FROM_VALUE) SMX_GEN(K_PIECES, P_FROM_J)
#undef SMX_GEN
  smx_set_error("smx_gen_draw: unsupported key/payload mode %d/%d", key_mode, pay_mode);
  return -1;
}

extern "C" int smx_gen_pairs(int mode, uint64_t n, uint64_t n_src, const uint32_t* key_tab,
                             const uint32_t* pay_tab, uint32_t* keys, uint32_t* vals, void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); pairs_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(mode, n, n_src, key_tab, pay_tab, keys, vals);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_mark_values(const uint32_t* pos_bits, const int64_t* sources, uint64_t n, uint32_t* vbits,
                               void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); mark_values_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(pos_bits, sources, n, vbits);
  SMX_LAUNCH_CHECK();
  return 0;
}

// Assign image ids m0, m0+1, ... to the values set in vbits (a concatenation
// of segments, one per (group, source rank) map, in ascending source-rank
// order) that are not yet present in their map.  Returns the number of new
// images in *n_new (host).
extern "C" int smx_assign_images(const uint32_t* vbits, uint64_t nwords, const void* segs_host, int ns,
                                 int64_t m0, int64_t* n_new, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *n_new = 0;
  if (nwords == 0 || ns == 0) return 0;
  Segment* segs = nullptr;
  uint32_t* cnt = nullptr;
  int64_t* excl = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&segs, sizeof(Segment) * ns, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&cnt, sizeof(uint32_t) * nwords, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&excl, sizeof(int64_t) * (nwords + 1), st));
  if (smx_h2d_async(segs, segs_host, sizeof(Segment) * ns, st)) return -3;
  smx_count_launch(); new_counts_kernel<<<nblk(nwords), T256, 0, st>>>(vbits, nwords, segs, ns, cnt);
  SMX_LAUNCH_CHECK();
  if (int rc = smx_counts_to_offsets(cnt, nwords, excl, st)) return rc;
  smx_count_launch(); assign_kernel<<<nblk(nwords), T256, 0, st>>>(vbits, nwords, segs, ns, excl, m0);
  SMX_LAUNCH_CHECK();
  SMX_CUDA_CHECK(cudaMemcpyAsync(n_new, excl + nwords, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SMX_CUDA_CHECK(cudaStreamSynchronize(st));
  cudaFreeAsync(segs, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(excl, st);
  return 0;
}

extern "C" int smx_gather_lut(const int64_t* sources, uint64_t n, const int32_t* img_of, uint32_t* lut,
                              void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); gather_lut_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(sources, n, img_of, lut);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_bits_or(uint32_t* dst, const uint32_t* src, uint64_t nwords, void* stream) {
  if (nwords == 0) return 0;
  smx_count_launch(); bits_or_kernel<<<nblk(nwords), T256, 0, (cudaStream_t)stream>>>(dst, src, nwords);
  SMX_LAUNCH_CHECK();
  return 0;
}

// dst |= src[0] | src[1] | ... (up to 64 sources, host array of device
// pointers): the source-rank segments of several targets' used-value bitmaps
// merged into one mirror / roster in one launch.
constexpr int MAX_OR_SRCS = 64;
struct OrSrcs {
  const uint32_t* p[MAX_OR_SRCS];
  int n;
};
__global__ void bits_or_many_kernel(uint32_t* dst, OrSrcs S, uint64_t nwords) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  uint32_t x = 0;
  for (int i = 0; i < S.n; ++i) x |= S.p[i][w];
  if (x) dst[w] |= x;
}

extern "C" int smx_bits_or_many(uint32_t* dst, const uint32_t* const* srcs_host, int n_srcs, uint64_t nwords,
                                void* stream) {
  if (nwords == 0 || n_srcs == 0) return 0;
  for (int a = 0; a < n_srcs; a += MAX_OR_SRCS) {
    OrSrcs S{};
    S.n = std::min(MAX_OR_SRCS, n_srcs - a);
    for (int i = 0; i < S.n; ++i) S.p[i] = srcs_host[a + i];
    smx_count_launch(); bits_or_many_kernel<<<nblk(nwords), T256, 0, (cudaStream_t)stream>>>(dst, S, nwords);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}

// Per-word exclusive popcount prefix of a bitmap (nwords + 1 entries).
extern "C" int smx_bits_prefix(const uint32_t* bits, uint64_t nwords, int64_t* excl, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* cnt = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&cnt, sizeof(uint32_t) * (nwords ? nwords : 1), st));
  if (nwords) {
    smx_count_launch(); popc_kernel<<<nblk(nwords), T256, 0, st>>>(bits, nwords, cnt);
    SMX_LAUNCH_CHECK();
  }
  if (int rc = smx_counts_to_offsets(cnt, nwords, excl, st)) return rc;
  cudaFreeAsync(cnt, st);
  return 0;
}

// Ascending values of the set bits (needs the prefix from smx_bits_prefix);
// optionally the image of each value (img_of null -> -1).
extern "C" int smx_bits_compact(const uint32_t* bits, uint64_t nwords, const int64_t* excl, int64_t* out,
                                const int32_t* img_of, int64_t* img_out, void* stream) {
  if (nwords == 0) return 0;
  smx_count_launch(); compact_kernel<<<nblk(nwords), T256, 0, (cudaStream_t)stream>>>(bits, nwords, excl, out, img_of, img_out);
  SMX_LAUNCH_CHECK();
  return 0;
}

// Build one source rank's routing CSR over nodes [0, n_nodes): first[n+1],
// dest[], pos[] (capacity from a first call with dest == null: returns the
// total entries in *n_entries).
extern "C" int smx_build_routes(const void* tabs_host, int nt, uint64_t n_nodes, uint32_t* cnt_scratch,
                                int64_t* first, int32_t* dest, uint32_t* pos, int64_t* n_entries, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *n_entries = 0;
  RouteTable* tabs = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&tabs, sizeof(RouteTable) * (nt ? nt : 1), st));
  if (nt && smx_h2d_async(tabs, tabs_host, sizeof(RouteTable) * nt, st)) return -3;
  if (n_nodes) {
    smx_count_launch(); route_count_kernel<<<nblk(n_nodes), T256, 0, st>>>(tabs, nt, n_nodes, cnt_scratch);
    SMX_LAUNCH_CHECK();
  }
  if (int rc = smx_counts_to_offsets(cnt_scratch, n_nodes, first, st)) return rc;
  SMX_CUDA_CHECK(cudaMemcpyAsync(n_entries, first + n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SMX_CUDA_CHECK(cudaStreamSynchronize(st));
  if (dest && n_nodes) {
    smx_count_launch(); route_fill_kernel<<<nblk(n_nodes), T256, 0, st>>>(tabs, nt, n_nodes, first, dest, pos);
    SMX_LAUNCH_CHECK();
  }
  cudaFreeAsync(tabs, st);
  return 0;
}

extern "C" int smx_fill_wide_const(double* w, uint32_t* meta, uint64_t n, double wv, uint32_t mv, void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); fill_wide_const_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(w, meta, n, wv, mv);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_promote_wide(const uint32_t* vals, uint64_t n, const double* cls_w, const uint32_t* cls_meta,
                                uint32_t* rows, double* w, uint32_t* meta, void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); promote_wide_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(vals, n, cls_w, cls_meta, rows, w, meta);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_gather_wide(const uint32_t* idx, uint64_t n, const uint32_t* rows_in, const double* w_in,
                               const uint32_t* meta_in, uint32_t* rows, double* w, uint32_t* meta, void* stream) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  WideRec* packed = nullptr;
  if (cudaMallocAsync((void**)&packed, sizeof(WideRec) * n, st) != cudaSuccess) {
    cudaGetLastError();   // no room for the packed copy: three separate gathers
    smx_count_launch(); gather_wide_kernel<<<nblk(n), T256, 0, st>>>(idx, n, rows_in, w_in, meta_in, rows, w, meta);
    SMX_LAUNCH_CHECK();
    return 0;
  }
  smx_count_launch(); pack_wide_kernel<<<nblk(n), T256, 0, st>>>(n, rows_in, w_in, meta_in, packed);
  smx_count_launch(); gather_packed_kernel<<<nblk(n), T256, 0, st>>>(idx, n, packed, rows, w, meta);
  SMX_LAUNCH_CHECK();
  cudaFreeAsync(packed, st);
  return 0;
}

// out3 = {max delay, max port, min delay} of wide records (meta = delay | port << 24)
extern "C" int smx_max_meta(const uint32_t* meta, uint64_t n, uint32_t* out3, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  SMX_CUDA_CHECK(cudaMemsetAsync(out3, 0, 8, st));
  SMX_CUDA_CHECK(cudaMemsetAsync(out3 + 2, 0xff, 4, st));
  if (n == 0) return 0;
  smx_count_launch(); max_meta_kernel<<<148 * 4, T256, 0, st>>>(meta, n, out3);
  SMX_LAUNCH_CHECK();
  return 0;
}

// Delays of a wide call drawn as numpy integers(lo, lo+ex, size=n) from u32
// cursor u0 (sm/construction.py:168-169), stored as meta = delay | port << 24.
extern "C" int smx_delay_fill(uint64_t k0, uint64_t k1, uint64_t u0, uint32_t lo, uint64_t ex, uint64_t n,
                              uint32_t port, uint32_t* meta, uint64_t* cursor_out, void* stream) {
  DrawChainScope chain_scope;
  MetaSink s{lo, port << 24, meta};
  if (cursor_out) *cursor_out = u0;
  if (n == 0 || ex == 1) {   // (a chained call's cursor passes through)
    const uint64_t* u0_dev = nullptr;
    uint64_t* cursor_dev = nullptr;
    smx_take_draw_chain(&u0_dev, &cursor_dev);
    if (n) {
      smx_count_launch(); draw_const_kernel<MetaSink><<<nblk(n), T256, 0, (cudaStream_t)stream>>>(n, s);
      SMX_LAUNCH_CHECK();
    }
    return smx_chain_passthrough(u0_dev, u0, cursor_dev, (cudaStream_t)stream);
  }
  DrawResult res;   // no cursor_out: asynchronous (window checked on the device)
  const int rc = run_draw(Key{k0, k1}, u0, ex, n, s, (cudaStream_t)stream, cursor_out ? &res : nullptr);
  if (cursor_out) *cursor_out = res.cursor;
  return rc;
}

// allow_autapses=False for fixed_indegree / fixed_total local calls
// (sm/construction.py:524-529): while any record connects a node to itself,
// redraw those records' sources -- in ascending record order -- from the
// call's stream, continuing at u32 cursor u0.  keys/rows are the call's
// pending records (n of them); key_tab maps positions to source nodes.
extern "C" int smx_autapse_fix(uint64_t k0, uint64_t k1, uint64_t u0, uint64_t n_src, const uint32_t* key_tab,
                               uint32_t* keys, const uint32_t* rows, uint64_t n, const int32_t* node2row,
                               uint64_t n_nodes, uint64_t* cursor_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *cursor_out = u0;
  if (n == 0) return 0;
  uint32_t *flag = nullptr, *idx_a = nullptr, *idx_b = nullptr;
  int64_t *excl = nullptr, *draws = nullptr;
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&flag, sizeof(uint32_t) * n, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&excl, sizeof(int64_t) * (n + 1), st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&idx_a, sizeof(uint32_t) * n, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&idx_b, sizeof(uint32_t) * n, st));
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&draws, sizeof(int64_t) * n, st));
  // initial bad list over all records
  smx_count_launch(); autapse_flags_kernel<<<nblk(n), T256, 0, st>>>(nullptr, (uint32_t)n, keys, rows, node2row, n_nodes, flag);
  if (int rc = smx_counts_to_offsets(flag, n, excl, st)) return rc;
  smx_count_launch(); autapse_compact_kernel<<<nblk(n), T256, 0, st>>>(nullptr, (uint32_t)n, flag, excl, idx_a);
  SMX_LAUNCH_CHECK();
  int64_t m = 0;
  SMX_CUDA_CHECK(cudaMemcpyAsync(&m, excl + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SMX_CUDA_CHECK(cudaStreamSynchronize(st));
  uint64_t cur = u0;
  int rounds = 0;
  while (m > 0) {
    if (++rounds > 100000) { smx_set_error("autapse redraw did not terminate"); return -2; }
    if (n_src == 1) { smx_set_error("cannot avoid autapses with a single source"); return -1; }
    DrawResult res;
    if (int rc = run_draw(Key{k0, k1}, cur, n_src, (uint64_t)m, RawI64Sink{draws}, st, &res)) return rc;
    cur = res.cursor;
    smx_count_launch(); autapse_apply_kernel<<<nblk(m), T256, 0, st>>>(idx_a, (uint32_t)m, draws, key_tab, keys);
    smx_count_launch(); autapse_flags_kernel<<<nblk(m), T256, 0, st>>>(idx_a, (uint32_t)m, keys, rows, node2row, n_nodes, flag);
    if (int rc = smx_counts_to_offsets(flag, (uint64_t)m, excl, st)) return rc;
    smx_count_launch(); autapse_compact_kernel<<<nblk(m), T256, 0, st>>>(idx_a, (uint32_t)m, flag, excl, idx_b);
    SMX_LAUNCH_CHECK();
    SMX_CUDA_CHECK(cudaMemcpyAsync(&m, excl + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SMX_CUDA_CHECK(cudaStreamSynchronize(st));
    uint32_t* t = idx_a; idx_a = idx_b; idx_b = t;
  }
  *cursor_out = cur;
  cudaFreeAsync(flag, st);
  cudaFreeAsync(excl, st);
  cudaFreeAsync(idx_a, st);
  cudaFreeAsync(idx_b, st);
  cudaFreeAsync(draws, st);
  return 0;
}

// --- per-range record counts (modeled-byte accounting) ------------------------
// counts[s] += #{i : lo[s] <= keys[i] < hi[s]} for up to 16 disjoint ranges:
// the records of one distributed call per source rank (the reference appends
// one batch per source rank, sm/construction.py:689-703).
constexpr int MAX_COUNT_RANGES = 16;
struct CountRanges {
  uint32_t m;
  uint32_t lo[MAX_COUNT_RANGES], hi[MAX_COUNT_RANGES];
};

template <int M>
__global__ void __launch_bounds__(256) count_ranges_kernel(const uint32_t* keys, uint64_t n, CountRanges R,
                                                           unsigned long long* counts) {
  uint32_t c[M];
#pragma unroll
  for (int s = 0; s < M; ++s) c[s] = 0;
  const uint64_t n4 = n / 4;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4 + 1; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t kk[4];
    int m = 4;
    if (i < n4) {
      const uint4 q = k4[i];
      kk[0] = q.x; kk[1] = q.y; kk[2] = q.z; kk[3] = q.w;
    } else {
      m = (int)(n - 4 * n4);
#pragma unroll
      for (int j = 0; j < 4; ++j) kk[j] = j < m ? keys[4 * n4 + j] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= m) break;
#pragma unroll
      for (int s = 0; s < M; ++s) c[s] += (kk[j] - R.lo[s] < R.hi[s] - R.lo[s]) ? 1u : 0u;  // lo <= k < hi
    }
  }
#pragma unroll
  for (int s = 0; s < M; ++s) {
    uint32_t x = c[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(counts + s, (unsigned long long)x);
  }
}

template <int M>
static void launch_count_ranges(const uint32_t* keys, uint64_t n, const CountRanges& R, unsigned long long* counts,
                                cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<uint64_t>((n / 4 + 256) / 256, 148 * 8);
  smx_count_launch(); count_ranges_kernel<M><<<grid, 256, 0, st>>>(keys, n, R, counts);
}

// ranges_host = {m, lo[m], hi[m]}; counts (device, m u64) are accumulated.
extern "C" int smx_count_ranges(const uint32_t* keys, uint64_t n, const uint32_t* ranges_host,
                                unsigned long long* counts, void* stream) {
  CountRanges R{};
  R.m = ranges_host[0];
  if (R.m > (uint32_t)MAX_COUNT_RANGES) {
    smx_set_error("smx_count_ranges: %u ranges (at most %d)", R.m, MAX_COUNT_RANGES);
    return -1;
  }
  for (uint32_t s = 0; s < R.m; ++s) {
    R.lo[s] = ranges_host[1 + s];
    R.hi[s] = ranges_host[1 + R.m + s];
  }
  if (n == 0 || R.m == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (R.m) {  // pad to the next instantiated width (empty ranges count nothing)
    case 1: case 2: launch_count_ranges<2>(keys, n, R, counts, st); break;
    case 3: case 4: launch_count_ranges<4>(keys, n, R, counts, st); break;
    case 5: case 6: case 7: case 8: launch_count_ranges<8>(keys, n, R, counts, st); break;
    default: launch_count_ranges<16>(keys, n, R, counts, st); break;
  }
  SMX_LAUNCH_CHECK();
  return 0;
}

// --- choice without replacement (allow_multapses=False) ------------------------
// numpy 2.3.5 Generator.choice(n, size=k, replace=False), one row per target
// from one stream (sm/core.py:140-141, sm/construction.py:403-404, 680-683):
//   n > 10000 and k > n // 50: tail Fisher-Yates of arange(n), keep the last k
//   otherwise:                 Floyd's algorithm, then a Fisher-Yates shuffle
// every index draw is numpy's random_bounded_uint64 (Lemire on next_uint32,
// value in [0, rng], rng == 0 consumes nothing).  The rows form one chain
// through the stream (each row's length depends on its rejections): the
// chain of row starts is resolved warp-parallel (row_consumption), and the
// rows themselves are drawn concurrently, one per warp.
namespace {

struct U32Stream {  // next_uint32 with numpy's low-half-first buffering, from a u32 cursor
  smx::Key key;
  uint64_t pos;     // next u32 position
  uint64_t blk_w[4];
  uint64_t blk;
  __device__ void init(smx::Key k, uint64_t p) { key = k; pos = p; blk = 0; }
  __device__ uint32_t next32() {
    const uint64_t w = pos >> 1;
    const uint64_t b = (w >> 2) + 1;
    if (b != blk) { smx::philox4x64_10(b, key, blk_w); blk = b; }
    const uint64_t word = blk_w[w & 3];
    const uint32_t v = (pos & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
    ++pos;
    return v;
  }
  __device__ uint32_t bounded_incl(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t ex = rng + 1;
    uint64_t m = (uint64_t)next32() * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
      const uint32_t thr = (uint32_t)((0x100000000ULL - ex) % ex);
      while (left < thr) {
        m = (uint64_t)next32() * ex;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

constexpr uint32_t EMPTY32 = 0xFFFFFFFFu;

// One row of choice(n, k, replace=False) from u32 cursor `start`, serially on
// the calling thread, exactly as numpy walks it (Floyd's set sampling then a
// Fisher-Yates shuffle; the tail branch shuffles a virtual array).  `tab` is
// this row's private hash table.
__device__ void choice_row(smx::Key key, uint64_t start, uint32_t n, uint32_t k, bool tail, uint32_t* row,
                           uint32_t* tab, uint32_t tab_mask) {
  U32Stream s;
  s.init(key, start);
  if (tail) {
    // virtual array data[i] = i, swaps kept in an open-addressing map
    auto find = [&](uint32_t key_) -> uint32_t {
      uint32_t loc = (key_ * 2654435761u) & tab_mask;
      while (tab[loc] != EMPTY32 && tab[loc] != key_) loc = (loc + 1) & tab_mask;
      return loc;
    };
    auto get = [&](uint32_t idx) -> uint32_t {
      const uint32_t loc = find(idx);
      return tab[loc] == EMPTY32 ? idx : tab[tab_mask + 1 + loc];
    };
    auto put = [&](uint32_t idx, uint32_t val) {
      const uint32_t loc = find(idx);
      tab[loc] = idx;
      tab[tab_mask + 1 + loc] = val;
    };
    const uint32_t first = n - k > 1 ? n - k : 1;
    for (uint32_t i = n - 1; i >= first; --i) {
      const uint32_t j = s.bounded_incl(i);
      const uint32_t vi = get(i), vj = get(j);
      put(j, vi);
      put(i, vj);
      if (i == 0) break;
    }
    for (uint32_t q = 0; q < k; ++q) row[q] = get(n - k + q);
  } else {
    for (uint32_t j = n - k; j < n; ++j) {
      const uint32_t val = s.bounded_incl(j);
      uint32_t loc = val & tab_mask;
      while (tab[loc] != EMPTY32 && tab[loc] != val) loc = (loc + 1) & tab_mask;
      if (tab[loc] == EMPTY32) {
        tab[loc] = val;
        row[j - n + k] = val;
      } else {
        loc = j & tab_mask;
        while (tab[loc] != EMPTY32) loc = (loc + 1) & tab_mask;
        tab[loc] = j;
        row[j - n + k] = j;
      }
    }
    for (uint32_t i = k - 1; i >= 1 && k > 1; --i) {
      const uint32_t j = s.bounded_incl(i);
      const uint32_t t = row[j];
      row[j] = row[i];
      row[i] = t;
    }
  }
}

// The bounded range of stage t of a row (bounded_incl(rng) calls in order):
// Floyd stages rng = n - k + t (t < k), then shuffle stages rng = k - 1 - (t - k);
// tail stages rng = n - 1 - t.
struct RowStages {
  uint32_t n, k, m;
  bool tail;
  __device__ uint32_t rng(uint32_t t) const {
    if (tail) return n - 1 - t;
    return t < k ? n - k + t : k - 1 - (t - k);
  }
};

// u32 draws a row consumes from `start` (each stage: one draw plus one per
// Lemire rejection; a stage of range 0 draws nothing), found by the warp in
// windows of 256 stages: every lane checks 8 consecutive positions for a
// rejection under the no-rejection alignment; the first rejection moves the
// window to the stage that redraws.
__device__ uint64_t row_consumption(smx::Key key, uint64_t start, const RowStages& S, int lane) {
  uint64_t p = start;
  uint32_t t = 0;
  if (!S.tail && S.n == S.k && S.m > 0) t = 1;   // Floyd stage 0 has range 0: no draw
  while (t < S.m) {
    const uint32_t t0 = t + 8u * lane;
    uint64_t blk = ~0ull, w4[4];
    int hit = 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t ts = t0 + e;
      if (ts >= S.m || hit < 8) continue;
      const uint64_t q = p + 8ull * lane + e;
      const uint64_t w = q >> 1, b = (w >> 2) + 1;
      if (b != blk) { smx::philox4x64_10(b, key, w4); blk = b; }
      const uint32_t raw = (q & 1) ? (uint32_t)(w4[w & 3] >> 32) : (uint32_t)w4[w & 3];
      const uint32_t rng = S.rng(ts);
      if (rng == 0u || rng == 0xFFFFFFFFu) continue;   // (range 0 only at Floyd stage 0, skipped above)
      const uint32_t ex = rng + 1;
      const uint32_t left = (uint32_t)((uint64_t)raw * ex);
      if (left < ex && left < (uint32_t)((0x100000000ULL - ex) % ex)) hit = e;
    }
    const uint32_t any = __ballot_sync(0xffffffffu, hit < 8);
    if (!any) {
      const uint32_t adv = min(256u, S.m - t);
      t += adv;
      p += adv;
      continue;
    }
    const int l = __ffs(any) - 1;
    const int e = __shfl_sync(0xffffffffu, hit, l);
    // stage t + 8 l + e rejected its draw at position p + 8 l + e: it redraws at the next one
    t += 8u * l + e;
    p += 8ull * l + e + 1;
  }
  return p - start;
}

constexpr uint64_t CURSOR_UNSET = ~0ull;

// Rows in parallel: warps take rows by ticket.  Row r's start cursor is
// published by row r - 1's warp as soon as it knows its consumption.  A warp
// first speculates that rows r - D .. r - 1 consume the nominal m draws each
// (no rejection), starting from row r - D's start (published D hand-offs
// earlier), and computes its own consumption from there while the chain
// catches up; when the speculation holds, the chain advances by one flag
// hand-off per row.  Then lane 0 draws the row itself, beside every other
// warp's row.
constexpr uint64_t CHOICE_SPEC_DEPTH = 8;
// One warp per CTA.  With in_smem the row's hash table and the row itself
// live in shared memory (the serial draw is latency-bound on its probes and
// swaps) and the row is copied out at the end; otherwise both are global.
__global__ void __launch_bounds__(32) choice_rows_kernel(smx::Key key, uint32_t n, uint32_t k, uint64_t rows,
                                                         RowStages S, uint32_t* out, uint32_t* tab,
                                                         uint32_t tab_mask, uint64_t* starts, uint32_t* ticket,
                                                         int in_smem) {
  extern __shared__ uint32_t crs[];
  const int lane = threadIdx.x & 31;
  const uint64_t warp_id = blockIdx.x;
  const uint32_t tab_words = (tab_mask + 1) * (S.tail ? 2u : 1u);
  uint32_t* my_tab = in_smem ? crs : tab + warp_id * tab_words;
  uint32_t* srow = crs + tab_words;
  volatile uint64_t* vs = starts;
  for (;;) {
    uint64_t r = 0;
    if (lane == 0) r = atomicAdd(ticket, 1u);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (r >= rows) break;
    // speculate from the predecessor's start (published one row earlier)
    uint64_t spec = CURSOR_UNSET, c_spec = 0;
    if (r > 0) {
      const uint64_t b = r > CHOICE_SPEC_DEPTH ? r - CHOICE_SPEC_DEPTH : 0;
      uint64_t ps = CURSOR_UNSET;
      if (lane == 0) {
        while ((ps = vs[b]) == CURSOR_UNSET) __nanosleep(32);
      }
      ps = __shfl_sync(0xffffffffu, ps, 0);
      spec = ps + (r - b) * (uint64_t)S.m;
      c_spec = row_consumption(key, spec, S, lane);
    }
    uint64_t s0 = CURSOR_UNSET;
    if (lane == 0) {
      while ((s0 = vs[r]) == CURSOR_UNSET) __nanosleep(32);
    }
    s0 = __shfl_sync(0xffffffffu, s0, 0);
    const uint64_t c = s0 == spec ? c_spec : row_consumption(key, s0, S, lane);
    if (lane == 0) {
      __threadfence();
      vs[r + 1] = s0 + c;
    }
    for (uint32_t i = lane; i < tab_words; i += 32) my_tab[i] = i <= tab_mask ? EMPTY32 : 0u;
    __syncwarp();
    if (lane == 0) choice_row(key, s0, n, k, S.tail, in_smem ? srow : out + r * k, my_tab, tab_mask);
    __syncwarp();
    if (in_smem)
      for (uint32_t i = lane; i < k; i += 32) out[r * k + i] = srow[i];
  }
}

}  // namespace

// rows x k values (u32) of numpy choice(n, k, replace=False) drawn back to back
// from u32 cursor u0; *cursor_out_host = u32 cursor after the last row.
extern "C" int smx_choice_rows(uint64_t k0, uint64_t k1, uint64_t u0, uint64_t n, uint64_t k, uint64_t rows,
                               uint32_t* out, uint64_t* cursor_out_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (k > n) {
    smx_set_error("Cannot take a larger sample than population when replace is False");
    return -1;
  }
  if (n >= 0xFFFFFFFFULL) {
    smx_set_error("smx_choice_rows: population %llu exceeds 2^32 - 1", (unsigned long long)n);
    return -1;
  }
  *cursor_out_host = u0;
  if (rows == 0 || k == 0) return 0;
  const bool tail = n > 10000 && k > n / 50;
  // Floyd: set of k values (pow2 >= 1.2k, as numpy); tail: map of <= 2k touched indices
  uint64_t want = tail ? 4 * k : (uint64_t)(1.2 * (double)k) + 1;
  uint64_t cap = 1;
  while (cap < want) cap <<= 1;
  RowStages S;
  S.n = (uint32_t)n;
  S.k = (uint32_t)k;
  S.tail = tail;
  S.m = tail ? (uint32_t)(n - (n - k > 1 ? n - k : 1)) : (uint32_t)(k + (k > 1 ? k - 1 : 0));
  // one warp per CTA; the hash table and the row in SMEM when they fit
  // (<= 160 KB), otherwise global tables bounded to 256 MB in total
  const uint64_t tab_bytes = sizeof(uint32_t) * cap * (tail ? 2 : 1);
  const uint64_t smem = tab_bytes + sizeof(uint32_t) * k;
  const int in_smem = smem <= (160u << 10);
  uint64_t warps = std::min<uint64_t>(rows, 148ull * 16);
  if (!in_smem) warps = std::max<uint64_t>(1, std::min<uint64_t>(warps, (256ull << 20) / tab_bytes));
  const uint32_t blocks = (uint32_t)warps;
  uint32_t* tab = nullptr;
  uint64_t* starts = nullptr;
  if (in_smem) {
    SMX_CUDA_CHECK(cudaFuncSetAttribute(choice_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  } else {
    SMX_CUDA_CHECK(cudaMallocAsync((void**)&tab, tab_bytes * warps, st));
  }
  SMX_CUDA_CHECK(cudaMallocAsync((void**)&starts, sizeof(uint64_t) * (rows + 2), st));
  SMX_CUDA_CHECK(cudaMemsetAsync(starts, 0xff, sizeof(uint64_t) * (rows + 2), st));
  if (smx_h2d_async(starts, &u0, sizeof(uint64_t), st)) return -3;
  uint32_t* ticket = reinterpret_cast<uint32_t*>(starts + rows + 1);
  SMX_CUDA_CHECK(cudaMemsetAsync(ticket, 0, sizeof(uint32_t), st));
  smx_count_launch();
  choice_rows_kernel<<<blocks, 32, in_smem ? smem : 0, st>>>(smx::Key{k0, k1}, (uint32_t)n, (uint32_t)k, rows, S,
                                                              out, tab, (uint32_t)(cap - 1), starts, ticket,
                                                              in_smem);
  SMX_LAUNCH_CHECK();
  SMX_CUDA_CHECK(cudaMemcpyAsync(cursor_out_host, starts + rows, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  SMX_CUDA_CHECK(cudaStreamSynchronize(st));
  if (tab) cudaFreeAsync(tab, st);
  cudaFreeAsync(starts, st);
  return 0;
}

// Records from drawn source positions: keys[j] = key_tab[v] (or v), vals[j] =
// pay_tab[j / kdiv]; optional used-value bitmap bit (mark_tab ? mark_tab[v] : v).
__global__ void records_from_values_kernel(const uint32_t* values, uint64_t n, const uint32_t* key_tab,
                                           const uint32_t* pay_tab, smx::FastDiv kd, uint32_t* keys,
                                           uint32_t* vals, uint32_t* bits, const uint32_t* mark_tab) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t v = values[j];
  if (keys) keys[j] = key_tab ? key_tab[v] : v;
  if (vals) vals[j] = pay_tab[kd.div((uint32_t)j)];
  if (bits) {
    const uint32_t b = mark_tab ? mark_tab[v] : v;
    const uint32_t m = 1u << (b & 31);
    if (!(bits[b >> 5] & m)) atomicOr(&bits[b >> 5], m);
  }
}

extern "C" int smx_records_from_values(const uint32_t* values, uint64_t n, const uint32_t* key_tab,
                                       const uint32_t* pay_tab, uint32_t kdiv, uint32_t* keys, uint32_t* vals,
                                       uint32_t* bits, const uint32_t* mark_tab, void* stream) {
  if (n == 0) return 0;
  if (n >= (1ULL << 32)) {
    smx_set_error("smx_records_from_values: %llu records exceed 2^32", (unsigned long long)n);
    return -1;
  }
  smx_count_launch();
  records_from_values_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(values, n, key_tab, pay_tab,
                                                                         FastDiv::make(kdiv ? kdiv : 1), keys, vals,
                                                                         bits, mark_tab);
  SMX_LAUNCH_CHECK();
  return 0;
}
