// Propagation kernels: one simulation step of one rank (sm/engine.py:277-310).
//
//   lif_kernel          consume_inputs + lif_step (sm/dynamics.py:191-204,
//                       kernels/_speedups.pyx:13-35): read and zero the ring
//                       slot now%L of every real row (summed over ports), add
//                       i_e, advance V with the exact propagator in fp64
//                       without FMA, and ballot the spikes into a bitmap.
//   poisson_emit_kernel PoissonSource.emit_into (sm/dynamics.py:235-248) from
//                       precomputed numpy-exact counts (poisson.cu).
//   spikes_kernel       flatnonzero + SpikeRecorder.append + route_point_spikes /
//                       route_group_spikes (sm/engine.py:89-128): ordered spike
//                       list, raster append, per-destination packets, and the
//                       local delivery source list.
//   unpack_kernel       deliver_point_packets / deliver_gather_packets
//                       (sm/engine.py:146-190): packet positions -> image nodes
//                       via L (p2p) or I (collective, -1 dropped).
//   plan / deliver      deliver_spikes (kernels/_speedups.pyx:38-54): every
//                       (source node, emission step) expands its CSR range of
//                       records into atomicAdd(ring[(t+d)%L][port][row], w*m).
//
// Ring layout is slot-major [L][P][N_real] fp64, real rows only.  fp64 adds
// are exact for the dyadic weights of the reference models, so atomic order
// does not change any bit; for non-dyadic weights V stays within the stated
// tolerance.
#include <algorithm>
#include "common.cuh"

namespace {

constexpr int T256 = 256;
inline unsigned nblk(uint64_t n, int t = T256) { return (unsigned)((n + t - 1) / t); }

struct LifState {
  double* v;
  int32_t* ref;
  const double* decay;
  const double* v_rest;
  const double* v_reset;
  const double* v_th;
  const int32_t* ref_steps;
  const double* i_e;
};

__global__ void lif_kernel(LifState s, uint32_t n, double* ring, int n_ports, int L, const int64_t* now_dev,
                           uint32_t* spike_bits) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t now = *now_dev;
  bool spk = false;
  if (i < n) {
    const int slot = (int)(now % L);
    double* base = ring + (size_t)slot * n_ports * n;
    double in = base[i];
    base[i] = 0.0;
    for (int p = 1; p < n_ports; ++p) {
      in = __dadd_rn(in, base[(size_t)p * n + i]);
      base[(size_t)p * n + i] = 0.0;
    }
    in = __dadd_rn(in, s.i_e[i]);
    const int32_t r = s.ref[i];
    if (r > 0) {
      s.ref[i] = r - 1;
      s.v[i] = s.v_reset[i];
    } else {
      const double vr = s.v_rest[i];
      const double integ = __dadd_rn(__dadd_rn(vr, __dmul_rn(__dsub_rn(s.v[i], vr), s.decay[i])), in);
      if (integ >= s.v_th[i]) {
        spk = true;
        s.v[i] = s.v_reset[i];
        s.ref[i] = s.ref_steps[i];
      } else {
        s.v[i] = integ;
      }
    }
  }
  const uint32_t b = __ballot_sync(0xffffffffu, spk);
  if ((threadIdx.x & 31) == 0 && (i >> 5) < (n + 31) / 32) spike_bits[i >> 5] = b;
}

// counts: [S][n_t] batch of S steps starting at a multiple of S; the row
// and the ring slot (now + delay) % L are taken from the device step counter.
__global__ void poisson_emit_kernel(const uint8_t* counts, int S, uint32_t n_t, const uint32_t* rows, double w,
                                    double* ring, uint32_t n_rows, int n_ports, int L, int delay, int port,
                                    const int64_t* now_dev) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_t) return;
  const int64_t now = *now_dev;
  const uint32_t c = counts[(size_t)(now % S) * n_t + t];
  if (c) {
    const int slot = (int)((now + delay) % L);
    atomicAdd(ring + ((size_t)slot * n_ports + port) * n_rows + rows[t], __dmul_rn(w, (double)c));
  }
}

struct Routes {             // one routing family (p2p T/P or collective G/Q)
  const int64_t* first;     // [M+1]
  const int32_t* dest;      // destination rank (p2p) or group slot (collective)
  const uint32_t* pos;      // map / roster position
  int n_dest;               // number of packet buffers
  uint32_t* packets;        // [n_dest][cap] (position, step) pairs
  uint32_t* counts;         // [n_dest]
  uint32_t cap;
};

struct SpikeOut {
  const uint32_t* spike_bits;
  uint32_t n_rows;
  const uint32_t* row2node;
  const int64_t* gid;       // per row
  int64_t* now_dev;         // step counter, advanced by this kernel
  const int* record_dev;
  // local delivery source list (node, step)
  uint32_t* src_nodes;
  uint32_t* src_steps;
  uint32_t* n_src;          // device counter (appended to)
  uint32_t src_cap;
  // raster
  int64_t* rec;             // (step, gid) pairs
  uint64_t* n_rec;
  uint64_t rec_cap;
  uint32_t* spike_count;    // per-step total (optional accumulation)
  int* overflow;
};

// Single CTA: ordered compaction of the spike bitmap, raster append, local
// delivery list, and packets for both routing families.
__global__ void __launch_bounds__(1024) spikes_kernel(const __grid_constant__ SpikeOut o, const __grid_constant__ Routes p2p,
                                                      const __grid_constant__ Routes grp) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry, src_base;
  __shared__ uint32_t pk_base[2][64];
  const int tid = threadIdx.x;
  const int64_t now = *o.now_dev;
  const int record = *o.record_dev;
  if (tid == 0) { carry = 0; src_base = 0; }
  for (int d = tid; d < 64; d += blockDim.x) {
    pk_base[0][d] = d < p2p.n_dest ? p2p.counts[d] : 0;
    pk_base[1][d] = d < grp.n_dest ? grp.counts[d] : 0;
  }
  __syncthreads();
  const uint32_t nwords = (o.n_rows + 31) / 32;
  for (uint32_t w0 = 0; w0 < nwords; w0 += blockDim.x) {
    const uint32_t w = w0 + tid;
    uint32_t bits = w < nwords ? o.spike_bits[w] : 0;
    uint32_t tot;
    const uint32_t ex = smx::block_excl_scan(__popc(bits), ws, tot);
    uint32_t k = carry + ex;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint32_t row = w * 32 + b;
      const uint32_t node = o.row2node[row];
      const uint32_t si = src_base + k;
      if (si < o.src_cap) { o.src_nodes[si] = node; o.src_steps[si] = (uint32_t)now; }
      else atomicExch(o.overflow, 1);
      if (record) {
        const uint64_t ri = *o.n_rec + k;
        if (ri < o.rec_cap) { o.rec[2 * ri] = now; o.rec[2 * ri + 1] = o.gid[row]; }
        else atomicExch(o.overflow, 2);
      }
      ++k;
    }
    __syncthreads();
    if (tid == 0) carry += tot;
    __syncthreads();
  }
  const uint32_t n_spk = carry;
  // packets: positions in spike order, per destination in route order
  for (int fam = 0; fam < 2; ++fam) {
    const Routes& R = fam ? grp : p2p;
    if (R.n_dest == 0) continue;
    for (uint32_t c0 = 0; c0 < n_spk; c0 += blockDim.x) {
      const uint32_t c = c0 + tid;
      int64_t lo = 0, hi = 0;
      if (c < n_spk && src_base + c < o.src_cap) {
        const uint32_t node = o.src_nodes[src_base + c];
        lo = R.first[node];
        hi = R.first[node + 1];
      }
      for (int d = 0; d < R.n_dest; ++d) {
        uint32_t cnt = 0;
        for (int64_t e = lo; e < hi; ++e) cnt += (R.dest[e] == d);
        uint32_t tot;
        const uint32_t ex = smx::block_excl_scan(cnt, ws, tot);
        uint32_t q = pk_base[fam][d] + ex;
        for (int64_t e = lo; e < hi; ++e) {
          if (R.dest[e] != d) continue;
          if (q < R.cap) {
            R.packets[2 * ((size_t)d * R.cap + q)] = R.pos[e];
            R.packets[2 * ((size_t)d * R.cap + q) + 1] = (uint32_t)now;
          } else {
            atomicExch(o.overflow, 3);
          }
          ++q;
        }
        __syncthreads();
        if (tid == 0) pk_base[fam][d] += tot;
        __syncthreads();
      }
    }
    for (int d = tid; d < R.n_dest; d += blockDim.x) R.counts[d] = min(pk_base[fam][d], R.cap);
  }
  if (tid == 0) {
    *o.n_src = min(src_base + n_spk, o.src_cap);
    if (record) *o.n_rec += n_spk;
    if (o.spike_count) *o.spike_count += n_spk;
    *o.now_dev = now + 1;
  }
}

// Packet positions -> image nodes appended to a delivery source list.
// `count` comes from the sending rank: it is clamped to the block's capacity
// (max_count) so a corrupt or over-full block cannot read past it.
__global__ void unpack_kernel(const uint32_t* packets, const uint32_t* count, uint32_t max_count,
                              const int64_t* table, uint64_t table_len, uint32_t* src_nodes, uint32_t* src_steps,
                              uint32_t* n_src, uint32_t src_cap, int* err) {
  uint32_t n = *count;
  if (n > max_count) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(err, 5);
    n = max_count;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t p = packets[2 * i];
    if (p >= table_len) { atomicExch(err, 4); continue; }
    const int64_t img = table[p];
    if (img < 0) continue;
    const uint32_t k = atomicAdd(n_src, 1u);
    if (k < src_cap) { src_nodes[k] = (uint32_t)img; src_steps[k] = packets[2 * i + 1]; }
    else atomicExch(err, 1);
  }
}

constexpr uint32_t CHUNK = 1024;  // records per delivery work item

// Single CTA: work-item prefix over the source list (ceil(len/CHUNK) each).
__global__ void __launch_bounds__(1024) plan_kernel(const uint32_t* src_nodes, const uint32_t* n_src,
                                                    const int64_t* first, uint32_t* wprefix, uint32_t* n_work) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t n = *n_src;
  for (uint32_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const uint32_t c = c0 + threadIdx.x;
    uint32_t w = 0;
    if (c < n) {
      const uint32_t node = src_nodes[c];
      const int64_t len = first[node + 1] - first[node];
      w = (uint32_t)((len + CHUNK - 1) / CHUNK);
    }
    uint32_t tot;
    const uint32_t ex = smx::block_excl_scan(w, ws, tot);
    if (c < n) wprefix[c] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_work = carry;
}

struct SynTable {  // packed mode: class -> (weight, delay, port)
  const double* w;
  const uint32_t* delay;
  const uint32_t* port;
};

template <bool WIDE>
__global__ void __launch_bounds__(T256) deliver_kernel(const uint32_t* src_nodes, const uint32_t* src_steps,
                                                       const uint32_t* n_src, const uint32_t* wprefix,
                                                       const uint32_t* n_work, const int64_t* first,
                                                       const uint32_t* payload, SynTable syn, const double* wide_w,
                                                       const uint32_t* wide_meta, double* ring, uint32_t n_rows,
                                                       int n_ports, int L) {
  const uint32_t nw = *n_work, ns = *n_src;
  __shared__ double cw[256];
  __shared__ uint32_t cd[256], cp[256];
  if (!WIDE) {
    for (int c = threadIdx.x; c < 256; c += blockDim.x) {
      cw[c] = syn.w[c];
      cd[c] = syn.delay[c];
      cp[c] = syn.port[c];
    }
    __syncthreads();
  }
  const size_t slot_stride = (size_t)n_ports * n_rows;
  for (uint32_t w = blockIdx.x; w < nw; w += gridDim.x) {
    // source index: last c with wprefix[c] <= w
    uint32_t lo = 0, hi = ns - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (wprefix[mid] <= w) lo = mid; else hi = mid - 1;
    }
    const uint32_t node = src_nodes[lo];
    const int64_t now = src_steps[lo];
    const uint32_t slot0 = (uint32_t)(now % L);  // once per work item
    const int64_t a = first[node] + (int64_t)(w - wprefix[lo]) * CHUNK;
    int64_t b = first[node + 1];
    if (b > a + CHUNK) b = a + CHUNK;
    for (int64_t k = a + threadIdx.x; k < b; k += blockDim.x) {
      const uint32_t pl = payload[k];
      double wt;
      uint32_t d, port, row;
      if (WIDE) {
        const uint32_t m = wide_meta[k];
        wt = wide_w[k];
        d = m & 0xffffffu;
        port = m >> 24;
        row = pl;
      } else {
        const uint32_t c = pl >> SMX_ROW_BITS;
        wt = cw[c];
        d = cd[c];
        port = cp[c];
        row = pl & SMX_ROW_MASK;
      }
      uint32_t slot = slot0 + d;  // d < L: one conditional wrap
      if (slot >= (uint32_t)L) slot -= (uint32_t)L;
      atomicAdd(ring + slot * slot_stride + (size_t)port * n_rows + row, wt);
    }
  }
}


// ---------------------------------------------------------------------------
// Fused step kernel: consume + LIF (all real rows), Poisson emission (every
// device with unique target rows, thread t = target t), spike compaction
// with warp-aggregated atomics, raster append, packet routing and the local
// delivery work list -- one launch per step.  Spike order inside the lists
// is not the reference's ascending order; delivery sums are exact for dyadic
// weights and the merged raster is sorted, so results are unchanged.
// ---------------------------------------------------------------------------
constexpr int MAX_FUSED_DEV = 8;

struct FusedDev {
  const uint8_t* counts;  // [S][n_t]
  const int32_t* inv;     // row -> target index, -1 if the row is not a target
  uint32_t n_t;
  double w;
  int delay, port;
};

struct StepArgs {
  LifState s;
  uint32_t n;
  double* ring;
  int n_ports, L;
  int64_t* now_dev;
  const int* record_dev;
  int S;
  int n_dev;
  FusedDev dev[MAX_FUSED_DEV];
  const uint32_t* row2node;
  const int64_t* gid;
  const int64_t* first;           // CSR of the store (for work chunks)
  uint32_t* src_nodes;
  uint32_t* src_steps;
  uint32_t* wbase;                // first work item of each listed source
  uint32_t* owner;                // work item -> list entry
  uint32_t owner_cap;
  unsigned long long* ctr;        // [2] (n_src << 32 | n_work), by step parity
  uint32_t src_cap;
  int64_t* rec;
  unsigned long long* n_rec;
  uint64_t rec_cap;
  int* err;
  int step_offset;                // now = *now_dev (block start) + step_offset
  Routes p2p, grp;
};

__device__ __forceinline__ void route_spike(const Routes& R, uint32_t node, int64_t now, int* err) {
  if (R.n_dest == 0) return;
  const int64_t a = R.first[node], b = R.first[node + 1];
  for (int64_t e = a; e < b; ++e) {
    const int d = R.dest[e];
    const uint32_t q = atomicAdd(&R.counts[d], 1u);
    if (q < R.cap) {
      R.packets[2 * ((size_t)d * R.cap + q)] = R.pos[e];
      R.packets[2 * ((size_t)d * R.cap + q) + 1] = (uint32_t)now;
    } else {
      atomicExch(err, 3);
    }
  }
}

// Poisson drive consumed at arrival time: the count a device emitted at
// step now - d onto this row (PoissonSource.emit_into adds w * count into
// slot (t + d) % L, sm/dynamics.py:235-248; for dyadic w the sum is the same
// whether it passes through the ring or is added here).  counts is a ring of
// A.S steps (three batches), so emissions up to one batch back are kept.
__device__ __forceinline__ double add_poisson_input(const StepArgs& A, uint32_t i, int64_t now, double in) {
  for (int k = 0; k < A.n_dev; ++k) {
    const FusedDev& D = A.dev[k];
    const int32_t t = D.inv[i];
    const int64_t te = now - D.delay;
    if (t < 0 || te < 0) continue;
    const uint32_t c = __ldg(D.counts + (size_t)(te % A.S) * D.n_t + t);
    if (c) in = __dadd_rn(in, __dmul_rn(D.w, (double)c));
  }
  return in;
}

__device__ __noinline__ void spike_lists(const StepArgs& A, uint32_t i, int lane, int64_t now, int par, bool spk,
                                              uint32_t ball) {
  // local delivery list: (index, work base) reserved with one 64-bit atomic per warp
  uint32_t node = 0, chunks = 0;
  if (spk) {
    node = A.row2node[i];
    const int64_t len = A.first[node + 1] - A.first[node];
    chunks = (uint32_t)((len + CHUNK - 1) / CHUNK);
  }
  uint32_t cpre = smx::warp_incl_scan(chunks);
  const uint32_t ctot = __shfl_sync(0xffffffffu, cpre, 31);
  cpre -= chunks;
  const int leader = __ffs(ball) - 1;
  unsigned long long old = 0;
  if (lane == leader)
    old = atomicAdd(&A.ctr[par], ((unsigned long long)__popc(ball) << 32) | (unsigned long long)ctot);
  old = __shfl_sync(0xffffffffu, old, leader);
  const int record = *A.record_dev;
  unsigned long long rbase = 0;
  if (record && lane == leader) rbase = atomicAdd(A.n_rec, (unsigned long long)__popc(ball));
  rbase = __shfl_sync(0xffffffffu, rbase, leader);
  if (!spk) return;
  const uint32_t rank = __popc(ball & ((1u << lane) - 1));
  const uint32_t idx = (uint32_t)(old >> 32) + rank;
  if (idx < A.src_cap) {
    A.src_nodes[idx] = node;
    A.src_steps[idx] = (uint32_t)now;
    const uint32_t wb = (uint32_t)old + cpre;
    A.wbase[idx] = wb;
    for (uint32_t j = 0; j < chunks; ++j) {
      if (wb + j < A.owner_cap) A.owner[wb + j] = idx;
      else atomicExch(A.err, 5);
    }
  } else {
    atomicExch(A.err, 1);
  }
  if (record) {
    const unsigned long long ri = rbase + rank;
    if (ri < A.rec_cap) { A.rec[2 * ri] = now; A.rec[2 * ri + 1] = A.gid[i]; }
    else atomicExch(A.err, 2);
  }
  route_spike(A.p2p, node, now, A.err);
  route_spike(A.grp, node, now, A.err);
}


__global__ void __launch_bounds__(T256) step_kernel(const __grid_constant__ StepArgs A) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t now = *A.now_dev + A.step_offset;
  const int par = (int)(now & 1);
  if (i == 0) A.ctr[par ^ 1] = 0ULL;  // next step's list (its last reader finished)
  // consume + LIF (sm/dynamics.py:191-204, kernels/_speedups.pyx:17-35)
  bool spk = false;
  if (i < A.n) {
    const int slot = (int)(now % A.L);
    double* base = A.ring + (size_t)slot * A.n_ports * A.n;
    double in = base[i];
    base[i] = 0.0;
    for (int p = 1; p < A.n_ports; ++p) {
      in = __dadd_rn(in, base[(size_t)p * A.n + i]);
      base[(size_t)p * A.n + i] = 0.0;
    }
    in = add_poisson_input(A, i, now, in);
    in = __dadd_rn(in, A.s.i_e[i]);
    const int32_t r = A.s.ref[i];
    if (r > 0) {
      A.s.ref[i] = r - 1;
      A.s.v[i] = A.s.v_reset[i];
    } else {
      const double vr = A.s.v_rest[i];
      const double integ = __dadd_rn(__dadd_rn(vr, __dmul_rn(__dsub_rn(A.s.v[i], vr), A.s.decay[i])), in);
      if (integ >= A.s.v_th[i]) {
        spk = true;
        A.s.v[i] = A.s.v_reset[i];
        A.s.ref[i] = A.s.ref_steps[i];
      } else {
        A.s.v[i] = integ;
      }
    }
  }
  const uint32_t ball = __ballot_sync(0xffffffffu, spk);
  if (ball) spike_lists(A, i, lane, now, par, spk, ball);
}


template <bool WIDE>
__global__ void __launch_bounds__(T256) deliver_step_kernel(const uint32_t* src_nodes, const uint32_t* src_steps,
                                                            const uint32_t* wbase, const uint32_t* owner,
                                                            const unsigned long long* ctr,
                                                            const int64_t* now_dev, const int64_t* first,
                                                            const uint32_t* payload, SynTable syn,
                                                            const double* wide_w, const uint32_t* wide_meta,
                                                            double* ring, uint32_t n_rows, int n_ports, int L,
                                                            int step_offset) {
  const unsigned long long c = now_dev ? ctr[(*now_dev + step_offset) & 1] : ctr[0];
  const uint32_t nw = (uint32_t)(c & 0xffffffffULL);
  if (nw == 0) return;
  __shared__ double cw[256];
  __shared__ uint32_t cd[256], cp[256];
  if (!WIDE) {
    for (int k = threadIdx.x; k < 256; k += blockDim.x) {
      cw[k] = syn.w[k];
      cd[k] = syn.delay[k];
      cp[k] = syn.port[k];
    }
    __syncthreads();
  }
  const size_t slot_stride = (size_t)n_ports * n_rows;
  for (uint32_t w = blockIdx.x; w < nw; w += gridDim.x) {
    const uint32_t e = owner[w];  // list entry whose chunk range holds w
    const uint32_t node = src_nodes[e];
    const int64_t now = src_steps[e];
    const uint32_t slot0 = (uint32_t)(now % L);  // once per work item
    const int64_t a = first[node] + (int64_t)(w - wbase[e]) * CHUNK;
    int64_t b = first[node + 1];
    if (b > a + CHUNK) b = a + CHUNK;
    for (int64_t k = a + threadIdx.x; k < b; k += blockDim.x) {
      const uint32_t pl = payload[k];
      double wt;
      uint32_t d, port, row;
      if (WIDE) {
        const uint32_t m = wide_meta[k];
        wt = wide_w[k];
        d = m & 0xffffffu;
        port = m >> 24;
        row = pl;
      } else {
        const uint32_t cl = pl >> SMX_ROW_BITS;
        wt = cw[cl];
        d = cd[cl];
        port = cp[cl];
        row = pl & SMX_ROW_MASK;
      }
      uint32_t slot = slot0 + d;  // d < L: one conditional wrap
      if (slot >= (uint32_t)L) slot -= (uint32_t)L;
      atomicAdd(ring + slot * slot_stride + (size_t)port * n_rows + row, wt);
    }
  }
}


// ---------------------------------------------------------------------------
// Multi-step block kernel: when every connection delay and every non-aligned
// Poisson delay is >= n_steps, the n_steps LIF updates of a block do not see
// each other's spikes (a spike emitted at t lands in slot t + d >= block end).
// Each thread then advances its neuron through the whole block with the state
// in registers -- ring slot, Poisson count and LIF per step -- and appends its
// spikes (node, step) to one delivery list for the block (sm/engine.py:285-296
// repeated n_steps times, identical results).
// ---------------------------------------------------------------------------
constexpr int MAX_BLOCK = 16;  // steps per LIF block (inputs staged in shared memory)
constexpr int TB = 128;        // threads per CTA of the block kernel

// n_steps (<= MAX_BLOCK) consecutive steps of every real row.  No ring slot
// read here is written during the block (every record delay >= n_steps, the
// Poisson drive is consumed at arrival), so all inputs are loaded up front
// with independent loads into shared memory, the slots are zeroed, and the
// LIF recurrence runs as a short rolled loop (small code: the kernel was
// instruction-fetch bound when fully unrolled).
__global__ void __launch_bounds__(TB) lif_block_kernel(const __grid_constant__ StepArgs A, int n_steps) {
  __shared__ double rin[MAX_BLOCK][TB];
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, tx = threadIdx.x;
  const int64_t t0 = *A.now_dev + A.step_offset;
  const bool live = i < A.n;
  const uint32_t L = (uint32_t)A.L;
  const size_t slot_stride = (size_t)A.n_ports * A.n;
  const uint32_t sl0 = (uint32_t)(t0 % A.L);
  if (live) {
    // slot sl0 + s, port p; summed over ports in port order as consume does
#pragma unroll 1
    for (int p = 0; p < A.n_ports; ++p) {
      double x[MAX_BLOCK];
      uint32_t sl = sl0;
#pragma unroll
      for (int s = 0; s < MAX_BLOCK; ++s) {
        x[s] = s < n_steps ? A.ring[(size_t)sl * slot_stride + (size_t)p * A.n + i] : 0.0;
        if (++sl == L) sl = 0;
      }
#pragma unroll
      for (int s = 0; s < MAX_BLOCK; ++s)
        if (s < n_steps) rin[s][tx] = p == 0 ? x[s] : __dadd_rn(rin[s][tx], x[s]);
    }
    // Poisson drive emitted at t0 + s - d (same association as step_kernel)
    for (int k = 0; k < A.n_dev; ++k) {
      const FusedDev& D = A.dev[k];
      const int32_t t = D.inv[i];
      if (t < 0) continue;
      const int64_t te0 = t0 - D.delay;
      uint32_t ci = (uint32_t)(((te0 % A.S) + A.S) % A.S);
      uint32_t cs[MAX_BLOCK];
#pragma unroll
      for (int s = 0; s < MAX_BLOCK; ++s) {  // independent loads first
        cs[s] = (s < n_steps && te0 + s >= 0) ? __ldg(D.counts + (size_t)ci * D.n_t + t) : 0u;
        if (++ci == (uint32_t)A.S) ci = 0;
      }
#pragma unroll
      for (int s = 0; s < MAX_BLOCK; ++s)
        if (cs[s]) rin[s][tx] = __dadd_rn(rin[s][tx], __dmul_rn(D.w, (double)cs[s]));
    }
#pragma unroll 1
    for (int p = 0; p < A.n_ports; ++p) {
      uint32_t sl = sl0;
#pragma unroll
      for (int s = 0; s < MAX_BLOCK; ++s) {
        if (s < n_steps) A.ring[(size_t)sl * slot_stride + (size_t)p * A.n + i] = 0.0;
        if (++sl == L) sl = 0;
      }
    }
  }
  double v = 0.0, vr = 0.0, vreset = 0.0, vth = 0.0, decay = 0.0, ie = 0.0;
  int32_t ref = 0, refsteps = 0;
  if (live) {
    v = A.s.v[i]; ref = A.s.ref[i];
    vr = A.s.v_rest[i]; vreset = A.s.v_reset[i]; vth = A.s.v_th[i]; decay = A.s.decay[i]; ie = A.s.i_e[i];
    refsteps = A.s.ref_steps[i];
  }
#pragma unroll 1
  for (int s = 0; s < n_steps; ++s) {
    bool spk = false;
    if (live) {
      const double in = __dadd_rn(rin[s][tx], ie);
      if (ref > 0) {
        ref -= 1;
        v = vreset;
      } else {
        const double integ = __dadd_rn(__dadd_rn(vr, __dmul_rn(__dsub_rn(v, vr), decay)), in);
        if (integ >= vth) { spk = true; v = vreset; ref = refsteps; }
        else v = integ;
      }
    }
    const uint32_t ball = __ballot_sync(0xffffffffu, spk);
    if (ball) spike_lists(A, i, lane, t0 + s, 0, spk, ball);
  }
  if (live) { A.s.v[i] = v; A.s.ref[i] = ref; }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI (engine layout)
// ---------------------------------------------------------------------------

extern "C" int smx_lif_update(double* v, int32_t* ref, const double* decay, const double* v_rest,
                              const double* v_reset, const double* v_th, const int32_t* ref_steps,
                              const double* i_e, uint32_t n, double* ring, int n_ports, int L,
                              const int64_t* now_dev, uint32_t* spike_bits, void* stream) {
  if (n == 0) return 0;
  LifState s{v, ref, decay, v_rest, v_reset, v_th, ref_steps, i_e};
  smx_count_launch(); lif_kernel<<<nblk(n), T256, 0, (cudaStream_t)stream>>>(s, n, ring, n_ports, L, now_dev, spike_bits);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_poisson_emit(const uint8_t* counts, int S, uint32_t n_t, const uint32_t* rows, double w,
                                double* ring, uint32_t n_rows, int n_ports, int L, int delay, int port,
                                const int64_t* now_dev, void* stream) {
  if (n_t == 0) return 0;
  smx_count_launch(); poisson_emit_kernel<<<nblk(n_t), T256, 0, (cudaStream_t)stream>>>(counts, S, n_t, rows, w, ring, n_rows, n_ports, L, delay, port, now_dev);
  SMX_LAUNCH_CHECK();
  return 0;
}

// Route-family descriptor as laid out by the host (matches Routes).
struct SmxRoutes {
  const int64_t* first;
  const int32_t* dest;
  const uint32_t* pos;
  int n_dest;
  uint32_t* packets;
  uint32_t* counts;
  uint32_t cap;
};

extern "C" int smx_spikes(const uint32_t* spike_bits, uint32_t n_rows, const uint32_t* row2node,
                          const int64_t* gid, int64_t* now_dev, uint32_t* src_nodes, uint32_t* src_steps,
                          uint32_t* n_src, uint32_t src_cap, const int* record_dev, int64_t* rec, uint64_t* n_rec,
                          uint64_t rec_cap, uint32_t* spike_count, int* overflow, const SmxRoutes* p2p,
                          const SmxRoutes* grp, void* stream) {
  SpikeOut o;
  o.spike_bits = spike_bits;
  o.n_rows = n_rows;
  o.row2node = row2node;
  o.gid = gid;
  o.now_dev = now_dev;
  o.record_dev = record_dev;
  o.src_nodes = src_nodes;
  o.src_steps = src_steps;
  o.n_src = n_src;
  o.src_cap = src_cap;
  o.rec = rec;
  o.n_rec = n_rec;
  o.rec_cap = rec_cap;
  o.spike_count = spike_count;
  o.overflow = overflow;
  Routes a{}, b{};
  if (p2p) a = Routes{p2p->first, p2p->dest, p2p->pos, p2p->n_dest, p2p->packets, p2p->counts, p2p->cap};
  if (grp) b = Routes{grp->first, grp->dest, grp->pos, grp->n_dest, grp->packets, grp->counts, grp->cap};
  if (a.n_dest > 64 || b.n_dest > 64) {
    smx_set_error("at most 64 packet destinations per routing family");
    return -1;
  }
  smx_count_launch(); spikes_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(o, a, b);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_unpack(const uint32_t* packets, const uint32_t* count, uint32_t max_count, const int64_t* table,
                          uint64_t table_len, uint32_t* src_nodes, uint32_t* src_steps, uint32_t* n_src,
                          uint32_t src_cap, int* err, void* stream) {
  smx_count_launch(); unpack_kernel<<<148, T256, 0, (cudaStream_t)stream>>>(packets, count, max_count, table, table_len,
                                                                         src_nodes, src_steps, n_src, src_cap, err);
  SMX_LAUNCH_CHECK();
  return 0;
}

// Deliver every (node, step) of the source list through the CSR tables.
// wprefix needs src_cap entries, work a 1-word counter.
extern "C" int smx_deliver(const uint32_t* src_nodes, const uint32_t* src_steps, const uint32_t* n_src,
                           uint32_t* wprefix, uint32_t* n_work, const int64_t* first, const uint32_t* payload,
                           const double* cls_w, const uint32_t* cls_delay, const uint32_t* cls_port,
                           const double* wide_w, const uint32_t* wide_meta, double* ring, uint32_t n_rows,
                           int n_ports, int L, int grid, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  smx_count_launch(); plan_kernel<<<1, 1024, 0, st>>>(src_nodes, n_src, first, wprefix, n_work);
  SynTable syn{cls_w, cls_delay, cls_port};
  if (grid <= 0) grid = 148 * 8;
  if (wide_w) {
    smx_count_launch(); deliver_kernel<true><<<grid, T256, 0, st>>>(src_nodes, src_steps, n_src, wprefix, n_work, first, payload, syn,
                                                 wide_w, wide_meta, ring, n_rows, n_ports, L);
  } else {
    smx_count_launch(); deliver_kernel<false><<<grid, T256, 0, st>>>(src_nodes, src_steps, n_src, wprefix, n_work, first, payload, syn,
                                                  wide_w, wide_meta, ring, n_rows, n_ports, L);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}

// Host mirror of the fused-device descriptor.
struct SmxFusedDev {
  const uint8_t* counts;
  const int32_t* inv;
  uint32_t n_t;
  double w;
  int delay, port;
};

// One complete local step (sm/engine.py:285-296) in two launches: fused
// LIF/Poisson/compaction/routing, then local delivery.  The step is
// *now_dev + step_offset: the host sets *now_dev once per exchange block, so a
// block of steps replays from one CUDA graph with no counter kernels.
// ctr: 2 x u64 list counters indexed by step parity.
extern "C" int smx_step(double* v, int32_t* ref, const double* decay, const double* v_rest, const double* v_reset,
                        const double* v_th, const int32_t* ref_steps, const double* i_e, uint32_t n, double* ring,
                        int n_ports, int L, int64_t* now_dev, int step_offset, const int* record_dev, int S,
                        const SmxFusedDev* devs_host, int n_dev, const uint32_t* row2node, const int64_t* gid,
                        const int64_t* first, uint32_t* src_nodes, uint32_t* src_steps, uint32_t* wbase,
                        uint32_t* owner, uint32_t owner_cap, unsigned long long* ctr, uint32_t src_cap, int64_t* rec, unsigned long long* n_rec,
                        uint64_t rec_cap, int* err, const SmxRoutes* p2p, const SmxRoutes* grp,
                        const uint32_t* payload, const double* cls_w, const uint32_t* cls_delay,
                        const uint32_t* cls_port, const double* wide_w, const uint32_t* wide_meta, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_dev > MAX_FUSED_DEV) {
    smx_set_error("smx_step: at most %d fused Poisson devices", MAX_FUSED_DEV);
    return -1;
  }
  StepArgs A;
  A.s = LifState{v, ref, decay, v_rest, v_reset, v_th, ref_steps, i_e};
  A.n = n;
  A.ring = ring;
  A.n_ports = n_ports;
  A.L = L;
  A.now_dev = now_dev;
  A.record_dev = record_dev;
  A.S = S;
  A.n_dev = n_dev;
  uint32_t threads = n;
  for (int k = 0; k < n_dev; ++k) {
    A.dev[k] = FusedDev{devs_host[k].counts, devs_host[k].inv, devs_host[k].n_t, devs_host[k].w,
                        devs_host[k].delay, devs_host[k].port};
  }
  A.row2node = row2node;
  A.gid = gid;
  A.first = first;
  A.src_nodes = src_nodes;
  A.src_steps = src_steps;
  A.wbase = wbase;
  A.owner = owner;
  A.owner_cap = owner_cap;
  A.ctr = ctr;
  A.src_cap = src_cap;
  A.rec = rec;
  A.n_rec = n_rec;
  A.rec_cap = rec_cap;
  A.err = err;
  A.step_offset = step_offset;
  A.p2p = p2p ? Routes{p2p->first, p2p->dest, p2p->pos, p2p->n_dest, p2p->packets, p2p->counts, p2p->cap} : Routes{};
  A.grp = grp ? Routes{grp->first, grp->dest, grp->pos, grp->n_dest, grp->packets, grp->counts, grp->cap} : Routes{};
  if (threads == 0) threads = 1;
  smx_count_launch(); step_kernel<<<nblk(threads), T256, 0, st>>>(A);
  // deliver the step's local spikes: the list counters live in ctr[now & 1]
  // (n_src << 32 | n_work); the deliver kernel picks the word by parity
  SynTable syn{cls_w, cls_delay, cls_port};
  const int grid = 148 * 8;
  if (wide_w) {
    smx_count_launch(); deliver_step_kernel<true><<<grid, T256, 0, st>>>(src_nodes, src_steps, wbase, owner, ctr, now_dev, first,
                                                        payload, syn, wide_w, wide_meta, ring, n, n_ports, L, step_offset);
  } else {
    smx_count_launch(); deliver_step_kernel<false><<<grid, T256, 0, st>>>(src_nodes, src_steps, wbase, owner, ctr, now_dev, first,
                                                         payload, syn, wide_w, wide_meta, ring, n, n_ports, L, step_offset);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}

// A block of n_steps local steps in two launches (lif_block_kernel, then the
// delivery of every spike of the block); preconditions in lif_block_kernel.
extern "C" int smx_block(double* v, int32_t* ref, const double* decay, const double* v_rest, const double* v_reset,
                         const double* v_th, const int32_t* ref_steps, const double* i_e, uint32_t n, double* ring,
                         int n_ports, int L, int64_t* now_dev, int step_offset, int n_steps, const int* record_dev,
                         int S, const SmxFusedDev* devs_host, int n_dev, const uint32_t* row2node, const int64_t* gid,
                         const int64_t* first, uint32_t* src_nodes, uint32_t* src_steps, uint32_t* wbase,
                         uint32_t* owner, uint32_t owner_cap, unsigned long long* ctr, uint32_t src_cap, int64_t* rec,
                         unsigned long long* n_rec, uint64_t rec_cap, int* err, const SmxRoutes* p2p,
                         const SmxRoutes* grp, const uint32_t* payload, const double* cls_w, const uint32_t* cls_delay,
                         const uint32_t* cls_port, const double* wide_w, const uint32_t* wide_meta, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_dev > MAX_FUSED_DEV) {
    smx_set_error("smx_block: at most %d fused Poisson devices", MAX_FUSED_DEV);
    return -1;
  }
  StepArgs A;
  A.s = LifState{v, ref, decay, v_rest, v_reset, v_th, ref_steps, i_e};
  A.n = n;
  A.ring = ring;
  A.n_ports = n_ports;
  A.L = L;
  A.now_dev = now_dev;
  A.record_dev = record_dev;
  A.S = S;
  A.n_dev = n_dev;
  uint32_t threads = n;
  for (int k = 0; k < n_dev; ++k) {
    A.dev[k] = FusedDev{devs_host[k].counts, devs_host[k].inv, devs_host[k].n_t, devs_host[k].w,
                        devs_host[k].delay, devs_host[k].port};
  }
  A.row2node = row2node;
  A.gid = gid;
  A.first = first;
  A.src_nodes = src_nodes;
  A.src_steps = src_steps;
  A.wbase = wbase;
  A.owner = owner;
  A.owner_cap = owner_cap;
  A.ctr = ctr;
  A.src_cap = src_cap;
  A.rec = rec;
  A.n_rec = n_rec;
  A.rec_cap = rec_cap;
  A.err = err;
  A.step_offset = step_offset;
  A.p2p = p2p ? Routes{p2p->first, p2p->dest, p2p->pos, p2p->n_dest, p2p->packets, p2p->counts, p2p->cap} : Routes{};
  A.grp = grp ? Routes{grp->first, grp->dest, grp->pos, grp->n_dest, grp->packets, grp->counts, grp->cap} : Routes{};
  if (threads == 0) threads = 1;
  SMX_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
  if (n_steps > MAX_BLOCK) {
    smx_set_error("smx_block: at most %d steps per block", MAX_BLOCK);
    return -1;
  }
  smx_count_launch(); lif_block_kernel<<<nblk(threads, TB), TB, 0, st>>>(A, n_steps);
  SynTable syn{cls_w, cls_delay, cls_port};
  const int grid = 148 * 8;
  if (wide_w) {
    smx_count_launch(); deliver_step_kernel<true><<<grid, T256, 0, st>>>(src_nodes, src_steps, wbase, owner, ctr, nullptr, first,
                                                        payload, syn, wide_w, wide_meta, ring, n, n_ports, L, 0);
  } else {
    smx_count_launch(); deliver_step_kernel<false><<<grid, T256, 0, st>>>(src_nodes, src_steps, wbase, owner, ctr, nullptr, first,
                                                         payload, syn, wide_w, wide_meta, ring, n, n_ports, L, 0);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}
