// numpy-exact Poisson drive: Generator.poisson(lam, size=n) for lam < 10 on a
// Philox stream whose word cursor carries across calls (PoissonSource draws
// one count per target per step from one stream, sm/dynamics.py:232-248).
//
// numpy's multiplication method (random_poisson_mult) consumes X+1 words per
// sample: prod *= next_double until prod <= exp(-lam).  The word where a
// sample starts therefore depends on every earlier sample.  Parallel form:
//   chunk kernel    per chunk of C words: U and len(w) (= X+1 for a sample
//                   starting at word w) for every word; the orbit of starts
//                   from entry offset 0 (bitmap S0); and for each entry
//                   offset e < E the (exit offset, sample count) -- chains
//                   from different entries merge with S0 after a few samples,
//                   so each is a short walk.
//   compose kernels sequential composition of the per-chunk entry->exit maps
//                   in groups of 64 chunks, then across groups (one thread),
//                   then back into each chunk: true entry and first sample
//                   index of every chunk.
//   emit kernel     walks from the true entry to the merge point, then ranks
//                   the S0 starts in parallel: count[k] = len(start_k) - 1.
// Exact for every input: no speculation is assumed beyond E (a sample longer
// than E-1 words raises the error flag instead of being mis-composed).
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int PC = 2048;          // words per chunk
constexpr int PE = 64;            // entry offsets tracked per chunk
constexpr int PG = 64;            // chunks per composition group
constexpr int P_THREADS = 128;
constexpr int J_RAW_WORDS = PC;   // emit_kernel's staged words (normals start inside the chunk)

struct PoisJob {
  smx::Key key;
  const uint64_t* w0_dev;  // word cursor before the batch (device)
  int kind;           // 0 = poisson counts (u8), 1 = normal(loc, scale) (f64), 2 = poisson PTRS (u8)
  double enlam;       // exp(-lam), computed by the host's libm like numpy
  double lam, slam, loglam, pa, pb, invalpha, vr;  // PTRS constants (lam >= 10)
  double loc, scale;
  uint64_t n;         // samples wanted
  int n_chunks;
  uint8_t* len;       // [n_chunks * PC]
  uint32_t* s0;       // [n_chunks * PC/32]
  uint8_t* ex;        // [n_chunks * PE] exit offsets
  uint16_t* cnt;      // [n_chunks * PE] samples started inside the chunk
  uint8_t* gex;       // [n_groups * PE]
  uint32_t* gcnt;     // [n_groups * PE]
  uint8_t* entry;     // [n_chunks]
  uint64_t* kbase;    // [n_chunks]
  void* out;          // counts[n] (u8) or values[n] (f64)
  uint64_t* cursor;   // word after the n-th sample
  int* err;
};

// numpy random_loggam (Stirling series shifted to x >= 7), fp64 without FMA
__device__ double loggam(double x) {
  const double a[10] = {8.333333333333333e-02, -2.777777777777778e-03, 7.936507936507937e-04,
                        -5.952380952380952e-04, 8.417508417508418e-04, -1.917526917526918e-03,
                        6.410256410256410e-03, -2.955065359477124e-02, 1.796443723688307e-01,
                        -1.39243221690590e+00};
  if (x == 1.0 || x == 2.0) return 0.0;
  const long long n = x < 7.0 ? (long long)(7 - x) : 0;
  double x0 = __dadd_rn(x, (double)n);
  const double r = __ddiv_rn(1.0, x0);
  const double x2 = __dmul_rn(r, r);
  double gl0 = a[9];
  for (int k = 8; k >= 0; --k) gl0 = __dadd_rn(__dmul_rn(gl0, x2), a[k]);
  double gl = __dadd_rn(__dadd_rn(__dadd_rn(__ddiv_rn(gl0, x0), __dmul_rn(0.5, 1.8378770664093453e+00)),
                                  __dmul_rn(__dadd_rn(x0, -0.5), log(x0))), -x0);
  if (x < 7.0) {
    for (long long k = 1; k <= n; ++k) {
      gl = __dadd_rn(gl, -log(__dadd_rn(x0, -1.0)));
      x0 = __dadd_rn(x0, -1.0);
    }
  }
  return gl;
}

// One PTRS trial on (next_double, next_double) = (u, v): returns true and the
// count when accepted (numpy random_poisson_ptrs; log is CUDA's, <= 1 ulp).
__device__ __forceinline__ bool ptrs_trial(const PoisJob& J, double u, double v, long long& k) {
  const double U = __dadd_rn(u, -0.5);
  const double us = __dadd_rn(0.5, -fabs(U));
  k = (long long)floor(__dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(__dmul_rn(2.0, J.pa), us), J.pb), U), J.lam),
                                 0.43));
  if (us >= 0.07 && v <= J.vr) return true;
  if (k < 0 || (us < 0.013 && v > us)) return false;
  const double lhs = __dadd_rn(__dadd_rn(log(v), log(J.invalpha)),
                               -log(__dadd_rn(__ddiv_rn(J.pa, __dmul_rn(us, us)), J.pb)));
  const double rhs = __dadd_rn(__dadd_rn(-J.lam, __dmul_rn((double)k, J.loglam)), -loggam(__dadd_rn((double)k, 1.0)));
  return lhs <= rhs;
}

template <int KIND>
__global__ void __launch_bounds__(P_THREADS) chunk_kernel(PoisJob J) {
  __shared__ double U[PC + PE];
  __shared__ uint8_t L[PC + PE];
  __shared__ uint32_t S0[PC / 32];
  __shared__ uint32_t cnt0_pos[PC / 32 + 1];  // S0 popcount prefix per word
  __shared__ int seg_exit[P_THREADS];
  __shared__ uint16_t M16[P_THREADS];
  __shared__ int exit0, count0;
  const int c = blockIdx.x, tid = threadIdx.x;
  const uint64_t cw = (*J.w0_dev & ~3ULL) + (uint64_t)c * PC;
  // U for words [cw, cw + PC + PE)
  for (int q = tid; q < (PC + PE) / 4; q += P_THREADS) {
    uint64_t b[4];
    smx::philox4x64_10(((cw >> 2) + q) + 1, J.key, b);  // cw is a multiple of 4
#pragma unroll
    for (int i = 0; i < 4; ++i) U[4 * q + i] = KIND == 1 ? __longlong_as_double((long long)b[i]) : smx::u53(b[i]);
  }
  __syncthreads();
  // len(w) for w in [0, PC + PE): products forward; words past the window
  // tail are regenerated one at a time (rare).
  for (int w = tid; w < PC + PE; w += P_THREADS) {
    int k = 0;
    if (KIND == 0) {
      double prod = 1.0;
      for (;;) {
        const int idx = w + k;
        double u;
        if (idx < PC + PE) {
          u = U[idx];
        } else {
          u = smx::u53(smx::philox_word(J.key, cw + idx));
        }
        prod = __dmul_rn(prod, u);
        ++k;
        if (!(prod > J.enlam)) break;
        if (k >= 255) break;
      }
    } else if (KIND == 2) {
      // PTRS: two doubles per trial until one is accepted
      for (;;) {
        const int i0 = w + k, i1 = w + k + 1;
        const double u = i0 < PC + PE ? U[i0] : smx::u53(smx::philox_word(J.key, cw + i0));
        const double v = i1 < PC + PE ? U[i1] : smx::u53(smx::philox_word(J.key, cw + i1));
        k += 2;
        long long cnt;
        if (ptrs_trial(J, u, v, cnt)) break;
        if (k >= 254) break;
      }
    } else {
      // ziggurat: one word on the fast path (raw words staged in U), else
      // run the sampler from the word to count
      double x;
      if (smx::zig_first((uint64_t)__double_as_longlong(U[w]), x)) {
        k = 1;
      } else {
        smx::SeqStream st;
        st.init(J.key, cw + w);
        (void)smx::zig_standard_normal(st);
        const uint64_t used = st.word - (cw + w);
        k = used > 255 ? 255 : (int)used;
      }
    }
    if (k >= PE) atomicExch(J.err, 11);
    L[w] = (uint8_t)k;
  }
  __syncthreads();
  // Orbit of starts from entry offset 0 (bitmap S0), segment-parallel: thread
  // t owns words [SEG*t, SEG*(t+1)) and walks them from its entry (the first
  // orbit position >= SEG*t).  Round 0 guesses the segment start; each later
  // round takes the previous thread's exit as the entry and re-walks only
  // until the walk lands on a start of its previous chain (from there on the
  // chain is unchanged).  After round r segments 0..r are exact, so the loop
  // ends at the exact orbit; chains merge within a few samples, so it
  // normally ends after two or three rounds.
  {
    constexpr int SEG = PC / P_THREADS;
    static_assert(SEG == 16, "segment mask is 16 bits");
    const int lo = SEG * tid, hi = lo + SEG;
    uint32_t mask = 0;
    int entry = lo, ex_ = lo;
    while (ex_ < hi) { mask |= 1u << (ex_ - lo); ex_ += L[ex_]; }
    seg_exit[tid] = ex_;
    for (;;) {
      __syncthreads();
      const int e_in = tid == 0 ? 0 : seg_exit[tid - 1];
      bool changed = false;
      if (e_in != entry) {
        entry = e_in;
        uint32_t m = 0;
        int p = e_in;
        while (p < hi && !((mask >> (p - lo)) & 1)) { m |= 1u << (p - lo); p += L[p]; }
        const int ex_new = p < hi ? ex_ : p;  // merged: same exit as before
        mask = p < hi ? (m | (mask & ~((1u << (p - lo)) - 1))) : m;
        changed = ex_new != ex_;
        ex_ = ex_new;
      }
      __syncthreads();
      seg_exit[tid] = ex_;
      if (!__syncthreads_or(changed)) break;
    }
    M16[tid] = (uint16_t)mask;
    __syncthreads();
    if (tid < PC / 32) S0[tid] = (uint32_t)M16[2 * tid] | ((uint32_t)M16[2 * tid + 1] << 16);
    __syncthreads();
    if (tid < 32) {  // popcount prefix of the 64 S0 words (two per lane)
      const uint32_t a = __popc(S0[2 * tid]), b = __popc(S0[2 * tid + 1]);
      uint32_t x = a + b;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (tid >= o) x += y;
      }
      cnt0_pos[2 * tid] = x - a - b;
      cnt0_pos[2 * tid + 1] = x - b;
      if (tid == 31) { cnt0_pos[PC / 32] = x; count0 = (int)x; exit0 = seg_exit[P_THREADS - 1] - PC; }
    }
  }
  __syncthreads();
  // per entry offset: walk until merging with S0 or leaving the chunk
  for (int e = tid; e < PE; e += P_THREADS) {
    int p = e, pre = 0;
    int ex_ = -1, ct = 0;
    while (p < PC) {
      if ((S0[p >> 5] >> (p & 31)) & 1) {  // merged at start p
        const int rank = cnt0_pos[p >> 5] + __popc(S0[p >> 5] & ((1u << (p & 31)) - 1));
        ex_ = exit0;
        ct = pre + (count0 - rank);
        break;
      }
      ++pre;
      p += L[p];
    }
    if (ex_ < 0) { ex_ = p - PC; ct = pre; }
    if (ex_ >= PE) { atomicExch(J.err, 12); ex_ = PE - 1; }
    J.ex[(size_t)c * PE + e] = (uint8_t)ex_;
    J.cnt[(size_t)c * PE + e] = (uint16_t)ct;
  }
  for (int w = tid; w < PC; w += P_THREADS) J.len[(size_t)c * PC + w] = L[w];
  for (int q = tid; q < PC / 32; q += P_THREADS) J.s0[(size_t)c * (PC / 32) + q] = S0[q];
}

// One CTA per group of PG chunks: the group's entry->exit tables are staged
// in shared memory, then thread e composes them sequentially from entry e.
__global__ void __launch_bounds__(PE) group_kernel(PoisJob J) {
  __shared__ uint8_t ex[PG * PE];
  __shared__ uint16_t ct[PG * PE];
  const int g = blockIdx.x, e0 = threadIdx.x;
  const int c0 = g * PG, c1 = min(J.n_chunks, c0 + PG), nc = c1 - c0;
  for (int q = threadIdx.x; q < nc * PE; q += blockDim.x) {
    ex[q] = J.ex[(size_t)c0 * PE + q];
    ct[q] = J.cnt[(size_t)c0 * PE + q];
  }
  __syncthreads();
  int e = e0;
  uint32_t tot = 0;
  for (int c = 0; c < nc; ++c) {
    tot += ct[c * PE + e];
    e = ex[c * PE + e];
  }
  J.gex[(size_t)g * PE + e0] = (uint8_t)e;
  J.gcnt[(size_t)g * PE + e0] = tot;
}

// Single CTA: the groups' tables are staged in shared memory (in slices),
// then one thread walks the groups in order.
constexpr int ACROSS_SLICE = 96;  // groups per shared-memory slice
__global__ void __launch_bounds__(256) across_kernel(PoisJob J, int n_groups, uint8_t* gentry, uint64_t* gbase) {
  __shared__ uint8_t gx[ACROSS_SLICE * PE];
  __shared__ uint32_t gc[ACROSS_SLICE * PE];
  __shared__ int e_sh;
  __shared__ unsigned long long k_sh;
  if (threadIdx.x == 0) { e_sh = (int)(*J.w0_dev & 3); k_sh = 0; }
  for (int g0 = 0; g0 < n_groups; g0 += ACROSS_SLICE) {
    const int ng = min(ACROSS_SLICE, n_groups - g0);
    __syncthreads();
    for (int q = threadIdx.x; q < ng * PE; q += blockDim.x) {
      gx[q] = J.gex[(size_t)g0 * PE + q];
      gc[q] = J.gcnt[(size_t)g0 * PE + q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int e = e_sh;
      unsigned long long k = k_sh;
      for (int g = 0; g < ng; ++g) {
        gentry[g0 + g] = (uint8_t)e;
        gbase[g0 + g] = k;
        k += gc[g * PE + e];
        e = gx[g * PE + e];
      }
      e_sh = e;
      k_sh = k;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && k_sh < J.n) atomicExch(J.err, 13);  // window too small
}

// One CTA per group: chunk tables staged in shared memory, one thread walks
// the group's chunks from the group's true entry.
__global__ void __launch_bounds__(PE) within_kernel(PoisJob J, const uint8_t* gentry, const uint64_t* gbase) {
  __shared__ uint8_t ex[PG * PE];
  __shared__ uint16_t ct[PG * PE];
  const int g = blockIdx.x;
  const int c0 = g * PG, c1 = min(J.n_chunks, c0 + PG), nc = c1 - c0;
  for (int q = threadIdx.x; q < nc * PE; q += blockDim.x) {
    ex[q] = J.ex[(size_t)c0 * PE + q];
    ct[q] = J.cnt[(size_t)c0 * PE + q];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int e = gentry[g];
  uint64_t k = gbase[g];
  for (int c = 0; c < nc; ++c) {
    J.entry[c0 + c] = (uint8_t)e;
    J.kbase[c0 + c] = k;
    k += ct[c * PE + e];
    e = ex[c * PE + e];
  }
}

// KIND < 0: dispatch on J.kind at run time (the one-pass kernel)
template <int KIND = -1>
__device__ __forceinline__ void emit(const PoisJob& J, uint64_t k, int c, int p, int len, const uint64_t* raw) {
  const int kind = KIND >= 0 ? KIND : J.kind;
  if (k < J.n) {
    const uint64_t start = (*J.w0_dev & ~3ULL) + (uint64_t)c * PC + p;
    if (kind == 0) {
      static_cast<uint8_t*>(J.out)[k] = (uint8_t)(len - 1);
    } else if (kind == 2) {  // PTRS: the count of the accepted (last) trial
      const double u = smx::u53(smx::philox_word(J.key, start + len - 2));
      const double v = smx::u53(smx::philox_word(J.key, start + len - 1));
      long long cnt = 0;
      if (!ptrs_trial(J, u, v, cnt) || cnt < 0 || cnt > 255) atomicExch(J.err, 14);  // u8 counts
      static_cast<uint8_t*>(J.out)[k] = (uint8_t)cnt;
    } else {  // numpy random_normal: loc + scale * z, no FMA
      double z;
      if (len != 1 || !smx::zig_first(raw[p], z)) {   // (raw: the chunk's words, staged)
        smx::SeqStream st;
        st.init(J.key, start);
        z = smx::zig_standard_normal(st);
      }
      static_cast<double*>(J.out)[k] = __dadd_rn(J.loc, __dmul_rn(J.scale, z));
    }
    if (k == J.n - 1) *J.cursor = start + len;
  }
}

// One instance per kind: the Poisson counts' instance carries neither the
// normals' staged words (16 KB of SMEM) nor the samplers' registers.
template <int KIND>
__global__ void __launch_bounds__(P_THREADS) emit_kernel(PoisJob J) {
  __shared__ uint32_t ws[32];
  __shared__ int merge_p, pre_n;
  extern __shared__ uint64_t raw[];   // normals: the chunk's words (dynamic: kind 1 only)
  const int c = blockIdx.x, tid = threadIdx.x;
  const uint64_t kb = J.kbase[c];
  if (kb >= J.n) return;
  const uint8_t* L = J.len + (size_t)c * PC;
  const uint32_t* S0 = J.s0 + (size_t)c * (PC / 32);
  if (KIND == 1) {
    const uint64_t cw = (*J.w0_dev & ~3ULL) + (uint64_t)c * PC;
    for (int q = tid; q < PC / 4; q += P_THREADS) {
      uint64_t b[4];
      smx::philox4x64_10(((cw >> 2) + q) + 1, J.key, b);
#pragma unroll
      for (int i = 0; i < 4; ++i) raw[4 * q + i] = b[i];
    }
    __syncthreads();
  }
  if (tid == 0) {
    int p = J.entry[c], pre = 0;
    while (p < PC && !((S0[p >> 5] >> (p & 31)) & 1)) {
      emit<KIND>(J, kb + pre, c, p, L[p], raw);
      ++pre;
      p += L[p];
    }
    merge_p = p;
    pre_n = pre;
  }
  __syncthreads();
  const int m = merge_p;
  if (m >= PC) return;
  // S0 starts >= m, ranked in order.  Normals (nearly every word starts a
  // sample): word prefix counts first, then every thread takes positions
  // p = m + tid, m + tid + P_THREADS, ... (all threads busy, neighbouring
  // samples to neighbouring threads: coalesced 8-byte stores)
  static_assert(PC / 32 <= P_THREADS, "one S0 word per thread in the prefix");
  if constexpr (KIND != 1) {   // counts (about one start per two words): one S0 word per thread
    const int q = tid;
    uint32_t bits = 0;
    if (q < PC / 32) {
      bits = S0[q];
      const int lo = q * 32;
      if (m > lo) bits &= (m - lo >= 32) ? 0u : ~((1u << (m - lo)) - 1);
    }
    uint32_t tot;
    const uint32_t ex = smx::block_excl_scan(__popc(bits), ws, tot);
    uint64_t k = kb + pre_n + ex;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int p = q * 32 + b;
      emit<KIND>(J, k, c, p, L[p], raw);
      ++k;
    }
    return;
  }
  __shared__ uint32_t wmask[PC / 32], wpre[PC / 32];
  {
    const int q = tid;
    uint32_t bits = 0;
    if (q < PC / 32) {
      bits = S0[q];
      const int lo = q * 32;
      if (m > lo) bits &= (m - lo >= 32) ? 0u : ~((1u << (m - lo)) - 1);
    }
    uint32_t tot;
    const uint32_t ex = smx::block_excl_scan(__popc(bits), ws, tot);
    if (q < PC / 32) {
      wmask[q] = bits;
      wpre[q] = ex;
    }
  }
  __syncthreads();
  const uint64_t k0 = kb + pre_n;
  for (int p = m + tid; p < PC; p += P_THREADS) {
    const uint32_t bits = wmask[p >> 5];
    const int b = p & 31;
    if ((bits >> b) & 1u) emit<KIND>(J, k0 + wpre[p >> 5] + __popc(bits & ((1u << b) - 1u)), c, p, L[p], raw);
  }
}

// ---------------------------------------------------------------------------
// One-pass form of the same chain (opt-in, see run_chain): one CTA per chunk, chunks taken
// by ticket.  A chunk computes U, len and its entry->exit map exactly as
// chunk_kernel does, then publishes a 64-bit descriptor for its successors:
//   MAP  its exit when every entry offset leads to the same exit (orbits
//        merge inside the chunk: nearly always), so the successor knows its
//        entry without waiting for this chunk's entry;
//   AGG  its true entry is known: true exit and the samples started here;
//   INC  also the samples started in every earlier chunk (inclusive).
// Its true entry comes from the predecessor (MAP with a constant exit, or
// AGG / INC), its first sample index from a decoupled look-back over the
// predecessors' counts, and it emits its samples from its shared memory.
// Replaces chunk + group + across + within + emit (no len / s0 round trip).
// ---------------------------------------------------------------------------
constexpr uint64_t CD_STATE = 62, CD_CONST = 61, CD_EXIT = 48;
constexpr uint64_t CD_CNT_MASK = (1ULL << 48) - 1;
constexpr uint64_t CD_MAP = 1, CD_AGG = 2, CD_INC = 3;

__device__ __forceinline__ uint64_t ld_vol64(const uint64_t* p) { return *(const volatile uint64_t*)p; }

__global__ void __launch_bounds__(P_THREADS) chain_onepass_kernel(PoisJob J, uint64_t* desc, uint32_t* ticket) {
  __shared__ double U[PC + PE];
  __shared__ uint8_t L[PC + PE];
  __shared__ uint32_t S0[PC / 32];
  __shared__ uint32_t cnt0_pos[PC / 32 + 1];
  __shared__ int seg_exit[P_THREADS];
  __shared__ uint16_t M16[P_THREADS];
  __shared__ uint8_t exs[PE];
  __shared__ uint16_t cts[PE];
  __shared__ uint32_t ws[32];
  __shared__ int exit0, count0, s_c, s_entry, merge_p, pre_n;
  __shared__ unsigned long long s_kb;
  const int tid = threadIdx.x;
  if (tid == 0) s_c = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int c = s_c;
  const uint64_t cw = (*J.w0_dev & ~3ULL) + (uint64_t)c * PC;
  for (int q = tid; q < (PC + PE) / 4; q += P_THREADS) {
    uint64_t b[4];
    smx::philox4x64_10(((cw >> 2) + q) + 1, J.key, b);
#pragma unroll
    for (int i = 0; i < 4; ++i) U[4 * q + i] = J.kind == 1 ? __longlong_as_double((long long)b[i]) : smx::u53(b[i]);
  }
  __syncthreads();
  for (int w = tid; w < PC + PE; w += P_THREADS) {
    int k = 0;
    if (J.kind == 0) {
      double prod = 1.0;
      for (;;) {
        const int idx = w + k;
        const double u = idx < PC + PE ? U[idx] : smx::u53(smx::philox_word(J.key, cw + idx));
        prod = __dmul_rn(prod, u);
        ++k;
        if (!(prod > J.enlam)) break;
        if (k >= 255) break;
      }
    } else if (J.kind == 2) {
      for (;;) {
        const int i0 = w + k, i1 = w + k + 1;
        const double u = i0 < PC + PE ? U[i0] : smx::u53(smx::philox_word(J.key, cw + i0));
        const double v = i1 < PC + PE ? U[i1] : smx::u53(smx::philox_word(J.key, cw + i1));
        k += 2;
        long long cnt;
        if (ptrs_trial(J, u, v, cnt)) break;
        if (k >= 254) break;
      }
    } else {
      double x;
      if (smx::zig_first((uint64_t)__double_as_longlong(U[w]), x)) {
        k = 1;
      } else {
        smx::SeqStream st;
        st.init(J.key, cw + w);
        (void)smx::zig_standard_normal(st);
        const uint64_t used = st.word - (cw + w);
        k = used > 255 ? 255 : (int)used;
      }
    }
    if (k >= PE) atomicExch(J.err, 11);
    L[w] = (uint8_t)k;
  }
  __syncthreads();
  {  // orbit of starts from entry 0 (as chunk_kernel)
    constexpr int SEG = PC / P_THREADS;
    const int lo = SEG * tid, hi = lo + SEG;
    uint32_t mask = 0;
    int entry = lo, ex_ = lo;
    while (ex_ < hi) { mask |= 1u << (ex_ - lo); ex_ += L[ex_]; }
    seg_exit[tid] = ex_;
    for (;;) {
      __syncthreads();
      const int e_in = tid == 0 ? 0 : seg_exit[tid - 1];
      bool changed = false;
      if (e_in != entry) {
        entry = e_in;
        uint32_t m = 0;
        int p = e_in;
        while (p < hi && !((mask >> (p - lo)) & 1)) { m |= 1u << (p - lo); p += L[p]; }
        const int ex_new = p < hi ? ex_ : p;
        mask = p < hi ? (m | (mask & ~((1u << (p - lo)) - 1))) : m;
        changed = ex_new != ex_;
        ex_ = ex_new;
      }
      __syncthreads();
      seg_exit[tid] = ex_;
      if (!__syncthreads_or(changed)) break;
    }
    M16[tid] = (uint16_t)mask;
    __syncthreads();
    if (tid < PC / 32) S0[tid] = (uint32_t)M16[2 * tid] | ((uint32_t)M16[2 * tid + 1] << 16);
    __syncthreads();
    if (tid < 32) {
      const uint32_t a = __popc(S0[2 * tid]), b = __popc(S0[2 * tid + 1]);
      uint32_t x = a + b;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (tid >= o) x += y;
      }
      cnt0_pos[2 * tid] = x - a - b;
      cnt0_pos[2 * tid + 1] = x - b;
      if (tid == 31) { cnt0_pos[PC / 32] = x; count0 = (int)x; exit0 = seg_exit[P_THREADS - 1] - PC; }
    }
  }
  __syncthreads();
  for (int e = tid; e < PE; e += P_THREADS) {  // entry -> (exit, samples started here)
    int p = e, pre = 0, ex_ = -1, ct = 0;
    while (p < PC) {
      if ((S0[p >> 5] >> (p & 31)) & 1) {
        const int rank = cnt0_pos[p >> 5] + __popc(S0[p >> 5] & ((1u << (p & 31)) - 1));
        ex_ = exit0;
        ct = pre + (count0 - rank);
        break;
      }
      ++pre;
      p += L[p];
    }
    if (ex_ < 0) { ex_ = p - PC; ct = pre; }
    if (ex_ >= PE) { atomicExch(J.err, 12); ex_ = PE - 1; }
    exs[e] = (uint8_t)ex_;
    cts[e] = (uint16_t)ct;
  }
  __syncthreads();
  if (tid < 32) {  // warp 0: publish, take the entry, look back
    const int lane = tid;
    int entry = 0;
    uint64_t mine = 0, myexit = 0;
    if (lane == 0) {
      bool cons = true;
      for (int e = 1; e < PE; ++e) cons &= exs[e] == exs[0];
      // MAP: a constant exit lets the successor start without this chunk's entry
      __threadfence();
      *(volatile uint64_t*)(desc + c) = (CD_MAP << CD_STATE) | ((uint64_t)cons << CD_CONST) |
                                        ((uint64_t)exs[0] << CD_EXIT);
      // true entry: the predecessor's exit (constant map, or its true exit)
      if (c == 0) {
        entry = (int)(*J.w0_dev & 3);
      } else {
        uint64_t d;
        for (;;) {
          d = ld_vol64(desc + c - 1);
          const uint64_t s = d >> CD_STATE;
          if (s >= CD_AGG || (s == CD_MAP && ((d >> CD_CONST) & 1))) break;
          __nanosleep(32);
        }
        entry = (int)((d >> CD_EXIT) & 0xff);
      }
      mine = cts[entry];
      myexit = exs[entry];
      __threadfence();
      *(volatile uint64_t*)(desc + c) = (CD_AGG << CD_STATE) | (myexit << CD_EXIT) | mine;
    }
    // first sample index: warp-wide decoupled look-back, 32 descriptors per step
    uint64_t kb = 0;
    for (int q = c - 1; q >= 0;) {
      const int qi = q - lane;
      const uint64_t d = qi >= 0 ? ld_vol64(desc + qi) : (CD_INC << CD_STATE);
      const uint64_t s = d >> CD_STATE;
      const uint32_t inc = __ballot_sync(0xffffffffu, s == CD_INC);
      const uint32_t notyet = __ballot_sync(0xffffffffu, s < CD_AGG);
      const int first_inc = inc ? __ffs(inc) - 1 : 32;
      const int first_wait = notyet ? __ffs(notyet) - 1 : 32;
      if (first_wait < first_inc) {   // a predecessor before the nearest INC has no count yet
        if (first_wait > 0) {         // take the ready ones and move on
          uint64_t v = lane < first_wait ? (d & CD_CNT_MASK) : 0;
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          kb += v;
          q -= first_wait;
        } else {
          __nanosleep(32);
        }
        continue;
      }
      uint64_t v = (lane <= first_inc && qi >= 0) ? (d & CD_CNT_MASK) : 0;
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      kb += v;
      if (first_inc < 32) break;
      q -= 32;
    }
    if (lane == 0) {
      __threadfence();
      *(volatile uint64_t*)(desc + c) = (CD_INC << CD_STATE) | (myexit << CD_EXIT) | ((kb + mine) & CD_CNT_MASK);
      if (c == J.n_chunks - 1 && kb + mine < J.n) atomicExch(J.err, 13);  // window too small
      s_kb = kb;
      s_entry = entry;
    }
  }
  __syncthreads();
  const uint64_t kb = s_kb;
  if (kb >= J.n) return;
  const uint64_t* raw = reinterpret_cast<const uint64_t*>(U);   // kind 1: the words themselves
  if (tid == 0) {  // from the true entry to the merge with the entry-0 orbit
    int p = s_entry, pre = 0;
    while (p < PC && !((S0[p >> 5] >> (p & 31)) & 1)) {
      emit(J, kb + pre, c, p, L[p], raw);
      ++pre;
      p += L[p];
    }
    merge_p = p;
    pre_n = pre;
  }
  __syncthreads();
  const int m = merge_p;
  if (m >= PC) return;
  for (int q0 = 0; q0 < PC / 32; q0 += P_THREADS) {
    const int q = q0 + tid;
    uint32_t bits = 0;
    if (q < PC / 32) {
      bits = S0[q];
      const int lo = q * 32;
      if (m > lo) bits &= (m - lo >= 32) ? 0u : ~((1u << (m - lo)) - 1);
    }
    uint32_t tot;
    const uint32_t exq = smx::block_excl_scan(__popc(bits), ws, tot);
    uint64_t k = kb + pre_n + exq;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int p = q * 32 + b;
      emit(J, k, c, p, L[p], raw);
      ++k;
    }
  }
}

int launch_emit(const PoisJob& J, int n_chunks, cudaStream_t st) {
  smx_count_launch();
  if (J.kind == 0) {
    emit_kernel<0><<<n_chunks, P_THREADS, 0, st>>>(J);
  } else if (J.kind == 2) {
    emit_kernel<2><<<n_chunks, P_THREADS, 0, st>>>(J);
  } else {
    emit_kernel<1><<<n_chunks, P_THREADS, sizeof(uint64_t) * J_RAW_WORDS, st>>>(J);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}

// The chain on `ws`: the one-pass kernel when SMX_CHAIN_ONEPASS=1, else
// (default) the five kernels above.  Measured on B200 (C3 drive, C2
// weights): the one-pass form is exact but slower -- RTF 0.057 vs 0.040, C2
// 87 vs 69 ms -- its CTAs live through the entry wait, the look-back and the
// emission while the multi-kernel form keeps every phase fully parallel.
int run_chain(PoisJob& J, int n_chunks, void* ws, cudaStream_t st) {
  static const bool onepass = [] {
    const char* e = getenv("SMX_CHAIN_ONEPASS");
    return e && e[0] == '1';
  }();
  if (onepass) {
    uint64_t* desc = static_cast<uint64_t*>(ws);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(desc + n_chunks);
    SMX_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(uint64_t) * (n_chunks + 1), st));
    J.n_chunks = n_chunks;
    smx_count_launch(); chain_onepass_kernel<<<n_chunks, P_THREADS, 0, st>>>(J, desc, ticket);
    SMX_LAUNCH_CHECK();
    return 0;
  }
  return 1;   // caller runs the multi-kernel form
}

}  // namespace

// Workspace sizes for a window of n_chunks chunks (bytes).
extern "C" uint64_t smx_poisson_workspace(int n_chunks) {
  const int ng = (n_chunks + PG - 1) / PG;
  return (uint64_t)n_chunks * PC + (uint64_t)n_chunks * (PC / 32) * 4 + (uint64_t)n_chunks * PE * 3 +
         (uint64_t)ng * PE * 5 + (uint64_t)n_chunks * 9 + (uint64_t)ng * 9 + 256;
}

extern "C" int smx_poisson_chunks_for(uint64_t n, double lam) {
  // multiplication method: lam + 1 words per sample; PTRS (lam >= 10): two
  // words per trial, about 1.2 trials per sample
  const double per = lam >= 10.0 ? 3.0 : 1.0 + lam;
  const double words = (double)n * per + 10.0 * sqrt((double)n * per) + 2.0 * PC + PE;
  return (int)((words + PC - 1) / PC);
}

// counts[0..n) = numpy poisson(lam) samples drawn from the word cursor
// *cursor_in of stream (k0, k1); *cursor_out (a different word) receives the
// cursor after the last sample.  No host synchronisation.  `ws` is a device
// workspace of smx_poisson_workspace(n_chunks) bytes.
extern "C" int smx_poisson_counts(uint64_t k0, uint64_t k1, const uint64_t* cursor_in, double enlam, uint64_t n,
                                  int n_chunks, void* ws, uint8_t* counts, uint64_t* cursor_out, int* err,
                                  void* stream) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  PoisJob J;
  J.key = smx::Key{k0, k1};
  J.w0_dev = cursor_in;
  J.kind = 0;
  J.enlam = enlam;
  J.loc = J.scale = 0.0;
  J.n = n;
  J.n_chunks = n_chunks;
  const int ng = (n_chunks + PG - 1) / PG;
  uint8_t* p = (uint8_t*)ws;
  J.len = p; p += (size_t)n_chunks * PC;
  J.s0 = (uint32_t*)p; p += (size_t)n_chunks * (PC / 32) * 4;
  J.cnt = (uint16_t*)p; p += (size_t)n_chunks * PE * 2;
  J.gcnt = (uint32_t*)p; p += (size_t)ng * PE * 4;
  J.kbase = (uint64_t*)p; p += (size_t)n_chunks * 8;
  uint64_t* gbase = (uint64_t*)p; p += (size_t)ng * 8;
  J.ex = p; p += (size_t)n_chunks * PE;
  J.gex = p; p += (size_t)ng * PE;
  J.entry = p; p += (size_t)n_chunks;
  uint8_t* gentry = p; p += (size_t)ng;
  J.out = counts;
  J.cursor = cursor_out;
  J.err = err;
  if (const int rc = run_chain(J, n_chunks, ws, st); rc <= 0) return rc;
  smx_count_launch();
  if (J.kind == 0) chunk_kernel<0><<<n_chunks, P_THREADS, 0, st>>>(J);
  else if (J.kind == 2) chunk_kernel<2><<<n_chunks, P_THREADS, 0, st>>>(J);
  else chunk_kernel<1><<<n_chunks, P_THREADS, 0, st>>>(J);
  smx_count_launch(); group_kernel<<<ng, PE, 0, st>>>(J);
  smx_count_launch(); across_kernel<<<1, 256, 0, st>>>(J, ng, gentry, gbase);
  smx_count_launch(); within_kernel<<<ng, PE, 0, st>>>(J, gentry, gbase);
  if (const int rc = launch_emit(J, n_chunks, st); rc) return rc;
  SMX_LAUNCH_CHECK();
  return 0;
}

// counts[0..n) = numpy poisson(lam) samples for lam >= 10 (random_poisson_ptrs,
// two words per trial), same chain machinery and contract as smx_poisson_counts;
// counts above 255 raise the error flag (u8 counts).
extern "C" int smx_poisson_counts_ptrs(uint64_t k0, uint64_t k1, const uint64_t* cursor_in, double lam, uint64_t n,
                                       int n_chunks, void* ws, uint8_t* counts, uint64_t* cursor_out, int* err,
                                       void* stream) {
  if (n == 0) return 0;
  if (!(lam >= 10.0)) {
    smx_set_error("smx_poisson_counts_ptrs: lam %g < 10", lam);
    return -1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  PoisJob J;
  J.key = smx::Key{k0, k1};
  J.w0_dev = cursor_in;
  J.kind = 2;
  J.enlam = 0.0;
  J.loc = J.scale = 0.0;
  // the constants of random_poisson_ptrs, on the host like numpy's C code
  J.lam = lam;
  J.slam = sqrt(lam);
  J.loglam = log(lam);
  J.pb = 0.931 + 2.53 * J.slam;
  J.pa = -0.059 + 0.02483 * J.pb;
  J.invalpha = 1.1239 + 1.1328 / (J.pb - 3.4);
  J.vr = 0.9277 - 3.6224 / (J.pb - 2);
  J.n = n;
  J.n_chunks = n_chunks;
  const int ng = (n_chunks + PG - 1) / PG;
  uint8_t* p = (uint8_t*)ws;
  J.len = p; p += (size_t)n_chunks * PC;
  J.s0 = (uint32_t*)p; p += (size_t)n_chunks * (PC / 32) * 4;
  J.cnt = (uint16_t*)p; p += (size_t)n_chunks * PE * 2;
  J.gcnt = (uint32_t*)p; p += (size_t)ng * PE * 4;
  J.kbase = (uint64_t*)p; p += (size_t)n_chunks * 8;
  uint64_t* gbase = (uint64_t*)p; p += (size_t)ng * 8;
  J.ex = p; p += (size_t)n_chunks * PE;
  J.gex = p; p += (size_t)ng * PE;
  J.entry = p; p += (size_t)n_chunks;
  uint8_t* gentry = p; p += (size_t)ng;
  J.out = counts;
  J.cursor = cursor_out;
  J.err = err;
  if (const int rc = run_chain(J, n_chunks, ws, st); rc <= 0) return rc;
  smx_count_launch();
  if (J.kind == 0) chunk_kernel<0><<<n_chunks, P_THREADS, 0, st>>>(J);
  else if (J.kind == 2) chunk_kernel<2><<<n_chunks, P_THREADS, 0, st>>>(J);
  else chunk_kernel<1><<<n_chunks, P_THREADS, 0, st>>>(J);
  smx_count_launch(); group_kernel<<<ng, PE, 0, st>>>(J);
  smx_count_launch(); across_kernel<<<1, 256, 0, st>>>(J, ng, gentry, gbase);
  smx_count_launch(); within_kernel<<<ng, PE, 0, st>>>(J, gentry, gbase);
  if (const int rc = launch_emit(J, n_chunks, st); rc) return rc;
  SMX_LAUNCH_CHECK();
  return 0;
}

// values[0..n) = numpy Generator.normal(loc, scale, size=n) drawn from the
// word cursor *cursor_in (the ziggurat consumes a variable number of words per
// sample: the same chunked chain + composition as the Poisson counts).
extern "C" int smx_normal_fill(uint64_t k0, uint64_t k1, const uint64_t* cursor_in, double loc, double scale,
                               uint64_t n, int n_chunks, void* ws, double* values, uint64_t* cursor_out, int* err,
                               void* stream) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  PoisJob J;
  J.key = smx::Key{k0, k1};
  J.w0_dev = cursor_in;
  J.kind = 1;
  J.enlam = 0.0;
  J.loc = loc;
  J.scale = scale;
  J.n = n;
  J.n_chunks = n_chunks;
  const int ng = (n_chunks + PG - 1) / PG;
  uint8_t* p = (uint8_t*)ws;
  J.len = p; p += (size_t)n_chunks * PC;
  J.s0 = (uint32_t*)p; p += (size_t)n_chunks * (PC / 32) * 4;
  J.cnt = (uint16_t*)p; p += (size_t)n_chunks * PE * 2;
  J.gcnt = (uint32_t*)p; p += (size_t)ng * PE * 4;
  J.kbase = (uint64_t*)p; p += (size_t)n_chunks * 8;
  uint64_t* gbase = (uint64_t*)p; p += (size_t)ng * 8;
  J.ex = p; p += (size_t)n_chunks * PE;
  J.gex = p; p += (size_t)ng * PE;
  J.entry = p; p += (size_t)n_chunks;
  uint8_t* gentry = p; p += (size_t)ng;
  J.out = values;
  J.cursor = cursor_out;
  J.err = err;
  if (const int rc = run_chain(J, n_chunks, ws, st); rc <= 0) return rc;
  smx_count_launch();
  if (J.kind == 0) chunk_kernel<0><<<n_chunks, P_THREADS, 0, st>>>(J);
  else if (J.kind == 2) chunk_kernel<2><<<n_chunks, P_THREADS, 0, st>>>(J);
  else chunk_kernel<1><<<n_chunks, P_THREADS, 0, st>>>(J);
  smx_count_launch(); group_kernel<<<ng, PE, 0, st>>>(J);
  smx_count_launch(); across_kernel<<<1, 256, 0, st>>>(J, ng, gentry, gbase);
  smx_count_launch(); within_kernel<<<ng, PE, 0, st>>>(J, gentry, gbase);
  if (const int rc = launch_emit(J, n_chunks, st); rc) return rc;
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_normal_chunks_for(uint64_t n) {
  // 1.015 words per sample on average (slow path ~1.5%), wide margin
  const double words = (double)n * 1.1 + 16.0 * sqrt((double)n + 1.0) + 2.0 * PC + PE;
  return (int)((words + PC - 1) / PC);
}
