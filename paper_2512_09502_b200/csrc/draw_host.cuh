// Host driver for the ordered Lemire draw engine (draw.cuh).
#pragma once
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include "draw.cuh"

namespace smx {

struct DrawResult {
  uint64_t cursor;  // u32 cursor after the last consumed draw
};

template <class Sink, int MARK>
int launch_write(int G, size_t smem, cudaStream_t st, const DrawRange& r, const uint64_t* offs, uint64_t n_out,
                 const Sink& sink, uint64_t* cur_d, const DrawMark& mk) {
  static unsigned long long configured = 0;   // one bit per device
  const unsigned long long dbit = smx_device_bit();
  if (smem > 0 && !(configured & dbit)) {  // static (staging) + dynamic (bitmap) may exceed the 48 KB default
    SMX_CUDA_CHECK(cudaFuncSetAttribute(draw_write_kernel<Sink, MARK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(DRAW_MARK_SMEM_WORDS * 4)));
    configured |= dbit;
  }
  smx_count_launch(); draw_write_kernel<Sink, MARK><<<G, DRAW_THREADS, smem, st>>>(r, offs, n_out, sink, cur_d, mk);
  return 0;
}

template <class Sink, int MARK>
int launch_op(int G, size_t smem, cudaStream_t st, const DrawRange& r, uint32_t tile, uint32_t n_tiles,
              uint64_t* desc, uint32_t* ticket, uint64_t* total_d, uint64_t n_out, const Sink& sink, uint64_t* cur_d,
              const DrawMark& mk) {
  static size_t configured[64] = {};   // per device: the largest limit set so far
  int dev = 0;
  cudaGetDevice(&dev);
  smem += (size_t)DRAW_WARPS * tile * 4;
  if (smem > 48 * 1024 && smem > configured[dev & 63]) {
    SMX_CUDA_CHECK(cudaFuncSetAttribute(draw_onepass_kernel<Sink, MARK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    configured[dev & 63] = smem;
  }
  smx_count_launch();
  draw_onepass_kernel<Sink, MARK><<<G, DRAW_THREADS, smem, st>>>(r, tile, n_tiles, desc, ticket, total_d, n_out,
                                                                  sink, cur_d, mk);
  return 0;
}

// Sinks that may mark used values say so with `static constexpr bool kMark`.
template <class Sink, class = void>
struct sink_marks { static constexpr bool value = false; };
template <class Sink>
struct sink_marks<Sink, decltype((void)Sink::kMark, void())> { static constexpr bool value = Sink::kMark; };

template <class Sink>
int launch_draw_write(int mode, int G, size_t smem, cudaStream_t st, const DrawRange& r, const uint64_t* offs,
                      uint64_t n_out, const Sink& sink, uint64_t* cur_d, const DrawMark& mk) {
  if constexpr (sink_marks<Sink>::value) {
    if (mode == 1) return launch_write<Sink, 1>(G, smem, st, r, offs, n_out, sink, cur_d, mk);
    if (mode == 2) return launch_write<Sink, 2>(G, smem, st, r, offs, n_out, sink, cur_d, mk);
  } else if (mode != 0) {
    smx_set_error("run_draw: this sink does not mark used values");
    return -1;
  }
  return launch_write<Sink, 0>(G, smem, st, r, offs, n_out, sink, cur_d, mk);
}

template <class Sink>
int launch_onepass(int mode, int G, size_t smem, cudaStream_t st, const DrawRange& r, uint32_t tile, uint32_t n_tiles,
                   uint64_t* desc, uint32_t* ticket, uint64_t* total_d, uint64_t n_out, const Sink& sink,
                   uint64_t* cur_d, const DrawMark& mk) {
  if constexpr (sink_marks<Sink>::value) {
    if (mode == 1) return launch_op<Sink, 1>(G, smem, st, r, tile, n_tiles, desc, ticket, total_d, n_out, sink, cur_d, mk);
    if (mode == 2) return launch_op<Sink, 2>(G, smem, st, r, tile, n_tiles, desc, ticket, total_d, n_out, sink, cur_d, mk);
  } else if (mode != 0) {
    smx_set_error("run_draw: this sink does not mark used values");
    return -1;
  }
  return launch_op<Sink, 0>(G, smem, st, r, tile, n_tiles, desc, ticket, total_d, n_out, sink, cur_d, mk);
}

// numpy integers(lo, lo+ex, size=n) on stream `key` from u32 cursor u0.
// Hands every (index, value-lo) to `sink`; returns 0 or a negative status.
template <class Sink>
int run_draw(Key key, uint64_t u0, uint64_t ex, uint64_t n_out, const Sink& sink,
             cudaStream_t st, DrawResult* res, DrawMark mk = DrawMark{nullptr, nullptr, 0, 0, 0, 0, 0}) {
  // device-side chaining (smx_draw_chain): start at *u0_dev, end cursor to
  // *cursor_dev, no host readback
  const uint64_t* u0_dev = nullptr;
  uint64_t* cursor_dev = nullptr;
  smx_take_draw_chain(&u0_dev, &cursor_dev);
  if (u0_dev || cursor_dev) res = nullptr;
  if (res) res->cursor = u0;
  if (n_out == 0) return smx_chain_passthrough(u0_dev, u0, cursor_dev, st);
  if (ex == 1) {  // numpy: range of one value consumes nothing
    smx_set_error("run_draw: ex == 1 must be handled by the caller");
    return -1;
  }
  if (ex < 1 || ex > (1ULL << 32)) {
    smx_set_error("integer range %llu outside [2, 2^32]", (unsigned long long)ex);
    return -1;
  }
  DrawRange r;
  r.key = key;
  r.u0 = u0;
  r.u0_dev = u0_dev;
  const bool async = res == nullptr;  // no cursor wanted: no host readback at all
  static const bool onepass_env = [] {
    const char* e = getenv("SMX_DRAW_ONEPASS");
    return !(e && e[0] == '0');
  }();
  if ((u0_dev || cursor_dev) && !onepass_env) {
    smx_set_error("run_draw: chained draws need the one-pass kernel");
    return -1;
  }
  r.lm.ex = (uint32_t)(ex & 0xffffffffULL);
  r.lm.threshold = ex == (1ULL << 32) ? 0u : (uint32_t)(((1ULL << 32) - ex) % ex);
  const double prej = (double)r.lm.threshold / 4294967296.0;
  uint64_t n_raw = n_out + (uint64_t)std::ceil(n_out * prej * 1.25 + 12.0 * std::sqrt(n_out * prej + 1.0) + 64.0);
  // test aid: start synchronous calls from a window of exactly n_out raw
  // positions, so any rejection exercises the widen-and-retry path
  static const bool short_window = getenv("SMX_DRAW_SHORT_WINDOW") != nullptr;
  if (short_window && res) n_raw = n_out;
  static const bool timing = getenv("SMX_DRAW_TIMING") != nullptr;  // tuning aid
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t_start = timing ? now_us() : 0.0;
  double t_count = 0.0;
  uint32_t* counts = nullptr;
  uint64_t* offs = nullptr;
  uint64_t* cur_d = nullptr;
  int rc = 0;
  static const bool onepass = [] {
    const char* e = getenv("SMX_DRAW_ONEPASS");
    return !(e && e[0] == '0');
  }();
  if (onepass) {
    mk.in_smem = mk.bits && mk.nwords <= DRAW_MARK_SMEM_WORDS;
    const size_t smem = mk.in_smem ? mk.nwords * 4 : 0;
    const int mode = mk.bits ? (mk.from_key ? 1 : 2) : 0;
    static const uint32_t tile = [] {  // tuning aid: SMX_DRAW_TILE_RT overrides the tile size
      const char* e = getenv("SMX_DRAW_TILE_RT");
      const long v = e ? atol(e) : 0;
      return v >= 256 && v % 256 == 0 && v <= 4096 ? (uint32_t)v : (uint32_t)OP_TILE;
    }();
    for (int attempt = 0; attempt < 8; ++attempt) {
      const uint64_t n_tiles = (n_raw + tile - 1) / tile;
      if (n_tiles >= 0xffffffffull) {
        smx_set_error("run_draw: %llu raw positions exceed the tile ticket range", (unsigned long long)n_raw);
        return -1;
      }
      r.n_raw = n_raw;
      r.per_warp = 0;
      // while pass A runs, the SMX_FG_FREE_SMS * 2 CTA slots it leaves
      const int G = smx_grid_cap((int)std::max<uint64_t>(1, std::min<uint64_t>((n_tiles + DRAW_WARPS - 1) / DRAW_WARPS,
                                                                   148 * SMX_DRAW_MIN_BLOCKS)),
                                  std::max(1, smx_pass_a_free_slots()));
      // [desc n_tiles][ticket][total][cursor]
      uint64_t* ws = nullptr;
      SMX_CUDA_CHECK(cudaMallocAsync((void**)&ws, sizeof(uint64_t) * (n_tiles + 3), st));
      SMX_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(uint64_t) * (n_tiles + 2), st));
      uint32_t* ticket = reinterpret_cast<uint32_t*>(ws + n_tiles);
      uint64_t* total_d = ws + n_tiles + 1;
      uint64_t* cur_p = cursor_dev ? cursor_dev : async ? nullptr : ws + n_tiles + 2;
      if (int rc2 = launch_onepass(mode, G, smem, st, r, tile, (uint32_t)n_tiles, ws, ticket, total_d, n_out, sink, cur_p, mk))
        return rc2;
      SMX_LAUNCH_CHECK();
      if (async) {
        int* err = smx_device_error_word();
        if (!err) {
          smx_set_error("run_draw: no device error word");
          return -3;
        }
        smx_count_launch(); draw_window_check_kernel<<<1, 1, 0, st>>>(total_d, n_out, err);
        cudaFreeAsync(ws, st);
        return 0;
      }
      uint64_t tc[2] = {0, 0};
      SMX_CUDA_CHECK(cudaMemcpyAsync(tc, total_d, sizeof(tc), cudaMemcpyDeviceToHost, st));
      SMX_CUDA_CHECK(cudaStreamSynchronize(st));
      cudaFreeAsync(ws, st);
      if (timing) fprintf(stderr, "run_draw onepass n=%llu G=%d: %.0f us\n", (unsigned long long)n_out, G, now_us() - t_start);
      if (tc[0] >= n_out) {
        res->cursor = tc[1];
        return 0;
      }
      n_raw = n_raw + n_raw / 2 + 1024;
    }
    smx_set_error("run_draw: could not cover %llu accepted draws", (unsigned long long)n_out);
    return -3;
  }
  for (int attempt = 0; attempt < 8; ++attempt) {
    int G = (int)std::min<uint64_t>((n_raw + 16383) / 16384, 148 * 8);
    if (G < 1) G = 1;
    const int NW = G * DRAW_WARPS;
    r.n_raw = n_raw;
    r.per_warp = ((n_raw + NW - 1) / NW + 7) / 8 * 8;
    SMX_CUDA_CHECK(cudaMallocAsync((void**)&counts, sizeof(uint32_t) * NW, st));
    SMX_CUDA_CHECK(cudaMallocAsync((void**)&offs, sizeof(uint64_t) * (NW + 1), st));
    SMX_CUDA_CHECK(cudaMallocAsync((void**)&cur_d, sizeof(uint64_t), st));
    smx_count_launch(); draw_count_kernel<<<G, DRAW_THREADS, 0, st>>>(r, counts);
    smx_count_launch(); cta_offsets_kernel<<<1, 1024, 0, st>>>(counts, NW, offs);
    SMX_LAUNCH_CHECK();
    if (async) {
      // the window covers n_out accepted draws by 12 sigma; a short window is
      // flagged on the device (smx_check_device_errors) instead of retried
      int* err = smx_device_error_word();
      if (!err) {
        smx_set_error("run_draw: no device error word");
        return -3;
      }
      smx_count_launch(); draw_window_check_kernel<<<1, 1, 0, st>>>(offs + NW, n_out, err);
      mk.in_smem = mk.bits && mk.nwords <= DRAW_MARK_SMEM_WORDS;
      const size_t smem = mk.in_smem ? mk.nwords * 4 : 0;
      const int mode = mk.bits ? (mk.from_key ? 1 : 2) : 0;
      if (int rc2 = launch_draw_write(mode, G, smem, st, r, offs, n_out, sink, nullptr, mk)) return rc2;
      SMX_LAUNCH_CHECK();
      cudaFreeAsync(counts, st);
      cudaFreeAsync(offs, st);
      cudaFreeAsync(cur_d, st);
      return 0;
    }
    uint64_t total = 0;
    SMX_CUDA_CHECK(cudaMemcpyAsync(&total, offs + NW, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SMX_CUDA_CHECK(cudaStreamSynchronize(st));
    if (timing) t_count = now_us();
    if (total >= n_out) {
      mk.in_smem = mk.bits && mk.nwords <= DRAW_MARK_SMEM_WORDS;
      const size_t smem = mk.in_smem ? mk.nwords * 4 : 0;
      const int mode = mk.bits ? (mk.from_key ? 1 : 2) : 0;
      if (rc = launch_draw_write(mode, G, smem, st, r, offs, n_out, sink, cur_d, mk); rc) return rc;
      SMX_LAUNCH_CHECK();
      SMX_CUDA_CHECK(cudaMemcpyAsync(&res->cursor, cur_d, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      SMX_CUDA_CHECK(cudaStreamSynchronize(st));
      if (timing)
        fprintf(stderr, "run_draw n=%llu G=%d: count+sync %.0f us, write+sync %.0f us\n", (unsigned long long)n_out, G,
                t_count - t_start, now_us() - t_count);
      rc = 0;
    } else {
      rc = 1;
    }
    cudaFreeAsync(counts, st);
    cudaFreeAsync(offs, st);
    cudaFreeAsync(cur_d, st);
    if (rc == 0) return 0;
    n_raw = n_raw + n_raw / 2 + 1024;
  }
  smx_set_error("run_draw: could not cover %llu accepted draws", (unsigned long long)n_out);
  return -3;
}

}  // namespace smx
