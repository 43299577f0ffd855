// C-ABI plumbing: error strings and library identity.
// Status codes (include/spikemesh_b200.h): 0 ok, -1 ValueError, -2
// ConsistencyError, -3 CUDA error, -4 ProtocolError, -5 DelayRangeError --
// the reference's exception classes (sm/core.py:39-52).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <vector>

#include "common.cuh"

static thread_local char g_err[1024] = {0};
static std::atomic<uint64_t> g_launches{0};

// Every kernel launch of the library bumps this counter (bench.py reports
// the launches inside its timed region from it).
extern "C" void smx_count_launch(void) { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" uint64_t smx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" void smx_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" int smx_last_error(char* buf, size_t cap) {
  if (!buf || cap == 0) return (int)strlen(g_err);
  strncpy(buf, g_err, cap - 1);
  buf[cap - 1] = 0;
  return (int)strlen(buf);
}

// Host -> device copy of a small host array without the pageable-copy
// semantics (a pageable cudaMemcpyAsync first waits for the stream to drain,
// blocking the host behind every queued kernel): the bytes are staged in a
// pinned block that is reused once its previous copy has completed.
namespace {
struct Staging {
  char* p;
  size_t cap;
  cudaEvent_t ev;
  int device;
};
std::mutex g_stage_mu;
std::vector<Staging> g_stage;
}  // namespace

int smx_h2d_async(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return 0;
  int dev = 0;
  SMX_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_stage_mu);
  Staging* s = nullptr;
  for (auto& b : g_stage)
    if (b.device == dev && b.cap >= bytes && cudaEventQuery(b.ev) == cudaSuccess) {
      s = &b;
      break;
    }
  if (!s) {
    Staging b{nullptr, bytes < (64u << 10) ? (size_t)(64u << 10) : bytes, nullptr, dev};
    SMX_CUDA_CHECK(cudaHostAlloc((void**)&b.p, b.cap, cudaHostAllocPortable));
    SMX_CUDA_CHECK(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
    g_stage.push_back(b);
    s = &g_stage.back();
  }
  memcpy(s->p, src, bytes);
  SMX_CUDA_CHECK(cudaMemcpyAsync(dst, s->p, bytes, cudaMemcpyHostToDevice, st));
  SMX_CUDA_CHECK(cudaEventRecord(s->ev, st));
  return 0;
}

// Long-kernel tracking: pass A (fused.cu) keeps all but a few CTA slots of
// the GPU for its whole run.  A kernel launched on another stream meanwhile
// only completes once every one of its CTAs has been placed, so the ticketed
// draw kernels launched while pass A is in flight use a grid that fits the
// free slots (their tiles are taken by ticket: any grid size is correct).
namespace {
constexpr int MAX_DEVICES = 64;
cudaEvent_t g_long_ev[MAX_DEVICES] = {};
}  // namespace

void smx_long_kernel_mark(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= MAX_DEVICES) return;
  if (!g_long_ev[dev] && cudaEventCreateWithFlags(&g_long_ev[dev], cudaEventDisableTiming) != cudaSuccess) {
    g_long_ev[dev] = nullptr;
    return;
  }
  cudaEventRecord(g_long_ev[dev], st);
}

int smx_grid_cap(int grid, int concurrent_cap) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= MAX_DEVICES || !g_long_ev[dev]) return grid;
  if (cudaEventQuery(g_long_ev[dev]) != cudaErrorNotReady) return grid;
  return grid < concurrent_cap ? grid : concurrent_cap;
}

// Device-side chaining of draws on one stream (a draw that continues where
// the previous one ended, e.g. fixed_total's targets after its positions, or
// a syn stream's delays after its normal weights): smx_draw_chain sets, for
// the next draw entry point called on this thread, where its start cursor
// comes from and where its end cursor goes -- both device words, no host
// synchronisation.  run_draw takes (and clears) the setting.
namespace {
thread_local const uint64_t* t_chain_u0 = nullptr;
thread_local uint64_t* t_chain_cur = nullptr;

__global__ void chain_copy_kernel(const uint64_t* u0_dev, uint64_t u0, uint64_t* cursor_dev) {
  *cursor_dev = u0_dev ? *u0_dev : u0;
}
}  // namespace

extern "C" int smx_draw_chain(const uint64_t* u0_dev, uint64_t* cursor_dev) {
  t_chain_u0 = u0_dev;
  t_chain_cur = cursor_dev;
  return 0;
}

void smx_take_draw_chain(const uint64_t** u0_dev, uint64_t** cursor_dev) {
  *u0_dev = t_chain_u0;
  *cursor_dev = t_chain_cur;
  t_chain_u0 = nullptr;
  t_chain_cur = nullptr;
}

int smx_chain_passthrough(const uint64_t* u0_dev, uint64_t u0, uint64_t* cursor_dev, cudaStream_t st) {
  if (!cursor_dev) return 0;
  smx_count_launch(); chain_copy_kernel<<<1, 1, 0, st>>>(u0_dev, u0, cursor_dev);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" const char* smx_version(void) { return "spikemesh-b200 0.1.0 sm_100a"; }

// Host-thread wait policy for synchronisations (must run before the CUDA
// context is created): 1 = spin, 2 = yield, 4 = blocking sync.
extern "C" int smx_set_sync_policy(int flags) {
  cudaError_t e = cudaSetDeviceFlags((unsigned)flags);
  if (e != cudaSuccess) {
    smx_set_error("cudaSetDeviceFlags: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

// Keep the stream-ordered allocator's freed memory mapped between calls
// (release threshold = max): without it every synchronisation trims the
// default pool and the next cudaMallocAsync re-maps physical pages.
// A stream that does not synchronise with the legacy default stream (the one
// torch's default stream is): work on it runs beside the default stream's
// kernels instead of serialising with them.
extern "C" int smx_stream_create(int priority, void** out) {
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority);
  if (e != cudaSuccess) {
    smx_set_error("stream create: %s", cudaGetErrorString(e));
    return -3;
  }
  *out = (void*)s;
  return 0;
}

extern "C" int smx_pool_setup(int device) {
  cudaMemPool_t pool;
  cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
  if (e == cudaSuccess) {
    uint64_t thr = ~0ULL;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (e == cudaSuccess) {
    // no reuse through inserted dependencies: a block freed on the
    // generation stream behind a long pass-A kernel would otherwise be
    // handed to an allocation on another stream together with a wait on that
    // kernel, serialising the streams (opportunistic reuse of blocks whose
    // free has completed stays on)
    int no = 0;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
  if (e != cudaSuccess) {
    smx_set_error("mempool setup: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

extern "C" int smx_stream_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    smx_set_error("stream sync: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

// Device-side error word per device (asynchronous paths that cannot return a
// status at launch time, e.g. a draw window found short on the device).
static int* g_dev_err[64] = {nullptr};

extern "C" int* smx_device_error_word(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  int*& p = g_dev_err[dev & 63];
  if (!p) {
    if (cudaMalloc((void**)&p, sizeof(int)) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, sizeof(int)) != cudaSuccess) return nullptr;
  }
  return p;
}

// Reads and clears the device error word of the current device (synchronises
// the stream); 0 = no error.
extern "C" int smx_check_device_errors(void* stream) {
  int* p = smx_device_error_word();
  if (!p) {
    smx_set_error("smx_check_device_errors: no device error word");
    return -3;
  }
  int v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, p, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    smx_set_error("smx_check_device_errors: %s", cudaGetErrorString(e));
    return -3;
  }
  if (v) {
    cudaMemsetAsync(p, 0, sizeof(int), (cudaStream_t)stream);
    smx_set_error("device error %d (1: a draw window was short of accepted draws, 3: a connection target that is "
                  "not a real neuron of its rank)", v);
    return -2;
  }
  return 0;
}
