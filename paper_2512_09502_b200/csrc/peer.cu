// Spike exchange over NVLink peer memory (one process per GPU, one node).
//
// The reference's synchronous rounds (LockstepTransport.exchange_allgather /
// exchange_point_to_point, sm/transport.py:92-168) move, per round, one
// packet [count | (position, step) pairs] from every rank to every receiver.
// Here each receiver owns a receive area in its HBM that every sender maps
// through CUDA IPC.  Per exchange block:
//   peer_send  one CTA per (destination, source buffer): copies the occupied
//              part of the packet (count + 2 * count words) straight into the
//              destination's slot for this rank over NVLink, fences at system
//              scope and publishes the block's sequence number in the slot's
//              flag;
//   peer_wait  spins until every expected flag carries the sequence number,
//              then copies each slot into the fixed receive blocks the unpack
//              kernels read and advances the sequence.
// No NCCL launch, no padding (only occupied packets travel), no host step:
// both kernels are captured in the block's CUDA graph.  Slots alternate
// between two parities so a fast sender never overwrites a block the
// receiver has not copied yet (a sender reaches block b + 2 only after this
// receiver's block b + 1 data, sent after its block b copy).
#include <cstring>
#include "common.cuh"

namespace {

constexpr int PEER_MAX = 64;  // sends / slots per launch

struct PeerSend {
  const uint32_t* count;  // sender's packet count (device)
  const uint32_t* packets;  // sender's packets, 2 words each
  uint32_t* slot[2];      // receiver's slot per parity (mapped): [count, 0, packets...]
  unsigned long long* flag[2];  // receiver's flag per parity (mapped)
  uint32_t cap;           // packets per slot
};

struct PeerSendArgs {
  int n;
  PeerSend s[PEER_MAX];
};

struct PeerSlot {
  const uint32_t* slot[2];              // local slot per parity
  const unsigned long long* flag[2];    // local flag per parity
  uint32_t* out;                        // fixed receive block [count, 0, packets...]
  uint32_t cap;
};

struct PeerWaitArgs {
  int n;
  PeerSlot s[PEER_MAX];
};

__global__ void peer_send_kernel(const __grid_constant__ PeerSendArgs A, const unsigned long long* seq) {
  const PeerSend& P = A.s[blockIdx.x];
  const unsigned long long s = *seq + 1;
  const int par = (int)(s & 1);
  uint32_t n = *P.count;
  if (n > P.cap) n = P.cap;  // over-full blocks are flagged by the engine's capacity check
  uint32_t* dst = P.slot[par];
  const uint32_t words = 2 * n;
  if ((reinterpret_cast<uintptr_t>(P.packets) & 15) == 0) {  // 16-byte NVLink stores
    const uint4* src4 = reinterpret_cast<const uint4*>(P.packets);
    uint4* dst4 = reinterpret_cast<uint4*>(dst + 4);  // packets start 16-byte aligned at word 4
    for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x) dst4[i] = src4[i];
    for (uint32_t i = (words / 4) * 4 + threadIdx.x; i < words; i += blockDim.x) dst[4 + i] = P.packets[i];
  } else {
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[4 + i] = P.packets[i];
  }
  if (threadIdx.x == 0) dst[0] = n;
  __threadfence_system();  // every thread's stores reach the peer before the flag
  __syncthreads();
  if (threadIdx.x == 0) *(volatile unsigned long long*)P.flag[par] = s;
}

__global__ void peer_wait_kernel(const __grid_constant__ PeerWaitArgs A, unsigned long long* seq) {
  const PeerSlot& P = A.s[blockIdx.x];
  const unsigned long long s = *seq + 1;
  const int par = (int)(s & 1);
  __shared__ uint32_t n;
  if (threadIdx.x == 0) {
    while (*(volatile const unsigned long long*)P.flag[par] != s) __nanosleep(100);
    __threadfence_system();
    n = *(volatile const uint32_t*)P.slot[par];
  }
  __syncthreads();
  const uint32_t* src = P.slot[par];
  const uint32_t words = 2 * n;
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) P.out[2 + i] = ((volatile const uint32_t*)src)[4 + i];
  if (threadIdx.x == 0) {
    P.out[0] = n;
    P.out[1] = 0;
  }
}

__global__ void peer_advance_kernel(unsigned long long* seq) { *seq += 1; }

}  // namespace

// Receive area in this process: cudaMalloc'd (IPC-exportable), zeroed.
extern "C" int smx_peer_alloc(uint64_t bytes, void** ptr) {
  SMX_CUDA_CHECK(cudaMalloc(ptr, bytes ? bytes : 16));
  SMX_CUDA_CHECK(cudaMemset(*ptr, 0, bytes ? bytes : 16));
  return 0;
}

extern "C" int smx_peer_free(void* ptr) {
  SMX_CUDA_CHECK(cudaFree(ptr));
  return 0;
}

// 64-byte IPC handle of an allocation made by smx_peer_alloc.
extern "C" int smx_peer_handle(void* ptr, void* handle_out) {
  cudaIpcMemHandle_t h;
  SMX_CUDA_CHECK(cudaIpcGetMemHandle(&h, ptr));
  memcpy(handle_out, &h, sizeof(h));
  return 0;
}

// Maps a peer's receive area into this process (NVLink peer access).
extern "C" int smx_peer_open(const void* handle, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SMX_CUDA_CHECK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

extern "C" int smx_peer_close(void* ptr) {
  SMX_CUDA_CHECK(cudaIpcCloseMemHandle(ptr));
  return 0;
}

// One exchange round: sends (host array of n_send descriptors, laid out as
// PeerSend), then waits for n_slot incoming slots (PeerSlot) and copies them
// into their fixed receive blocks; *seq (device) advances by one.
extern "C" int smx_peer_exchange(const void* sends_host, int n_send, const void* slots_host, int n_slot,
                                 unsigned long long* seq, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_send > PEER_MAX || n_slot > PEER_MAX) {
    smx_set_error("smx_peer_exchange: at most %d sends / slots", PEER_MAX);
    return -1;
  }
  if (n_send) {
    PeerSendArgs A;
    A.n = n_send;
    memcpy(A.s, sends_host, sizeof(PeerSend) * n_send);
    smx_count_launch(); peer_send_kernel<<<n_send, 256, 0, st>>>(A, seq);
  }
  if (n_slot) {
    PeerWaitArgs W;
    W.n = n_slot;
    memcpy(W.s, slots_host, sizeof(PeerSlot) * n_slot);
    smx_count_launch(); peer_wait_kernel<<<n_slot, 256, 0, st>>>(W, seq);
  }
  smx_count_launch(); peer_advance_kernel<<<1, 1, 0, st>>>(seq);
  SMX_LAUNCH_CHECK();
  return 0;
}
