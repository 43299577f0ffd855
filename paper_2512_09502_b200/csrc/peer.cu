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
//              then unpacks each slot in place: map / roster position ->
//              image node through the slot's lookup table (L or I, -1
//              skipped), appended to the delivery source list; the last CTA
//              advances the sequence.  The capacity check and the byte
//              counter of the round ride along in peer_send.
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
  uint32_t* slot[2];      // receiver's slot per parity (mapped): [count, 0, 0, 0, packets...]
  unsigned long long* flag[2];  // receiver's flag per parity (mapped)
  uint32_t cap;           // packets per slot
  int account;            // this descriptor adds the buffer's count to the byte counter
};

struct PeerSendArgs {
  int n;
  unsigned long long* sent;  // packets put on the wire (TransportStats bytes / 8)
  int* over;                 // set when a buffer exceeds its capacity
  uint32_t* n_src;           // delivery list length, reset for this round's unpack
  PeerSend s[PEER_MAX];
};

struct PeerSlot {
  const uint32_t* slot[2];              // local slot per parity
  const unsigned long long* flag[2];    // local flag per parity
  const int64_t* table;                 // position -> image node (-1: not an image here)
  uint64_t table_len;
  uint32_t cap;
};

struct PeerWaitArgs {
  int n;
  uint32_t* src_nodes;
  uint32_t* src_steps;
  uint32_t* n_src;
  uint32_t src_cap;
  int* err;
  unsigned int* done;     // CTA counter: the last one advances the sequence
  uint32_t* zero[2];      // the senders' packet counts, cleared for the next block
  uint32_t nzero[2];
  PeerSlot s[PEER_MAX];
};

__global__ void peer_send_kernel(const __grid_constant__ PeerSendArgs A, const unsigned long long* seq) {
  const PeerSend& P = A.s[blockIdx.x];
  const unsigned long long s = *seq + 1;
  const int par = (int)(s & 1);
  uint32_t n = *P.count;
  if (threadIdx.x == 0) {
    if (n > P.cap) atomicExch(A.over, 1);
    if (P.account) atomicAdd(A.sent, (unsigned long long)n);
    if (blockIdx.x == 0) *A.n_src = 0;
  }
  if (n > P.cap) n = P.cap;
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
    while (*(volatile const unsigned long long*)P.flag[par] != s) __nanosleep(64);
    __threadfence_system();
    n = *(volatile const uint32_t*)P.slot[par];
    if (n > P.cap) { atomicExch(A.err, 5); n = P.cap; }
    if (P.table == nullptr) n = 0;  // no lookup for this source here: nothing to deliver
  }
  __syncthreads();
  if (blockIdx.x == 0) {  // the sends of this round are complete (stream order)
    for (int z = 0; z < 2; ++z)
      for (uint32_t i = threadIdx.x; i < A.nzero[z]; i += blockDim.x) A.zero[z][i] = 0;
  }
  const volatile uint32_t* src = P.slot[par] + 4;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {  // unpack (smx_unpack) in place
    const uint32_t p = src[2 * i];
    if (p >= P.table_len) { atomicExch(A.err, 4); continue; }
    const int64_t img = P.table[p];
    if (img < 0) continue;
    const uint32_t k = atomicAdd(A.n_src, 1u);
    if (k < A.src_cap) { A.src_nodes[k] = (uint32_t)img; A.src_steps[k] = src[2 * i + 1]; }
    else atomicExch(A.err, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // every CTA has read *seq: the last one advances it
    __threadfence();
    if (atomicAdd(A.done, 1u) == gridDim.x - 1) {
      *A.done = 0;
      *seq = s;
    }
  }
}

__global__ void peer_reset_kernel(uint32_t* n_src, unsigned long long* seq, int advance, uint32_t* z0, uint32_t n0,
                                  uint32_t* z1, uint32_t n1) {
  *n_src = 0;
  if (advance) {
    *seq += 1;
    for (uint32_t i = 0; i < n0; ++i) z0[i] = 0;
    for (uint32_t i = 0; i < n1; ++i) z1[i] = 0;
  }
}


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



// One exchange round, two kernels: sends (n_send PeerSend descriptors; they
// also reset the delivery list, check capacities and count the packets),
// then the wait + in-place unpack of n_slot incoming slots (PeerSlot) into
// (src_nodes, src_steps, *n_src); *seq (device) advances by one.  `done` is
// a zeroed device word (CTA counter); zero0 / zero1 (the senders' packet
// counts) are cleared once the round is sent.
extern "C" int smx_peer_exchange(const void* sends_host, int n_send, const void* slots_host, int n_slot,
                                 unsigned long long* seq, unsigned long long* sent, int* over, uint32_t* src_nodes,
                                 uint32_t* src_steps, uint32_t* n_src, uint32_t src_cap, int* err, unsigned int* done,
                                 uint32_t* zero0, uint32_t nzero0, uint32_t* zero1, uint32_t nzero1, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_send > PEER_MAX || n_slot > PEER_MAX) {
    smx_set_error("smx_peer_exchange: at most %d sends / slots", PEER_MAX);
    return -1;
  }
  if (n_send) {
    PeerSendArgs A;
    A.n = n_send;
    A.sent = sent;
    A.over = over;
    A.n_src = n_src;
    memcpy(A.s, sends_host, sizeof(PeerSend) * n_send);
    smx_count_launch(); peer_send_kernel<<<n_send, 256, 0, st>>>(A, seq);
  }
  if (n_slot) {
    PeerWaitArgs W;
    W.n = n_slot;
    W.src_nodes = src_nodes;
    W.src_steps = src_steps;
    W.n_src = n_src;
    W.src_cap = src_cap;
    W.err = err;
    W.done = done;
    W.zero[0] = zero0;
    W.zero[1] = zero1;
    W.nzero[0] = nzero0;
    W.nzero[1] = nzero1;
    memcpy(W.s, slots_host, sizeof(PeerSlot) * n_slot);
    if (!n_send) { smx_count_launch(); peer_reset_kernel<<<1, 1, 0, st>>>(n_src, seq, 0, nullptr, 0, nullptr, 0); }
    smx_count_launch(); peer_wait_kernel<<<n_slot, 256, 0, st>>>(W, seq);
  } else {
    smx_count_launch(); peer_reset_kernel<<<1, 1, 0, st>>>(n_src, seq, 1, zero0, nzero0, zero1, nzero1);
  }
  SMX_LAUNCH_CHECK();
  return 0;
}
