// Reference-layout entry points: the two native kernels of the reference
// package (sm/kernels/__init__.py:25-26, _speedups.pyx:13-54) with their
// exact array layouts, on device pointers.  A reference maintainer can swap
// `kernels._active` for a ctypes module over these two functions
// and keep every other line of sm/engine.py unchanged.
#include "common.cuh"

namespace {

// kernels/_speedups.pyx:13-35 (element-for-element, fp64 without FMA)
__global__ void ref_lif_kernel(double* v, int64_t* ref_count, const uint8_t* real_mask, const double* inputs,
                               const double* decay, const double* v_rest, const double* v_reset,
                               const double* v_th, const int64_t* ref_steps, uint8_t* spiked_out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!real_mask[i]) { spiked_out[i] = 0; return; }
  if (ref_count[i] > 0) {
    ref_count[i] -= 1;
    v[i] = v_reset[i];
    spiked_out[i] = 0;
    return;
  }
  const double integ = __dadd_rn(__dadd_rn(v_rest[i], __dmul_rn(__dsub_rn(v[i], v_rest[i]), decay[i])), inputs[i]);
  if (integ >= v_th[i]) {
    spiked_out[i] = 1;
    v[i] = v_reset[i];
    ref_count[i] = ref_steps[i];
  } else {
    spiked_out[i] = 0;
    v[i] = integ;
  }
}

// kernels/_speedups.pyx:38-54: one CTA per listed source, threads over its
// CSR range; buffers[tgt, port, (now + delay) % L] += weight * mult.
__global__ void ref_deliver_kernel(const int64_t* src_nodes, const int64_t* mults, uint64_t k,
                                   const int64_t* first_index, const int64_t* tgt, const int64_t* port,
                                   const int64_t* delay, const double* weight, double* buffers, int64_t n_ports,
                                   int64_t L, int64_t now) {
  for (uint64_t j = blockIdx.x; j < k; j += gridDim.x) {
    const int64_t node = src_nodes[j];
    const double mult = (double)mults[j];
    const int64_t lo = first_index[node], hi = first_index[node + 1];
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
      const int64_t slot = (now + delay[e]) % L;
      atomicAdd(buffers + (tgt[e] * n_ports + port[e]) * L + slot, __dmul_rn(weight[e], mult));
    }
  }
}

}  // namespace

extern "C" int smx_ref_lif_step(double* v, int64_t* ref_count, const uint8_t* real_mask, const double* inputs,
                                const double* decay, const double* v_rest, const double* v_reset,
                                const double* v_th, const int64_t* ref_steps, uint8_t* spiked_out, uint64_t n,
                                void* stream) {
  if (n == 0) return 0;
  smx_count_launch(); ref_lif_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(v, ref_count, real_mask, inputs, decay, v_rest, v_reset, v_th, ref_steps, spiked_out, n);
  SMX_LAUNCH_CHECK();
  return 0;
}

extern "C" int smx_ref_deliver_spikes(const int64_t* src_nodes, const int64_t* mults, uint64_t k,
                                      const int64_t* first_index, const int64_t* tgt, const int64_t* port,
                                      const int64_t* delay, const double* weight, double* buffers, int64_t n_ports,
                                      int64_t L, int64_t now, void* stream) {
  if (k == 0) return 0;
  const unsigned grid = (unsigned)(k < 148 * 8 ? k : 148 * 8);
  smx_count_launch(); ref_deliver_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(src_nodes, mults, k, first_index, tgt, port, delay, weight, buffers, n_ports, L, now);
  SMX_LAUNCH_CHECK();
  return 0;
}
