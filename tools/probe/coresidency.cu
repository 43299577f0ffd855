// Probe: does a small kernel on another stream start while a persistent
// kernel (grid g1 x 512 threads, s1 bytes of dynamic smem, 2 CTAs/SM) holds
// the GPU?  Prints the host-measured latency from the small kernel's launch
// to its completion for several (g1, s1, small-kernel smem, grid) choices.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 2) spin(long long cycles, int* sink) {
  extern __shared__ int sm[];
  long long t0 = clock64();
  int acc = 0;
  if (threadIdx.x < 64) sm[threadIdx.x] = 0;
  __syncthreads();
  while (clock64() - t0 < cycles) acc += sm[threadIdx.x & 63];
  if (acc == 12345) *sink = acc;
}

__global__ void __launch_bounds__(256) small(int* out) {
  __shared__ int sm[256];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, sm[5]);
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(small, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spin, 512, 72 * 1024);
  printf("SMs %d, spin CTAs/SM at 72 KB: %d\n", sms, occ);
  const long long cyc = 20LL * 1900 * 1000;  // ~20 ms
  struct Cfg { int g1; int s1k; int s2k; int g2; int legacy; };
  Cfg cfgs[] = {{280, 72, 0, 1, 0}, {280, 72, 57, 1, 0}, {280, 72, 57, 148, 0}, {280, 72, 0, 1, 1},
                {140, 72, 57, 148, 0}, {148, 72, 57, 148, 0}, {296, 72, 0, 1, 0}, {264, 72, 57, 16, 0},
                {280, 40, 57, 148, 0}, {280, 100, 0, 1, 0}};
  for (auto c : cfgs) {
    cudaDeviceSynchronize();
    spin<<<c.g1, 512, c.s1k * 1024, a>>>(cyc, d);
    cudaStream_t sb = c.legacy ? (cudaStream_t)0 : b;
    double t0 = now_ms();
    while (now_ms() - t0 < 1.0) {}
    double t1 = now_ms();
    small<<<c.g2, 256, c.s2k * 1024, sb>>>(d);
    cudaStreamSynchronize(sb);
    double t2 = now_ms();
    cudaStreamSynchronize(a);
    double t3 = now_ms();
    printf("spin grid %3d smem %3d KB | small grid %3d smem %2d KB %s: small done after %6.2f ms (spin ends %6.2f ms) %s\n",
           c.g1, c.s1k, c.g2, c.s2k, c.legacy ? "legacy " : "nonblk ", t2 - t1, t3 - t1,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
