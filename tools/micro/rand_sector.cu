// Random-sector HBM microbenchmark: the attainable rate of uniformly random 4-byte
// loads and atomicOr read-modify-writes over a buffer much larger than L2, i.e. the denominator
// the Bloom stage's HBM roofline is compared against.  Each access touches one 32-B sector.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_sector rand_sector.cu
//   ./rand_sector [GB=48] [l2_fetch_granularity_bytes]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
  return z ^ (z >> 33);
}

// MODE 0: 17 independent random loads per thread (like K3); 1: 17 atomicOr with return (K4);
// 2: 17 atomicOr without return (red); 3: load then atomicOr of the same word (K3 then K4 in one).
template <int MODE>
__global__ void k(uint32_t* buf, uint64_t words, uint64_t n_threads, uint64_t salt, uint32_t* sink) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_threads) return;
  uint64_t pos[17];
#pragma unroll
  for (int i = 0; i < 17; i++) pos[i] = __umul64hi(mix(salt + t * 17 + i), words);
  uint32_t acc = 0;
  if (MODE == 0) {
    uint32_t v[17];
#pragma unroll
    for (int i = 0; i < 17; i++) v[i] = __ldcg(buf + pos[i]);
#pragma unroll
    for (int i = 0; i < 17; i++) acc |= v[i];
  } else if (MODE == 1) {
    uint32_t v[17];
#pragma unroll
    for (int i = 0; i < 17; i++) v[i] = atomicOr(buf + pos[i], 1u << (i & 31));
#pragma unroll
    for (int i = 0; i < 17; i++) acc |= v[i];
  } else if (MODE == 2) {
#pragma unroll
    for (int i = 0; i < 17; i++) atomicOr(buf + pos[i], 1u << (i & 31));
  } else if (MODE == 3) {
    uint32_t v[17];
#pragma unroll
    for (int i = 0; i < 17; i++) v[i] = __ldcg(buf + pos[i]);
#pragma unroll
    for (int i = 0; i < 17; i++)
      if (!(v[i] & 1u)) acc |= atomicOr(buf + pos[i], 1u);
  } else if (MODE == 4) {   // L2 prefetch of every line, then the atomics without waiting
#pragma unroll
    for (int i = 0; i < 17; i++) asm volatile("prefetch.global.L2 [%0];" ::"l"(buf + pos[i]));
    uint32_t v[17];
#pragma unroll
    for (int i = 0; i < 17; i++) v[i] = atomicOr(buf + pos[i], 1u << (i & 31));
#pragma unroll
    for (int i = 0; i < 17; i++) acc |= v[i];
  } else if (MODE == 6) {   // loads, then an unconditional atomic whose operand depends on the load
    uint32_t v[17];
#pragma unroll
    for (int i = 0; i < 17; i++) v[i] = __ldcg(buf + pos[i]);
#pragma unroll
    for (int i = 0; i < 17; i++) acc |= atomicOr(buf + pos[i], 1u | (v[i] & 0x80000000u));
  } else {                  // MODE 5: loads, then atomics on every word (like K4 after a reload)
    uint32_t v[17];
#pragma unroll
    for (int i = 0; i < 17; i++) v[i] = __ldcg(buf + pos[i]);
#pragma unroll
    for (int i = 0; i < 17; i++) acc |= atomicOr(buf + pos[i], v[i] | 2u);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE>
void run(const char* name, uint32_t* buf, uint64_t words, uint32_t* sink) {
  const uint64_t n_threads = 1ull << 24;   // 2.85e8 accesses per launch
  const int bs = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 6; r++) {
    cudaEventRecord(e0);
    k<MODE><<<(unsigned)((n_threads + bs - 1) / bs), bs>>>(buf, words, n_threads, 0x9E37ull * (r + 1) + MODE, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  const double acc = (double)n_threads * 17;
  printf("{\"mode\": \"%s\", \"ms\": %.3f, \"Gaccess_per_s\": %.3f, \"sector_GBps\": %.1f, \"err\": \"%s\"}\n", name,
         best, acc / best / 1e6, acc * 32 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 48.0;
  if (argc > 2) {   // cudaLimitMaxL2FetchGranularity (bytes): how much L2 fetches from DRAM per miss
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[2]));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity\": %zu, \"set\": \"%s\"}\n", v, cudaGetErrorString(e));
  } else {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity_default\": %zu}\n", v);
  }
  const uint64_t words = (uint64_t)(gb * 1e9 / 4);
  uint32_t *buf, *sink;
  if (cudaMalloc(&buf, words * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 0, words * 4);
  printf("{\"buffer_GB\": %.1f}\n", words * 4 / 1e9);
  // every mode starts from an all-zero buffer
  cudaMemset(buf, 0, words * 4); run<0>("load", buf, words, sink);
  cudaMemset(buf, 0, words * 4); run<2>("atomicOr_noret", buf, words, sink);
  cudaMemset(buf, 0, words * 4); run<1>("atomicOr_ret", buf, words, sink);
  cudaMemset(buf, 0, words * 4); run<5>("load_then_atomicOr_all", buf, words, sink);
  cudaMemset(buf, 0, words * 4); run<6>("load_then_atomicOr_dep", buf, words, sink);
  cudaMemset(buf, 0, words * 4); run<3>("load_then_atomicOr_if_clear", buf, words, sink);
  cudaMemset(buf, 0, words * 4); run<4>("prefetchL2_then_atomicOr", buf, words, sink);
  return 0;
}
