// Scatter microbenchmark for the sweep's binning (K7): N_REC 8-byte records, 17 per thread, go
// to uniformly random bins among NB, each bin a contiguous region of CAP slots filled through an
// atomic cursor -- the access pattern of k7_bin for one band.  Measures records/s as a function
// of the number of concurrently active bins (whose partly written tail lines must stay in L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter scatter.cu && ./scatter
// MODE 0: atomicAdd cursor + 8-B store (k7_bin); 1: atomicAdd only; 2: store only (slot from a
// per-bin hash counter, no atomic; measures the partial-sector store cost alone).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
  return z ^ (z >> 33);
}

template <int MODE>
__global__ void __launch_bounds__(128) k(uint32_t* cur, uint64_t* rec, uint32_t nb, uint32_t cap, uint64_t nthreads,
                                         uint64_t salt) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nthreads) return;
  uint32_t bin[17], slot[17];
#pragma unroll
  for (int i = 0; i < 17; i++) bin[i] = (uint32_t)__umul64hi(mix(salt + t * 17 + i), nb);
  if (MODE != 2) {
#pragma unroll
    for (int i = 0; i < 17; i++) slot[i] = atomicAdd(cur + bin[i], 1u);
  } else {
#pragma unroll
    for (int i = 0; i < 17; i++) slot[i] = (uint32_t)((t * 17 + i) / nb) % cap;
  }
  if (MODE != 1) {
#pragma unroll
    for (int i = 0; i < 17; i++)
      if (slot[i] < cap) rec[(uint64_t)bin[i] * cap + slot[i]] = (t << 8) | i;
  } else {
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 17; i++) acc += slot[i];
    if (acc == 0xFFFFFFFFu) rec[0] = acc;
  }
}

int main() {
  const uint64_t nrec = 68ull << 20;             // one C5 band per 4M-document batch
  const uint64_t nthreads = nrec / 17;
  uint32_t* cur;
  uint64_t* rec;
  const uint64_t rec_bytes = nrec * 8 * 2 + (64ull << 21) * 8;
  cudaMalloc(&cur, (1u << 22) * 4);
  cudaMalloc(&rec, rec_bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; mode++) {
    for (uint32_t lg = 10; lg <= 21; lg++) {
      const uint32_t nb = 1u << lg;
      const uint32_t cap = (uint32_t)(2 * nrec / nb + 64);
      float best = 1e9;
      for (int rep = 0; rep < 4; rep++) {
        cudaMemset(cur, 0, (size_t)nb * 4);
        cudaEventRecord(e0);
        const unsigned grid = (unsigned)((nthreads + 127) / 128);
        if (mode == 0) k<0><<<grid, 128>>>(cur, rec, nb, cap, nthreads, rep * 977);
        else if (mode == 1) k<1><<<grid, 128>>>(cur, rec, nb, cap, nthreads, rep * 977);
        else k<2><<<grid, 128>>>(cur, rec, nb, cap, nthreads, rep * 977);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("mode %d bins 2^%u: %.3f ms  %.1f Grec/s\n", mode, lg, best, nrec / best / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
