// Peak BLAKE2b compression rate on this GPU: register-only compressions (no memory traffic),
// enough threads to fill every SM.  This is the roofline denominator of the hash kernels
// (k_keys, k_digest), which are integer-ALU bound.  Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/b2b_peak tools/b2b_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2005_05837_b200/csrc/ef_blake2b.cuh"
#include "ef_b2b_fma.cuh"

template <int VARIANT>
__global__ void __launch_bounds__(128) peak(uint64_t* out, int iters, uint32_t one) {
  uint64_t h[8], m[16];
  for (int i = 0; i < 16; ++i) m[i] = (uint64_t)(threadIdx.x + 131 * blockIdx.x) * 0x9e3779b97f4a7c15ULL + i;
  for (int i = 0; i < 8; ++i) h[i] = ef::b2b_iv(i);
  for (int r = 0; r < iters; ++r) {
    if (VARIANT == 0) ef::b2b_compress(h, m, 128, false);
    else ef::b2b_compress_fma(h, m, 128, false, one);
    m[r & 15] ^= h[0];
  }
  uint64_t x = 0;
  for (int i = 0; i < 8; ++i) x ^= h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 16, threads = 128, iters = 2000;
  uint64_t* out;
  cudaMalloc(&out, (size_t)blocks * threads * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double rate[2] = {0, 0};
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      if (v == 0) peak<0><<<blocks, threads>>>(out, iters, 1);
      else peak<1><<<blocks, threads>>>(out, iters, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double r = (double)blocks * threads * iters / (ms * 1e-3);
      if (rep > 0 && r > rate[v]) rate[v] = r;
    }
  }
  printf("{\"b2b_compress_per_s\": %.6e, \"b2b_compress_fma_per_s\": %.6e, \"sms\": %d, \"threads\": %d, \"iters\": %d}\n",
         rate[0], rate[1], sms, blocks * threads, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
