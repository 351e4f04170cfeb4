// Micro-benchmark (diagnostic): latency of the serial XXH64 round chain on
// sm_100a, data in registers (no memory), 4 lanes = 4 accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2604_09107_b200/csrc xxh_chain.cu -o xxh_chain
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "dev_common.cuh"
using namespace rsb::dev::detail;

__global__ void chain(std::uint64_t* out, int rounds, int mode) {
  std::uint64_t acc = threadIdx.x * 0x1234567ull + 1;
  std::uint64_t w = threadIdx.x + 99;
  long long t0 = clock64();
  std::uint64_t g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (mode == 0) {
    for (int i = 0; i < rounds; ++i) { acc = xround(acc, w); w += 0x9E37; }
  } else if (mode == 1) {
    for (int i = 0; i < rounds; ++i) { acc = xround_pre(acc, w); w += 0x9E37; }
  } else {  // fused: the next product added inside the multiply
    for (int i = 0; i < rounds; ++i) { acc = xround_fused(acc, w); w += 0x9E37; }
  }
  long long t1 = clock64();
  std::uint64_t g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    out[32] = (t1 - t0);
    out[33] = g1 - g0;
  }
}

int main() {
  std::uint64_t* d;
  cudaMalloc(&d, 64 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    for (int lanes : {4, 32}) {
      int rounds = 1 << 24;
      chain<<<1, lanes>>>(d, rounds, mode);
      cudaDeviceSynchronize();
      std::uint64_t h[34];
      cudaMemcpy(h, d, 34 * 8, cudaMemcpyDeviceToHost);
      printf("{\"mode\": %d, \"lanes\": %d, \"cycles_per_round\": %.2f, \"ns_per_round\": %.2f, "
             "\"mhz\": %.0f}\n", mode, lanes, double(h[32]) / rounds, double(h[33]) / rounds,
             double(h[32]) / double(h[33]) * 1e3);
    }
  }
  return 0;
}
