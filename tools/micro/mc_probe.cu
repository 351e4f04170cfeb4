// NVLS multicast probe (single process, every visible GPU).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_probe mc_probe.cu -lcuda
//   ./mc_probe [MiB]
//
// Builds one multicast object over all GPUs (cuMulticastCreate + a physical
// allocation bound on each device), maps its multicast address on GPU 0 and
// pushes a buffer from GPU 0's HBM into it, once with SM stores
// (multimem.st.v4.f32 -> STG.128 to the multicast VA) and once with bulk
// copies (cp.async.bulk shared -> global at the multicast VA).  Every GPU's
// unicast view must then hold the bytes; the rate is bytes / kernel time, the
// ingress each receiver saw.  Also times a plain unicast peer write (GPU 0 ->
// GPU 1) for comparison.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    CUresult r_ = (x);                                                              \
    if (r_ != CUDA_SUCCESS) {                                                       \
      const char* s_ = nullptr;                                                     \
      cuGetErrorString(r_, &s_);                                                    \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?"); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)
#define RK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) {                                                                 \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                          \
    }                                                                                        \
  } while (0)

__global__ void fill(uint32_t* p, size_t n, uint32_t salt) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = uint32_t(i * 2654435761u) ^ salt;
}

// SM stores to the multicast address: 16 B per thread per iteration.
__global__ void push_st(const float4* __restrict__ src, float4* mc, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    float4 v = src[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  }
}

// plain stores (unicast peer write, or local copy)
__global__ void push_plain(const float4* __restrict__ src, float4* dst, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// Bulk copies: global -> smem (local HBM), then smem -> global at the
// multicast address; one warp-elected thread per CTA, kSlot bytes per step.
constexpr int kSlot = 32768;
__global__ void push_bulk(const uint8_t* __restrict__ src, uint8_t* mc, size_t bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint32_t phase = 0;
  for (size_t off = size_t(blockIdx.x) * kSlot; off < bytes; off += size_t(gridDim.x) * kSlot) {
    const uint32_t n = static_cast<uint32_t>(bytes - off < kSlot ? bytes - off : kSlot);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem free again
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
                 "l"(src + off), "r"(n), "r"(b)
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(b),
        "r"(phase)
        : "memory");
    phase ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(mc + off), "r"(s), "r"(n)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1024;
  CK(cuInit(0));
  int n = 0;
  RK(cudaGetDeviceCount(&n));
  std::printf("devices %d\n", n);
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    int mc = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    std::printf("dev %d multicast_supported %d\n", d, mc);
    if (!mc) return 2;
  }
  CUmulticastObjectProp mp{};
  mp.numDevices = n;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = mib << 20;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (mp.size + gran - 1) / gran * gran;
  mp.size = size;
  std::printf("granularity %zu size %zu\n", gran, size);
  CUmemGenericAllocationHandle mch;
  CK(cuMulticastCreate(&mch, &mp));
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    CK(cuMulticastAddDevice(mch, dev));
  }
  std::vector<CUdeviceptr> uva(n);
  std::vector<CUmemGenericAllocationHandle> mem(n);
  for (int d = 0; d < n; ++d) {
    RK(cudaSetDevice(d));
    RK(cudaFree(nullptr));  // primary context
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CK(cuMemCreate(&mem[d], size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem[d], 0, size, 0));
    CK(cuMemAddressReserve(&uva[d], size, ag, 0, 0));
    CK(cuMemMap(uva[d], size, 0, mem[d], 0));
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva[d], size, &ad, 1));
  }
  RK(cudaSetDevice(0));
  CUdeviceptr mcva;
  CK(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CK(cuMemMap(mcva, size, 0, mch, 0));
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcva, size, &ad, 1));
  uint8_t* src = nullptr;
  RK(cudaMalloc(&src, size));
  fill<<<1184, 256>>>(reinterpret_cast<uint32_t*>(src), size / 4, 77);
  RK(cudaDeviceSynchronize());
  int sms = 0;
  RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  auto check_all = [&](const char* what, uint32_t salt_expect) {
    std::vector<uint32_t> h(size / 4);
    int bad = 0;
    for (int d = 0; d < n; ++d) {
      RK(cudaSetDevice(d));
      RK(cudaMemcpy(h.data(), reinterpret_cast<void*>(uva[d]), size, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < h.size(); i += 4099)
        if (h[i] != (uint32_t(i * 2654435761u) ^ salt_expect)) {
          ++bad;
          break;
        }
    }
    RK(cudaSetDevice(0));
    std::printf("%s verify %s\n", what, bad ? "BAD" : "ok");
  };
  auto clear_all = [&]() {
    for (int d = 0; d < n; ++d) {
      RK(cudaSetDevice(d));
      RK(cudaMemset(reinterpret_cast<void*>(uva[d]), 0, size));
      RK(cudaDeviceSynchronize());
    }
    RK(cudaSetDevice(0));
  };
  auto timed = [&](const char* what, auto launch) {
    for (int w = 0; w < 2; ++w) launch();
    RK(cudaDeviceSynchronize());
    const int reps = 5;
    RK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    RK(cudaEventRecord(e1));
    RK(cudaEventSynchronize(e1));
    float ms = 0;
    RK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    std::printf("%s: %.3f ms, %.1f GB/s per receiver (%d receivers incl. GPU 0)\n", what, ms, size / (ms * 1e6),
                n);
  };
  for (int blocks_per_sm : {1, 2, 4}) {
    clear_all();
    char name[64];
    std::snprintf(name, sizeof(name), "multimem.st x%d/SM", blocks_per_sm);
    timed(name, [&] {
      push_st<<<sms * blocks_per_sm, 512>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(mcva),
                                            size / 16);
    });
    RK(cudaGetLastError());
    check_all(name, 77);
  }
  RK(cudaFuncSetAttribute(push_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlot));
  for (int blocks_per_sm : {1, 2, 4}) {
    clear_all();
    char name[64];
    std::snprintf(name, sizeof(name), "bulk copy x%d/SM", blocks_per_sm);
    timed(name, [&] {
      push_bulk<<<sms * blocks_per_sm, 32, kSlot>>>(src, reinterpret_cast<uint8_t*>(mcva), size);
    });
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      std::printf("%s: %s\n", name, cudaGetErrorString(e));
      break;
    }
    check_all(name, 77);
  }
  if (n > 1) {
    int can = 0;
    RK(cudaDeviceCanAccessPeer(&can, 0, 1));
    if (can) {
      cudaDeviceEnablePeerAccess(1, 0);
      cudaGetLastError();
      uint8_t* peer = nullptr;
      RK(cudaSetDevice(1));
      RK(cudaMalloc(&peer, size));
      RK(cudaSetDevice(0));
      timed("unicast peer write 0->1", [&] {
        push_plain<<<sms * 2, 512>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(peer),
                                     size / 16);
      });
    }
  }
  std::printf("done\n");
  return 0;
}
