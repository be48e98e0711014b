// Probe: pure-read HBM bandwidth on this B200 (the denominator a read-only
// stream such as k_schur_symv can be compared with; MEASURED_PEAKS.json's
// hbm_gbs is a copy, read + write).  Two read kernels over 16 GiB of doubles
// (far beyond L2): (1) grid-stride 16-byte loads with a per-thread sum,
// (2) 1D TMA bulk copies (cp.async.bulk) of 32 KB chunks into a shared-memory
// ring of 6 stages per CTA, one CTA per SM -- the access pattern of the
// relaxation's record streams.  Best of 10, CUDA events; clocks printed.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe/read_bw.cu -o tools/probe/read_bw -lnvidia-ml
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <nvml.h>

__global__ void read_ld(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const double2 v = __ldcs(a + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;  // keep the loads
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int kStages = 6, kChunk = 32768;
__global__ void __launch_bounds__(32) read_bulk(const char* __restrict__ a, size_t nchunks, double* out) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  double s = 0.0;
  size_t k = 0;
  auto issue = [&](size_t c, int st) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[st])), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(ring + st * kChunk)),
                 "l"(a + c * kChunk), "r"(kChunk), "r"(su32(&bar[st]))
                 : "memory");
  };
  for (int st = 0; st < kStages; ++st) {
    const size_t c = blockIdx.x + size_t(st) * gridDim.x;
    if (c < nchunks) issue(c, st);
  }
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    const int st = int(k % kStages);
    const uint32_t par = uint32_t((k / kStages) & 1);
    asm volatile(
        "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
            su32(&bar[st])),
        "r"(par)
        : "memory");
    s += reinterpret_cast<const double*>(ring + st * kChunk)[0];
    const size_t nx = c + size_t(kStages) * gridDim.x;
    if (nx < nchunks) issue(nx, st);
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  const size_t bytes = size_t(16) << 30;
  char* a = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&out, 8) != cudaSuccess) {
    std::printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 1, bytes);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  nvmlInit();
  nvmlDevice_t dev;
  nvmlDeviceGetHandleByIndex(0, &dev);
  auto best = [&](auto launch) {
    float b = 1e30f;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < b) b = ms;
    }
    return b;
  };
  const float t_ld = best([&] { read_ld<<<nsm * 8, 512>>>(reinterpret_cast<const double2*>(a), bytes / 16, out); });
  cudaFuncSetAttribute(read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk);
  const float t_bulk = best([&] { read_bulk<<<nsm, 32, kStages * kChunk>>>(a, bytes / kChunk, out); });
  unsigned sm_mhz = 0, mem_mhz = 0;
  nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &sm_mhz);
  nvmlDeviceGetClockInfo(dev, NVML_CLOCK_MEM, &mem_mhz);
  std::printf("read ld.global (16 B, grid-stride): %.1f GB/s\n", bytes / (t_ld * 1e-3) / 1e9);
  std::printf("read cp.async.bulk (32 KB chunks, 6-stage ring, 1 CTA/SM): %.1f GB/s\n", bytes / (t_bulk * 1e-3) / 1e9);
  std::printf("clocks after: sm %u MHz, mem %u MHz; err %s\n", sm_mhz, mem_mhz, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
