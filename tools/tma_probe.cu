// Bulk-copy (TMA engine) streaming probe: one CTA per SM, one producer thread
// issuing cp.async.bulk global->shared copies of CHUNK bytes into a ring of
// STAGES slots; consumers only wait for "full" and release the slot.  Reports
// the achieved HBM read bandwidth for several (chunk, stages, copies-per-stage)
// settings, and a plain LDG streaming kernel for comparison.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
//   ./tools/tma_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_parity(uint64_t* b, unsigned ph, int mode) {
  uint32_t ok = 0;
  if (mode == 1) {
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(su32(b)), "r"(ph));
  } else {
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(su32(b)), "r"(ph));
  }
}

__global__ void tma_stream(const char* __restrict__ src, size_t bytes, int chunk, int stages, int ncopy,
                           unsigned long long* sink, int mode) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(stages) * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + s)), "r"(mode >= 2 ? 1 : blockDim.x / 32 - 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t per_cta = bytes / gridDim.x / chunk * chunk;
  const char* base = src + per_cta * blockIdx.x;
  const int n = int(per_cta / chunk);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  unsigned long long acc = 0;
  if (warp == 0 && mode == 3) {
    const int np = 4;
    if (lane < np) {
      for (int i = lane; i < n; i += np) {
        const int s = i % stages;
        const unsigned ph = (i / stages) & 1;
        if (i >= stages) wait_parity(full + s, ph ^ 1, 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(chunk));
        const int part = chunk / ncopy;
        for (int c = 0; c < ncopy; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sm + size_t(s) * chunk + c * part)), "l"(base + size_t(i) * chunk + c * part),
                       "r"(part), "r"(su32(full + s)) : "memory");
      }
      const int last0 = ((n - 1) / np) * np + lane;
      for (int i = (last0 >= n ? last0 - np : last0); i >= 0 && i > (last0 >= n ? last0 - np : last0) - stages; i -= np)
        wait_parity(full + (i % stages), (i / stages) & 1, 1);
    }
  } else if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % stages;
        const unsigned ph = (i / stages) & 1;
        if (mode == 2) {   // producer alone: recycle the slot when its previous copy landed
          if (i >= stages) wait_parity(full + s, ph ^ 1, 1);
        } else {
          wait_parity(empty + s, ph ^ 1, mode);
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(chunk));
        const int part = chunk / ncopy;
        for (int c = 0; c < ncopy; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sm + size_t(s) * chunk + c * part)), "l"(base + size_t(i) * chunk + c * part),
                       "r"(part), "r"(su32(full + s)) : "memory");
      }
      if (mode == 2)
        for (int i = n; i < n + stages; ++i) wait_parity(full + (i % stages), ((i / stages) & 1) ^ 1, 1);
    }
  } else if (mode < 2) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      const unsigned ph = (i / stages) & 1;
      wait_parity(full + s, ph, mode);
      acc += *reinterpret_cast<const unsigned*>(sm + size_t(s) * chunk + (threadIdx.x * 4) % chunk);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)));
    }
  }
  if (acc == 12345) *sink = acc;
}

__global__ void ldg_stream(const double2* __restrict__ src, size_t n, double* sink) {
  double acc = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    double2 v = __ldcs(src + i);
    acc += v.x + v.y;
  }
  if (acc == 1.2345) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(4) << 30;   // 4 GiB
  char* src;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 1, bytes));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  const int chunks[] = {4096, 8192, 16384, 32768, 65536};
  const int ring_bytes[] = {65536, 131072, 196608};
  printf("{\"probe\": \"tma_stream\", \"sms\": %d, \"results\": [\n", sms);
  bool first = true;
  for (int mode = 2; mode < 4; ++mode)
  for (int rb : ring_bytes)
    for (int ch : chunks) {
      const int st = rb / ch;
      if (st < 2 || st > 48) continue;
      if (rb != 131072 && mode != 0) continue;
      for (int ncopy : {1, 4}) {
        if (ch / ncopy < 1024) continue;
        const size_t smem = size_t(st) * ch + 16 * st;
        float best = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          tma_stream<<<sms, 32 * 9, smem>>>(src, bytes, ch, st, ncopy, sink, mode);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        CK(cudaGetLastError());
        const double moved = double(bytes / sms / ch * ch) * sms;
        printf("%s {\"mode\": %d, \"chunk\": %d, \"stages\": %d, \"copies_per_stage\": %d, \"ring_kb\": %d, \"gbs\": %.1f}",
               first ? "" : ",\n", mode, ch, st, ncopy, rb / 1024, moved / (best * 1e-3) / 1e9);
        first = false;
      }
    }
  float best = 1e9f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    ldg_stream<<<sms * 4, 512>>>(reinterpret_cast<const double2*>(src), bytes / 16, reinterpret_cast<double*>(sink));
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf(",\n {\"ldg_stream\": true, \"gbs\": %.1f}\n]}\n", bytes / (best * 1e-3) / 1e9);
  return 0;
}
