// Read / write mix ceilings for the fused pass (reads g and acc, writes acc:
// 2 reads : 1 write per element), persistent CTAs claiming 64 KB chunks from
// a counter vs non-persistent one-shot blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rw_mix rw_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// kMode 0: read only (sum into a register, one store per thread at the end)
//       1: read a, write a (in place)          1:1
//       2: read g and a, write a               2:1 (the fused pass)
template <int kMode, uint32_t kChunk4>
__global__ void k_claim(const float4* __restrict__ g, float4* __restrict__ a, uint64_t n4, unsigned* counter,
                        float* sink) {
  __shared__ unsigned s_c;
  float acc = 0.f;
  const uint64_t chunks = n4 / kChunk4;
  for (;;) {
    if (threadIdx.x == 0) s_c = atomicAdd(counter, 1u);
    __syncthreads();
    const uint64_t c = s_c;
    __syncthreads();
    if (c >= chunks) break;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < kChunk4; i += blockDim.x) {
      const uint64_t j = c * kChunk4 + i;
      float4 x = __ldcs(a + j);
      if (kMode == 2) {
        const float4 y = __ldcs(g + j);
        x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
      }
      if (kMode == 0) acc += x.x + x.y + x.z + x.w;
      else __stcs(a + j, x);
    }
  }
  if (kMode == 0 && acc == 12345.f) *sink = acc;
}

template <int kMode>
__global__ void k_oneshot(const float4* __restrict__ g, float4* __restrict__ a, uint64_t n4, float* sink) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n4) return;
  float4 x = __ldcs(a + j);
  if (kMode == 2) {
    const float4 y = __ldcs(g + j);
    x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
  }
  if (kMode == 0) {
    if (x.x + x.y + x.z + x.w == 12345.f) *sink = x.x;
  } else {
    __stcs(a + j, x);
  }
}

int main() {
  const uint64_t n = 1ull << 28;
  float *g, *a, *sink;
  unsigned* ctr;
  cudaMalloc(&g, n * 4);
  cudaMalloc(&a, n * 4);
  cudaMalloc(&sink, 4);
  cudaMalloc(&ctr, 4096 * 4);
  cudaMemset(ctr, 0, 4096 * 4);
  cudaMemset(g, 0, n * 4);
  cudaMemset(a, 0, n * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int li = 0;
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    std::printf("%-46s %8.1f us %8.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  const uint64_t n4 = n / 4;
  const double B = double(n) * 4;
  for (int per : {2, 4, 8}) {
    char nm[96];
    std::snprintf(nm, sizeof nm, "read only, claimed 64 KB, %d CTAs", sms * per);
    run(nm, B, [&] { k_claim<0, 4096><<<sms * per, 256>>>((float4*)g, (float4*)a, n4, ctr + li++, sink); });
    std::snprintf(nm, sizeof nm, "read+write 1:1, claimed 64 KB, %d CTAs", sms * per);
    run(nm, 2 * B, [&] { k_claim<1, 4096><<<sms * per, 256>>>((float4*)g, (float4*)a, n4, ctr + li++, sink); });
    std::snprintf(nm, sizeof nm, "read 2 : write 1, claimed 64 KB, %d CTAs", sms * per);
    run(nm, 3 * B, [&] { k_claim<2, 4096><<<sms * per, 256>>>((float4*)g, (float4*)a, n4, ctr + li++, sink); });
  }
  run("read only, one-shot", B, [&] { k_oneshot<0><<<unsigned(n4 / 256), 256>>>((float4*)g, (float4*)a, n4, sink); });
  run("read+write 1:1, one-shot", 2 * B, [&] { k_oneshot<1><<<unsigned(n4 / 256), 256>>>((float4*)g, (float4*)a, n4, sink); });
  run("read 2 : write 1, one-shot", 3 * B, [&] { k_oneshot<2><<<unsigned(n4 / 256), 256>>>((float4*)g, (float4*)a, n4, sink); });
  std::printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
