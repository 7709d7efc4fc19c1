// The fused pass's data movement alone: a producer warp streams 4096-element
// tiles of g and acc into a ring of shared-memory stages (1-D TMA bulk copies,
// mbarriers); 8 consumer warps add them and store acc back (st.global.cs) plus
// a 16-bit index word per quad (12.5 B per element, the fused pass's 12.58).
// Is the ring the ceiling (the fused pass runs at 5.9 TB/s) or the consumers'
// classification work?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ring tma_ring.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTile = 4096;
constexpr int kCons = 256;
template <int S>
struct Ring {
  struct alignas(128) Stage {
    float g[kTile];
    float a[kTile];
  } st[S];
  unsigned long long full[S], empty[S];
};
__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mwait(unsigned long long* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra.uni W_%=;\n}\n" ::"r"(su(b)), "r"(par) : "memory");
}
template <int S>
__global__ void __launch_bounds__(288, 1) k_ring(const float* g, float* acc, uint16_t* idx, uint64_t tiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  Ring<S>& r = *reinterpret_cast<Ring<S>*>(sm);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t per = (tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = per * blockIdx.x, t1 = t0 + per < tiles ? t0 + per : tiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&r.full[s])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su(&r.empty[s])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      uint32_t i = 0;
      for (uint64_t t = t0; t < t1; ++t, ++i) {
        const int s = int(i % S);
        if (i >= uint32_t(S)) mwait(&r.empty[s], ((i / S) - 1) & 1u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&r.full[s])), "r"(2u * kTile * 4u) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su(r.st[s].g)), "l"(g + t * kTile), "r"(kTile * 4u), "r"(su(&r.full[s])), "l"(pol) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su(r.st[s].a)), "l"(acc + t * kTile), "r"(kTile * 4u), "r"(su(&r.full[s])), "l"(pol) : "memory");
      }
    }
    return;
  }
  uint32_t i = 0;
  for (uint64_t t = t0; t < t1; ++t, ++i) {
    const int s = int(i % S);
    mwait(&r.full[s], (i / S) & 1u);
#pragma unroll
    for (int k = 0; k < kTile / 4 / kCons; ++k) {
      const uint32_t q = k * kCons + threadIdx.x;
      const float4 x = reinterpret_cast<const float4*>(r.st[s].g)[q];
      const float4 y = reinterpret_cast<const float4*>(r.st[s].a)[q];
      const float4 v = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
      __stcs(reinterpret_cast<float4*>(acc + t * kTile) + q, v);
      idx[t * (kTile / 4) + q] = uint16_t((v.x > 1.f) | (v.y > 1.f) << 4 | (v.z > 1.f) << 8 | (v.w > 1.f) << 12);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&r.empty[s])) : "memory");
  }
}

int main() {
  const uint64_t n = 1ull << 28, tiles = n / kTile;
  float *g, *a;
  uint16_t* idx;
  cudaMalloc(&g, n * 4);
  cudaMalloc(&a, n * 4);
  cudaMalloc(&idx, n / 2);
  cudaMemset(g, 0, n * 4);
  cudaMemset(a, 0, n * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    const double bytes = double(n) * 12.5;
    std::printf("%-40s %8.1f us %8.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  const int s2 = sizeof(Ring<2>), s3 = sizeof(Ring<3>), s6 = sizeof(Ring<6>);
  cudaFuncSetAttribute(k_ring<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
  cudaFuncSetAttribute(k_ring<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3);
  cudaFuncSetAttribute(k_ring<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, s6);
  run("ring 3 stages, 2 CTAs/SM", [&] { k_ring<3><<<sms * 2, 288, s3>>>(g, a, idx, tiles); });
  run("ring 2 stages, 3 CTAs/SM", [&] { k_ring<2><<<sms * 3, 288, s2>>>(g, a, idx, tiles); });
  run("ring 3 stages, 1 CTA/SM", [&] { k_ring<3><<<sms, 288, s3>>>(g, a, idx, tiles); });
  run("ring 6 stages, 1 CTA/SM", [&] { k_ring<6><<<sms, 288, s6>>>(g, a, idx, tiles); });
  for (int per : {4, 8, 16, 32}) {
    char nm[80];
    std::snprintf(nm, sizeof nm, "non-persistent 3 stages, %d tiles per CTA", per);
    run(nm, [&] { k_ring<3><<<unsigned(tiles / per), 288, s3>>>(g, a, idx, tiles); });
    std::snprintf(nm, sizeof nm, "non-persistent 2 stages, %d tiles per CTA", per);
    run(nm, [&] { k_ring<2><<<unsigned(tiles / per), 288, s2>>>(g, a, idx, tiles); });
  }
  std::printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
