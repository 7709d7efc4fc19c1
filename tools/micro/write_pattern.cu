// Write-pattern probe for the dense emit (a 1 GB store): does the order in
// which CTAs cover the output matter for HBM write bandwidth?
//   a: grid-stride float4 stores (every CTA near the same address: a wavefront)
//   b: each CTA stores its own contiguous 1/G of the output with float4 stores
//   c: as b, 32 KB TMA bulk stores from a zeroed 2-buffer shared ring (k_emit)
//   d: as c, chunks dealt round-robin (chunk c -> CTA c % G: a wavefront)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_pattern write_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint32_t kChunk = 8192;  // floats (32 KB)

__global__ void k_a(float4* out, uint64_t n4) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void k_b(float4* out, uint64_t n4) {
  const uint64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const uint64_t b = per * blockIdx.x, e = b + per < n4 ? b + per : n4;
  for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// e: non-persistent, one float4 per thread; f: grid-stride streaming
// (st.global.cs) float4; g: grid-stride 32-byte stores (st.global.v8.f32);
// h: non-persistent, 4 float4 per thread (unrolled)
__global__ void k_e(float4* out, uint64_t n4) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n4) out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__global__ void k_f(float4* out, uint64_t n4) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += uint64_t(gridDim.x) * blockDim.x)
    __stcs(out + i, make_float4(0.f, 0.f, 0.f, 0.f));
}
__global__ void k_g(float* out, uint64_t n8) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += uint64_t(gridDim.x) * blockDim.x) {
    float* p = out + 8 * i;
    asm volatile("st.global.v8.f32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(p), "f"(0.0f) : "memory");
  }
}
__global__ void k_h(float4* out, uint64_t n4) {
  const uint64_t b = (uint64_t(blockIdx.x) * blockDim.x) * 4 + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (b + k * blockDim.x < n4) out[b + k * blockDim.x] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// i: persistent, chunks of kDyn float4 claimed from a counter (dynamic balance)
template <uint32_t kDyn>
__global__ void k_dyn(float4* out, uint64_t n4, unsigned* counter) {
  __shared__ unsigned s_c;
  const uint64_t chunks = n4 / kDyn;
  for (;;) {
    if (threadIdx.x == 0) s_c = atomicAdd(counter, 1u);
    __syncthreads();
    const uint64_t c = s_c;
    __syncthreads();
    if (c >= chunks) break;
    float4* p = out + c * kDyn;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < kDyn; i += blockDim.x) p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
// j: TMA ring with chunks claimed from a counter
__global__ void k_tma_dyn(float* out, uint64_t n, unsigned* counter) {
  extern __shared__ __align__(128) float buf[];
  __shared__ unsigned s_c;
  const uint64_t chunks = n / kChunk;
  for (uint32_t k = 0;; ++k) {
    if (threadIdx.x == 0) s_c = atomicAdd(counter, 1u);
    float* b = buf + (k & 1u) * kChunk;
    if (k >= 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const uint64_t c = s_c;
    if (c >= chunks) break;
    float4* b4 = reinterpret_cast<float4*>(b);
    for (uint32_t q = threadIdx.x; q < kChunk / 4; q += blockDim.x) b4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(b));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * kChunk), "r"(s),
                   "r"(kChunk * 4u)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <bool kRoundRobin>
__global__ void k_tma(float* out, uint64_t n) {
  extern __shared__ __align__(128) float buf[];
  const uint64_t chunks = n / kChunk;
  uint64_t c0, step, c1;
  if (kRoundRobin) {
    c0 = blockIdx.x;
    step = gridDim.x;
    c1 = chunks;
  } else {
    const uint64_t per = (chunks + gridDim.x - 1) / gridDim.x;
    c0 = per * blockIdx.x;
    step = 1;
    c1 = c0 + per < chunks ? c0 + per : chunks;
  }
  uint32_t k = 0;
  for (uint64_t c = c0; c < c1; c += step, ++k) {
    float* b = buf + (k & 1u) * kChunk;
    if (k >= 2) {
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
    }
    float4* b4 = reinterpret_cast<float4*>(b);
    for (uint32_t q = threadIdx.x; q < kChunk / 4; q += blockDim.x) b4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(b));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * kChunk), "r"(s),
                   "r"(kChunk * 4u)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t n = 1ull << 28;
  float* out;
  cudaMalloc(&out, n * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 2 * kChunk * 4;
  cudaFuncSetAttribute(k_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
    std::printf("%-44s %8.1f us %8.1f GB/s\n", name, ms * 1e3, n * 4 / (ms * 1e-3) / 1e9);
  };
  for (int per : {2, 3, 4, 8}) {
    const int g = sms * per;
    char nm[96];
    std::snprintf(nm, sizeof nm, "a grid-stride float4, %d CTAs", g);
    run(nm, [&] { k_a<<<g, 256>>>(reinterpret_cast<float4*>(out), n / 4); });
    std::snprintf(nm, sizeof nm, "b contiguous per CTA float4, %d CTAs", g);
    run(nm, [&] { k_b<<<g, 256>>>(reinterpret_cast<float4*>(out), n / 4); });
  }
  run("e one float4 per thread", [&] { k_e<<<unsigned(n / 4 / 256), 256>>>(reinterpret_cast<float4*>(out), n / 4); });
  run("h four float4 per thread", [&] { k_h<<<unsigned(n / 16 / 256), 256>>>(reinterpret_cast<float4*>(out), n / 4); });
  run("e one float4 per thread, 128 thr", [&] { k_e<<<unsigned(n / 4 / 128), 128>>>(reinterpret_cast<float4*>(out), n / 4); });
  for (int per : {2, 4, 8}) {
    char nm[96];
    std::snprintf(nm, sizeof nm, "f grid-stride st.global.cs, %d CTAs", sms * per);
    run(nm, [&] { k_f<<<sms * per, 256>>>(reinterpret_cast<float4*>(out), n / 4); });
    std::snprintf(nm, sizeof nm, "g grid-stride v8 (32 B) stores, %d CTAs", sms * per);
    run(nm, [&] { k_g<<<sms * per, 256>>>(out, n / 8); });
  }
  run("memset", [&] { cudaMemsetAsync(out, 0, n * 4); });
  unsigned* ctr;
  cudaMalloc(&ctr, 4096 * 4);
  cudaMemset(ctr, 0, 4096 * 4);
  int li = 0;
  cudaFuncSetAttribute(k_tma_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int per : {2, 4, 8}) {
    char nm[96];
    std::snprintf(nm, sizeof nm, "i dynamic 16 KB chunks, %d CTAs", sms * per);
    run(nm, [&] { k_dyn<1024><<<sms * per, 256>>>(reinterpret_cast<float4*>(out), n / 4, ctr + li++); });
    std::snprintf(nm, sizeof nm, "i dynamic 64 KB chunks, %d CTAs", sms * per);
    run(nm, [&] { k_dyn<4096><<<sms * per, 256>>>(reinterpret_cast<float4*>(out), n / 4, ctr + li++); });
  }
  for (int per : {1, 2, 3}) {
    char nm[96];
    std::snprintf(nm, sizeof nm, "j dynamic TMA ring 32 KB chunks, %d CTAs", sms * per);
    run(nm, [&] { k_tma_dyn<<<sms * per, 256, smem>>>(out, n, ctr + li++); });
  }
  for (int per : {1, 2, 3}) {
    const int g = sms * per;
    char nm[96];
    std::snprintf(nm, sizeof nm, "c contiguous per CTA TMA ring, %d CTAs", g);
    run(nm, [&] { k_tma<false><<<g, 256, smem>>>(out, n); });
    std::snprintf(nm, sizeof nm, "d round-robin chunks TMA ring, %d CTAs", g);
    run(nm, [&] { k_tma<true><<<g, 256, smem>>>(out, n); });
  }
  const cudaError_t err = cudaGetLastError();
  std::printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
