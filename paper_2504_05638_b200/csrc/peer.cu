// peer.cu — the exchange's collective as pulls over peer memory (NVLink /
// NVSwitch), no NCCL: every rank encodes into its own owner-major send blocks
// in a region its peers have mapped (CUDA IPC), raises a flag in every peer,
// and each owner reduces its block straight out of the W peers' regions:
//   sketch / raw f32 : sum over ranks in ascending rank order
//                      (the reference's World fold, collectives.cpp:127-166,
//                      so the reduced sketch is bit-identical to it)
//   index u32        : wrapping sum (merge_indices, index.cpp:80-93)
// Flags carry a per-rank step counter kept on the device, so a captured CUDA
// graph replays correctly. Send blocks alternate between two sets per step:
// a rank reuses a set only after every peer has signalled the following step,
// which each peer does after it finished reading that set.
#include "kernels.hpp"

namespace tagc_b200 {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long peer_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread: advance this rank's step counter and publish it to every peer
// after all of this rank's earlier writes (the encoded send blocks).
__global__ void k_peer_signal(PeerView v) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long step = *v.counter + 1;
  *v.counter = step;
  __threadfence_system();
  for (uint32_t q = 0; q < v.world; ++q) st_release_sys(v.flags[q] + v.rank, step);
}

// One CTA: wait until every peer has published this step (bounded: a peer
// that never arrives sets err[2] instead of hanging the device).
__global__ void k_peer_wait(PeerView v, uint32_t* err) {
  const unsigned long long step = *v.counter;
  const unsigned long long t0 = peer_clock();
  for (uint32_t q = threadIdx.x; q < v.world; q += blockDim.x) {
    while (ld_acquire_sys(v.flags[v.rank] + q) < step) {
      if (peer_clock() - t0 > v.timeout_ns) {
        atomicOr(err + 2, 1u);
        break;
      }
      __nanosleep(200);
    }
  }
}

// Owner-side reduction of block `rank` out of the W peers' send sets.
__global__ void __launch_bounds__(256) k_peer_pull(PeerView v, int set, float* __restrict__ recv_f,
                                                   uint32_t* __restrict__ recv_u, const uint32_t* err) {
  if (err[2]) return;  // a peer never arrived: its blocks are not ready
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t nf4 = v.block_f / 4, nu4 = v.block_u / 4;  // blocks are multiples of 32 elements
  for (uint64_t i = tid; i < nf4; i += stride) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t q = 0; q < v.world; ++q) {  // ascending rank order
      const float4 x = __ldcv(reinterpret_cast<const float4*>(v.send_f[set][q] + v.rank * v.block_f) + i);
      acc.x += x.x;
      acc.y += x.y;
      acc.z += x.z;
      acc.w += x.w;
    }
    reinterpret_cast<float4*>(recv_f)[i] = acc;
  }
  for (uint64_t i = tid; i < nu4; i += stride) {
    uint4 acc = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t q = 0; q < v.world; ++q) {
      const uint4 x = __ldcv(reinterpret_cast<const uint4*>(v.send_u[set][q] + v.rank * v.block_u) + i);
      acc.x += x.x;
      acc.y += x.y;
      acc.z += x.z;
      acc.w += x.w;
    }
    reinterpret_cast<uint4*>(recv_u)[i] = acc;
  }
}

}  // namespace

// Force the peer kernels' module to load now: with lazy loading, a first
// launch while another rank of this process spins in k_peer_wait was seen to
// stall (all ranks in one process on one GPU).
void peer_preload() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void*)k_peer_signal);
  cudaFuncGetAttributes(&a, (const void*)k_peer_wait);
  cudaFuncGetAttributes(&a, (const void*)k_peer_pull);
  cudaGetLastError();
}

int launch_peer_exchange(const DevInfo& di, const PeerView& v, int set, float* recv_f, uint32_t* recv_u,
                         uint32_t* err, cudaStream_t stream) {
  k_peer_signal<<<1, 32, 0, stream>>>(v);
  k_peer_wait<<<1, 32, 0, stream>>>(v, err);
  const uint64_t work = std::max(v.block_f, v.block_u) / 4;
  const uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, uint64_t(di.sms) * 4));
  k_peer_pull<<<int(g), 256, 0, stream>>>(v, set, recv_f, recv_u, err);
  return 3;
}

}  // namespace tagc_b200
