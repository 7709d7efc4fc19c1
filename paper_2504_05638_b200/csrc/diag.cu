// diag.cu — the reference's per-exchange diagnostics outside the simulated
// world (hook.cpp:171-196):
//   * index_lost / index_spurious: the merged index against the TRUE union of
//     the ranks' supports. With a 1-bit index the union is the OR of every
//     rank's own index words. Over NCCL it travels as one byte per position
//     (k_support_bytes), reduce-scattered with ncclMax (max of 0/1 bytes =
//     OR); over peer memory the owner ORs the peers' send blocks in place.
//   * collect_audit / audit_exchanged_sum: the rank-ordered sum of the
//     exchanged sparse vectors over compressed segments. A rank's sparse value
//     is recovered from the pre-encode combined value and the post-encode
//     residual: sparsify (sparsify.cpp:43, kernels.cpp:95) writes +0.0f into
//     the residual of every kept element and leaves the element itself in it
//     otherwise, so sparse = (bits(residual) == 0) ? combined : +0.0f (a
//     dropped +0.0f gives +0.0f either way).
#include "kernels.hpp"

namespace tagc_b200 {
namespace {

// bit j of word w -> byte 32 w + j (0 or 1)
__global__ void __launch_bounds__(256) k_support_bytes(const uint32_t* __restrict__ words, uint64_t n_words,
                                                       uint8_t* __restrict__ bytes) {
  for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_words;
       w += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t x = words[w];
    uint32_t b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t n = x >> (4 * k);
      b[k] = (n & 1u) | ((n >> 1 & 1u) << 8) | ((n >> 2 & 1u) << 16) | ((n >> 3 & 1u) << 24);
    }
    uint4* dst = reinterpret_cast<uint4*>(bytes + 32 * w);
    dst[0] = make_uint4(b[0], b[1], b[2], b[3]);
    dst[1] = make_uint4(b[4], b[5], b[6], b[7]);
  }
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
  return x;
}

// Width-1 merged words against a support byte map (one byte per position of
// the item, starting at support + 32 * word_off).
__global__ void __launch_bounds__(256) k_index_diag_support(const DiagItem* __restrict__ items,
                                                            const uint8_t* __restrict__ support,
                                                            unsigned long long* __restrict__ out) {
  const DiagItem it = items[blockIdx.y];
  uint32_t lost = 0, spur = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < it.n_words; w += gridDim.x * blockDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(support + 32 * (it.word_off + w));
    const uint4 a = s[0], b = s[1];
    const uint32_t q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t truth = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t v = q[k];
      truth |= (((v & 0xFFu) != 0) | (((v >> 8) & 0xFFu) != 0) << 1 | (((v >> 16) & 0xFFu) != 0) << 2 |
                ((v >> 24) != 0) << 3) << (4 * k);
    }
    const uint64_t first = uint64_t(w) * 32u;
    const uint64_t left = it.n > first ? it.n - first : 0;
    const uint32_t valid = left >= 32 ? 0xFFFFFFFFu : ((1u << left) - 1u);
    const uint32_t present = it.merged[w] & valid;
    truth &= valid;
    lost += __popc(truth & ~present);
    spur += __popc(present & ~truth);
  }
  lost = warp_sum_u32(lost);
  spur = warp_sum_u32(spur);
  if ((threadIdx.x & 31) == 0) {
    if (lost) atomicAdd(&out[2 * blockIdx.y], (unsigned long long)lost);
    if (spur) atomicAdd(&out[2 * blockIdx.y + 1], (unsigned long long)spur);
  }
}

// dst[i] = sum over ranks (ascending) of sparse_r[i], sparse_r recovered
// from comb_r (pre-encode g + acc) and res_r (post-encode residual).
__global__ void __launch_bounds__(256) k_audit(const AuditItem* __restrict__ items,
                                               const float* const* __restrict__ comb,
                                               const float* const* __restrict__ res, uint32_t world) {
  const AuditItem it = items[blockIdx.y];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < it.n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    float acc = 0.0f;
    for (uint32_t r = 0; r < world; ++r) {
      const float c = comb[r][it.src_off + i];
      const uint32_t rb = __float_as_uint(res[r][it.src_off + i]);
      acc += rb == 0u ? c : 0.0f;
    }
    it.dst[i] = acc;
  }
}

}  // namespace

int launch_support_bytes(const uint32_t* words, uint64_t n_words, uint8_t* bytes, cudaStream_t stream) {
  if (!n_words) return 0;
  const uint64_t g = std::min<uint64_t>((n_words + 255) / 256, 148 * 16);
  k_support_bytes<<<unsigned(g), 256, 0, stream>>>(words, n_words, bytes);
  return 1;
}

int launch_index_diag_support(const DiagItem* items, uint32_t n_items, uint32_t max_words,
                              const uint8_t* support, unsigned long long* lost_spurious, cudaStream_t stream) {
  if (!n_items) return 0;
  dim3 grid(std::min<uint32_t>((max_words + 255) / 256, 512), n_items);
  k_index_diag_support<<<grid, 256, 0, stream>>>(items, support, lost_spurious);
  return 1;
}

int launch_audit(const AuditItem* items, uint32_t n_items, uint64_t max_n, const float* const* comb,
                 const float* const* res, uint32_t world, cudaStream_t stream) {
  if (!n_items || !max_n) return 0;
  dim3 grid(std::min<uint64_t>((max_n + 255) / 256, 1024), n_items);
  k_audit<<<grid, 256, 0, stream>>>(items, comb, res, world);
  return 1;
}

// Loads every kernel of this file now (see preload_all_kernels).
void preload_diag_kernels() {
  const void* fns[] = {(const void*)k_audit, (const void*)k_index_diag_support, (const void*)k_support_bytes};
  cudaFuncAttributes a;
  for (const void* f : fns) cudaFuncGetAttributes(&a, f);
  cudaGetLastError();
}

}  // namespace tagc_b200
