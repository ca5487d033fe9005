// K5: FNV-1a 32-bit feature hashing (H:28-50), bit-exact.
//   hash = 0x811C9DC5; for each byte: hash = (hash ^ byte) * 0x01000193 mod 2^32
//   index = hash & (2^bits - 1)          (hash_feature masks to hash_bits, H:50)
// Input is a packed byte buffer plus int64 offsets (item i = bytes[off[i]:off[i+1]]),
// i.e. the already-joined "field 0x1F token" strings (H:49).  One thread per
// item: items are ~10-30 bytes, so the kernel is bound by the byte stream.
#include "common.cuh"

namespace dffm {

__global__ void __launch_bounds__(256) fnv1a_kernel(const uint8_t* __restrict__ bytes,
                                                     const int64_t* __restrict__ off, int64_t n,
                                                     uint32_t mask, uint32_t* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t b = __ldg(off + i), e = __ldg(off + i + 1);
    uint32_t h = 0x811C9DC5u;
    for (int64_t j = b; j < e; ++j) h = (h ^ (uint32_t)__ldg(bytes + j)) * 0x01000193u;
    out[i] = h & mask;
  }
}

}  // namespace dffm

using namespace dffm;

extern "C" int fw_hash_fnv1a32(const uint8_t* bytes, const int64_t* offsets, int64_t n,
                               int32_t bits, uint32_t* out, void* stream) {
  if (n < 0 || bits < 1 || bits > 32) { set_error("bad hash args (bits=%d)", bits); return DFFM_CONTRACT; }
  if (!n) return DFFM_OK;
  if (!offsets || !out) { set_error("null buffer"); return DFFM_CONTRACT; }
  const uint32_t mask = bits == 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
  const int64_t sms = sm_count_current();
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, sms * 8));
  note_launches(1), fnv1a_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(bytes, offsets, n, mask, out);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(fw_hash_fnv1a32)");
  return DFFM_OK;
}
