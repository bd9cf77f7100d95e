// Tensor-pipe peak probe: the roofline denominator for the attention kernels.
//
// One CTA per SM issues back-to-back tcgen05 MMAs (operands resident in
// shared memory, accumulator in TMEM, no HBM traffic) for the two MMA kinds
// the attention path uses: kind::mxf4nvf4 (NVFP4 block-scaled, K=64) and
// kind::f16 (bf16, K=16), both M=128 N=256 cta_group::1. FLOPs = CTAs x
// rounds x 2*M*N*K; the caller times the launch with CUDA events. This is a
// measurement utility for bench.py, not part of the attention path.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/attnqat_b200.h"
#include "ptx.cuh"

namespace aq {
namespace probe {

constexpr int M = 128, N = 256;
constexpr int kProbeSmemBig = 13 * 1024 + 8 * 12 * 1024;  // SF + 8 operand buffers (A 4 KB + B 8 KB)

__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int kind, int rounds) {
  // A: 128 x 64 fp4 (4 KB) or 128 x 16 bf16 (4 KB); B: 256 rows (8 KB); SF 2 x 512 B
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, bar_end;
  // kinds >= 5 stream operands from NB distinct buffers (no operand reuse) filled
  // with random codes (scales 0x38 = 1.0); kinds < 5 reuse one zero-filled tile
  const bool rnd = kind >= 5;
  for (int i = threadIdx.x; i < (rnd ? kProbeSmemBig : 13 * 1024) / 4; i += blockDim.x) {
    uint32_t x = rnd ? (static_cast<uint32_t>(i) * 2654435761u) ^ 0x5bd1e995u : 0u;
    reinterpret_cast<uint32_t*>(smem)[i] = x;
  }
  if (rnd)
    for (int i = threadIdx.x; i < 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem + 12 * 1024)[i] = 0x38383838u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar_end, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 4096), sf = smem_u32(smem + 12 * 1024);
    tmem_cp_32x128_x4(tmem + 256, smem_desc(sf, 0, 128));
    tmem_cp_32x128_x4(tmem + 264, smem_desc(sf + 512, 0, 128));
    const uint64_t da = smem_desc(a, 2048, 128), db = smem_desc(b, 4096, 128);
    if (kind == 0) {
      const uint32_t id = idesc_nvf4(M, N);
      for (int r = 0; r < rounds; ++r) mma_nvf4_ss(tmem, da, db, id, tmem + 256, tmem + 264, r > 0);
    } else if (kind == 1) {
      const uint32_t id = idesc_f16(M, N, 1, 0, 0);
      for (int r = 0; r < rounds; ++r) mma_f16_ss(tmem, da, db, id, r > 0);
    } else if (kind == 2) {  // NVFP4 M128 N128
      const uint32_t id = idesc_nvf4(M, 128);
      for (int r = 0; r < rounds; ++r) mma_nvf4_ss(tmem, da, db, id, tmem + 256, tmem + 264, r > 0);
    } else if (kind == 3) {  // NVFP4 M128 N128 with a tcgen05.cp of scale factors before each MMA
      const uint32_t id = idesc_nvf4(M, 128);
      for (int r = 0; r < rounds; ++r) {
        tmem_cp_32x128_x4(tmem + 264, smem_desc(sf + 512, 0, 128));
        mma_nvf4_ss(tmem, da, db, id, tmem + 256, tmem + 264, r > 0);
      }
    } else if (kind == 4) {  // round trip: MMA (N128) -> commit -> mbarrier wait, serialized
      const uint32_t id = idesc_nvf4(M, 128);
      for (int r = 0; r < rounds; ++r) {
        mma_nvf4_ss(tmem, da, db, id, tmem + 256, tmem + 264, r > 0);
        tc_commit(&bar);
        mbar_wait(&bar, r & 1);
      }
    }
    else if (kind >= 9) {  // 9/10/11: bf16 N128/N256/N64, 12: nvf4 N64; streaming random operands
      const int n = kind == 10 ? 256 : (kind == 9 ? 128 : 64);
      const uint32_t ob = smem_u32(smem + 13 * 1024);
      const uint32_t idf = idesc_f16(M, n, 1, 0, 0), id4 = idesc_nvf4(M, n);
      for (int r = 0; r < rounds; ++r) {
        const uint32_t o = ob + (r & 7) * 12 * 1024;
        if (kind == 12)
          mma_nvf4_ss(tmem, smem_desc(o, 2048, 128), smem_desc(o + 4096, 4096, 128), id4, tmem + 256, tmem + 264, r > 0);
        else
          mma_f16_ss(tmem, smem_desc(o, 2048, 128), smem_desc(o + 4096, 4096, 128), idf, r > 0);
      }
    }
    else if (kind >= 5) {  // 5: N128, 6: N256, 7: N128 + commit per 2 MMAs, 8: N256 one buffer (random)
      const int n = (kind == 6 || kind == 8) ? 256 : 128;
      const uint32_t id = idesc_nvf4(M, n);
      const uint32_t ob = smem_u32(smem + 13 * 1024);
      for (int r = 0; r < rounds; ++r) {
        const uint32_t o = kind == 8 ? ob : ob + (r & 7) * 12 * 1024;
        mma_nvf4_ss(tmem + ((kind == 7) ? 128 * (r & 1) : 0), smem_desc(o, 2048, 128), smem_desc(o + 4096, 4096, 128), id,
                    tmem + 256, tmem + 264, r > 0);
        if (kind == 7 && (r & 1)) tc_commit(&bar);
      }
    }
    if (kind == 7) {
      tc_commit(&bar_end);
      mbar_wait(&bar_end, 0);
    } else if (kind != 4) {
      tc_commit(&bar);
      mbar_wait(&bar, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace probe
}  // namespace aq

extern "C" {

/* FLOPs executed by one aq_probe_mma_peak launch. kind 0 = NVFP4 (K=64), 1 = bf16 (K=16). */
double aq_probe_mma_flops(int kind, int ctas, int rounds) {
  const double k = (kind == 1 || (kind >= 9 && kind <= 11)) ? 16.0 : 64.0;
  const double n = (kind == 0 || kind == 1 || kind == 6 || kind == 8 || kind == 10) ? 256.0
                   : (kind == 11 || kind == 12) ? 64.0 : 128.0;
  return 2.0 * aq::probe::M * n * k * static_cast<double>(ctas) * rounds;
}

int aq_probe_mma_peak(int kind, int ctas, int rounds, void* stream) {
  const int smem = kind >= 5 ? aq::probe::kProbeSmemBig : 13 * 1024;
  if (kind >= 5) cudaFuncSetAttribute(aq::probe::mma_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  aq::probe::mma_peak_kernel<<<ctas, 128, smem, static_cast<cudaStream_t>(stream)>>>(kind, rounds);
  return cudaGetLastError() == cudaSuccess ? AQ_OK : AQ_E_CUDA;
}

}  // extern "C"
