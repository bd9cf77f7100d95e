// FP4MM on tcgen05: C = A B^T from NVFP4 QuantTensors (tensors.py:54-86).
//
// The reference decodes both operands and sums, per 16-wide contraction
// block, (sa * sb) * (codes_a . codes_b) in ascending block order. On B200
// that is exactly one block-scaled tensor-core instruction,
// tcgen05.mma.kind::mxf4nvf4.block_scale.block16 (E2M1 operands, UE4M3 scale
// per 16 elements, fp32 accumulation in TMEM); only the fp32 summation order
// across blocks differs from the reference's left-to-right order.
//
//   A   : codes [M][K/2], scales [M][K/16]   (quantize(A), rows blocked along K)
//   B^T : codes [N][K/2], scales [N][K/16]   (quantize(B^T))
//   C   : [M][N] fp32, row stride ldc
//
// Step 1 (HBM-bound byte shuffle): both operands are re-laid into 128-row
// MMA tiles (T8x32 codes + SF512 scale images, layouts.cuh), K zero-padded
// to a multiple of BK (zero codes and zero scales contribute exactly 0).
// Step 2: persistent GEMM, one CTA per SM, 128 x 128 output tiles, K in
// 256-wide slabs through a 5-stage TMA-bulk ring (128-wide slabs in 11
// stages were 5-8 % slower: one commit / barrier round trip per 2 MMAs):
//   warp 0   producer: 1-D bulk copies of the A / B slabs (36 KB per stage)
//   warp 1   MMA issuer: per slab, tcgen05.cp of the 8 scale images into
//            TMEM, then 4 x M128 N128 K64 block-scaled MMAs; commits release
//            the stage and, after the last slab, publish the accumulator
//   warps 2-5 epilogue: TMEM -> registers -> C; two accumulator buffers
//            in TMEM so the epilogue of tile t overlaps the MMAs of tile t+1
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "ptx.cuh"

namespace aq {
namespace gemm {

#ifndef AQ_FP4MM_BK
#define AQ_FP4MM_BK 256
#endif
constexpr int BM = 128, BN = 128, BK = AQ_FP4MM_BK;  // output tile, K slab
// AQ_FP4MM_DIAG (timing diagnostics only, wrong results): 1 = no operand loads,
// 2 = no scale copies / MMAs, 3 = no scale copies, 4 = no C stores
#ifndef AQ_FP4MM_DIAG
#define AQ_FP4MM_DIAG 0
#endif
#ifndef AQ_FP4MM_STAGES
#define AQ_FP4MM_STAGES 5
#endif
constexpr int NST = AQ_FP4MM_STAGES;           // ring stages (bytes in flight per SM = NST x 36 KB)
constexpr int CODE_SLAB = TILE * BK / 2;       // BK/32 K-chunks of a 128-row T8x32 tile
constexpr int SF_SLAB = (BK / 64) * 512;       // BK/64 SF512 images
constexpr int SF_COLS = 8 * (BK / 64);         // TMEM columns of one stage's scales (A then B)
constexpr int STAGE = 2 * (CODE_SLAB + SF_SLAB);
constexpr int BAR0 = NST * STAGE;
constexpr int NUM_BARS = 2 * NST + 4;
constexpr int SMEM = BAR0 + NUM_BARS * 8 + 16;
constexpr int NUM_THREADS = 32 * 6;
constexpr uint32_t T_ACC = 0, T_SF = 256;      // acc buffers [0,128), [128,256); SF_COLS per stage
static_assert(SMEM <= 227 * 1024, "shared memory");
static_assert(T_SF + SF_COLS * NST <= 512, "TMEM columns");

// MX = MXFP4 operands (UE8M0 scale per 32 codes, codec.py:123-166): the same
// code tiles; the SF512 images then hold 4 scales per 128 K (one image per slab).
template <bool MX>
__global__ void __launch_bounds__(256) pack_operand(const uint8_t* __restrict__ codes,
                                                     const uint8_t* __restrict__ scales, int64_t rows, int64_t K,
                                                     int64_t kp, uint8_t* __restrict__ codes_t,
                                                     uint8_t* __restrict__ sf_t) {
  const int64_t nb = kp / 16;
  const int64_t tiles = ceil_div(rows, TILE);
  const int64_t total = tiles * TILE * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = t % nb;
    const int64_t r = t / nb;
    const int64_t tile = r / TILE;
    const int rr = static_cast<int>(r % TILE);
    uint2 c = make_uint2(0u, 0u);
    uint8_t s = 0;
    if (r < rows && b * 16 < K) {
      c = *reinterpret_cast<const uint2*>(codes + r * (K / 2) + b * 8);
      s = MX ? scales[r * (K / 32) + b / 2] : scales[r * (K / 16) + b];
    }
    // T8x32 with 128 rows and kp columns: 32-wide K chunks of 2 KB, K-chunk-major
    const int64_t kk = b * 16;
    *reinterpret_cast<uint2*>(codes_t + tile * (TILE * kp / 2) + (kk >> 5) * (TILE * 16) + (rr >> 3) * 128 +
                              (rr & 7) * 16 + ((kk & 31) >> 1)) = c;
    if (!MX) sf_t[tile * (kp / 64) * 512 + sf512_off(rr, static_cast<int>(b))] = s;
    else if ((b & 1) == 0) sf_t[tile * (kp / 64) * 512 + sf512_off(rr, static_cast<int>(b / 2))] = s;
  }
}

struct GemmParams {
  const uint8_t* a_codes;   // packed tiles
  const uint8_t* a_sf;
  const uint8_t* b_codes;
  const uint8_t* b_sf;
  float* c;
  int64_t M, N, ldc;
  int64_t kp;               // padded K (multiple of BK)
};

template <bool MX>
__global__ void __launch_bounds__(NUM_THREADS, 1) fp4mm_kernel(const GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR0);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* acc_full = bars + 2 * NST;       // 2
  uint64_t* acc_empty = bars + 2 * NST + 2;  // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR0 + NUM_BARS * 8);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int64_t tiles_m = ceil_div(p.M, BM), tiles_n = ceil_div(p.N, BN);
  const int64_t n_tiles = tiles_m * tiles_n;
  const int slabs = static_cast<int>(p.kp / BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    int it = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int64_t tm = t % tiles_m, tn = t / tiles_m;
      for (int s = 0; s < slabs; ++s, ++it) {
        const int st = it % NST;
        if (it >= NST) mbar_wait(&empty[st], ((it / NST) - 1) & 1);
        if (elect_one()) {
          uint8_t* dst = smem + st * STAGE;
          constexpr int SFB = MX ? SF_SLAB / 2 : SF_SLAB;  // scale bytes per operand per slab
#if AQ_FP4MM_DIAG == 1
          mbar_arrive(&full[st]);
          if (false) {
#else
          {
#endif
          mbar_expect_tx(&full[st], 2 * (CODE_SLAB + SFB));
          bulk_g2s(dst, p.a_codes + tm * (TILE * p.kp / 2) + s * CODE_SLAB, CODE_SLAB, &full[st]);
          bulk_g2s(dst + CODE_SLAB, p.a_sf + tm * (p.kp / 64) * 512 + s * SFB, SFB, &full[st]);
          bulk_g2s(dst + CODE_SLAB + SF_SLAB, p.b_codes + tn * (TILE * p.kp / 2) + s * CODE_SLAB, CODE_SLAB,
                   &full[st]);
          bulk_g2s(dst + 2 * CODE_SLAB + SF_SLAB, p.b_sf + tn * (p.kp / 64) * 512 + s * SFB, SFB, &full[st]);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint64_t t_code = desc_template(TILE * 16, 128);  // K-major T8x32, 128 rows
    constexpr uint64_t t_sf = desc_template(0, 128);
    constexpr uint32_t id = idesc_nvf4(BM, BN);
    const uint32_t s0 = smem_u32(smem);
    int it = 0, k = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
      const int ab = k & 1;
      if (k >= 2) mbar_wait(&acc_empty[ab], ((k >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t acc = tmem + T_ACC + ab * BN;
      for (int s = 0; s < slabs; ++s, ++it) {
        const int st = it % NST;
        mbar_wait(&full[st], (it / NST) & 1);
        tc_fence_after();
        const uint32_t base = s0 + st * STAGE;
        const uint32_t a_c = base, a_s = base + CODE_SLAB, b_c = base + CODE_SLAB + SF_SLAB,
                       b_s = base + 2 * CODE_SLAB + SF_SLAB;
        const uint32_t sfa = tmem + T_SF + SF_COLS * st, sfb = sfa + SF_COLS / 2;
        if (elect_one()) {
#if AQ_FP4MM_DIAG == 2
          if (false) {
#else
          if constexpr (MX) {
#endif
            // one image per 128 K: scales of K blocks 0-3 (32 wide); K step ks
            // starts at byte 2 (ks % 2) of each row's 32-bit scale cell
#pragma unroll
            for (int h = 0; h < BK / 128; ++h) {
              tmem_cp_32x128_x4(sfa + 4 * h, desc_at(t_sf, a_s + 512 * h));
              tmem_cp_32x128_x4(sfb + 4 * h, desc_at(t_sf, b_s + 512 * h));
            }
#pragma unroll
            for (int ks = 0; ks < BK / 64; ++ks) {
              const uint32_t sid = 2u * (ks & 1);
              const uint32_t h4 = 4u * (ks >> 1);
              mma_mxf4_ss(acc, desc_at(t_code, a_c + ks * 4096), desc_at(t_code, b_c + ks * 4096),
                          idesc_mxf4(BM, BN, sid), (sfa + h4) | (sid << 30), (sfb + h4) | (sid << 30),
                          (s > 0 || ks > 0));
            }
          } else {
#if AQ_FP4MM_DIAG == 2
            if (false)
#endif
#pragma unroll
            for (int ks = 0; ks < BK / 64; ++ks) {
#if AQ_FP4MM_DIAG == 3
              if (s < 2)
#endif
              tmem_cp_32x128_x4(sfa + 4 * ks, desc_at(t_sf, a_s + ks * 512));
#if AQ_FP4MM_DIAG == 3
              if (s < 2)
#endif
              tmem_cp_32x128_x4(sfb + 4 * ks, desc_at(t_sf, b_s + ks * 512));
            }
#if AQ_FP4MM_DIAG == 2
            if (false)
#endif
#pragma unroll
            for (int ks = 0; ks < BK / 64; ++ks)
              mma_nvf4_ss(acc, desc_at(t_code, a_c + ks * 4096), desc_at(t_code, b_c + ks * 4096), id, sfa + 4 * ks,
                          sfb + 4 * ks, (s > 0 || ks > 0));
          }
          tc_commit(&empty[st]);
          if (s == slabs - 1) tc_commit(&acc_full[ab]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row_in = quad * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    int k = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
      const int ab = k & 1;
      const int64_t tm = t % tiles_m, tn = t / tiles_m;
      mbar_wait(&acc_full[ab], (k >> 1) & 1);
      tc_fence_after();
      const int64_t row = tm * BM + row_in;
      const int64_t col0 = tn * BN;
      float v[32];
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        tmem_ld32f(t_lane + T_ACC + ab * BN + c, v);
        tmem_ld_wait();
        if (c == BN - 32) {
          tc_fence_before();
          mbar_arrive(&acc_empty[ab]);
        }
        if (AQ_FP4MM_DIAG != 4 && row < p.M) {
          float* dst = p.c + row * p.ldc + col0 + c;
          if (col0 + c + 32 <= p.N && (p.ldc % 4) == 0) {
#pragma unroll
            for (int e = 0; e < 32; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (col0 + c + e < p.N) dst[e] = v[e];
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int grid_for(int64_t work) {
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace gemm

int64_t fp4mm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const int64_t kp = ceil_div(K, gemm::BK) * gemm::BK;
  auto op = [&](int64_t rows) { return ceil_div(rows, TILE) * (TILE * kp / 2 + (kp / 64) * 512); };
  return op(M) + op(N) + 1024;
}

cudaError_t launch_fp4mm(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
                         const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, uint8_t* ws,
                         cudaStream_t st, bool mx) {
  using namespace gemm;
  const int64_t kp = ceil_div(K, BK) * BK;
  const int64_t a_codes_b = ceil_div(M, TILE) * (TILE * kp / 2), a_sf_b = ceil_div(M, TILE) * (kp / 64) * 512;
  const int64_t b_codes_b = ceil_div(N, TILE) * (TILE * kp / 2);
  uint8_t* ac = ws;
  uint8_t* as = ac + a_codes_b;
  uint8_t* bc = as + a_sf_b;
  uint8_t* bs = bc + b_codes_b;
  const int ga = grid_for(ceil_div(M, TILE) * TILE * (kp / 16)), gb = grid_for(ceil_div(N, TILE) * TILE * (kp / 16));
  if (mx) {
    pack_operand<true><<<ga, 256, 0, st>>>(a_codes, a_scales, M, K, kp, ac, as);
    pack_operand<true><<<gb, 256, 0, st>>>(b_codes, b_scales, N, K, kp, bc, bs);
  } else {
    pack_operand<false><<<ga, 256, 0, st>>>(a_codes, a_scales, M, K, kp, ac, as);
    pack_operand<false><<<gb, 256, 0, st>>>(b_codes, b_scales, N, K, kp, bc, bs);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  auto kern = mx ? fp4mm_kernel<true> : fp4mm_kernel<false>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  GemmParams p{ac, as, bc, bs, c, M, N, ldc, kp};
  kern<<<grid, NUM_THREADS, SMEM, st>>>(p);
  return cudaGetLastError();
}

}  // namespace aq
