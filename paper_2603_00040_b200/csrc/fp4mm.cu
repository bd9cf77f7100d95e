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
// Step 1 (HBM-bound byte shuffle): both operands are re-laid into MMA tiles
// (T8x32 codes + SF512 scale images, layouts.cuh; A in 128-row tiles, B in
// 256-row tiles when N >= 256), K zero-padded to a multiple of BK (zero codes
// and zero scales contribute exactly 0).
// Step 2, N >= 256 (wide::fp4mm_wide_kernel): persistent GEMM, one CTA per SM,
// 128 x 256 output tiles on M128 N256 K64 MMAs (with operands streaming from
// shared memory an N = 128 MMA costs ~65 ns against ~72 ns for N = 256,
// profiles/r02_pipe_probe.txt), K in 256-wide slabs through a 3-4 stage
// TMA-bulk ring:
//   warp 0     producer: 1-D bulk copies of the A / B slabs (54 KB per stage)
//   warp 1     MMA issuer: per slab, tcgen05.cp of 12 scale images into TMEM
//              (B rows 128.. at SFB + 4), then 4 block-scaled MMAs; commits
//              release the stage and, after the last slab, the accumulator
//   warps 2-9  epilogue: one 256-column accumulator (TMEM has no room for two
//              next to the scale factors); two warps per lane quadrant pull
//              128 columns each into registers and release it at once, then
//              store C while the next tile's MMAs run (through shared memory
//              when K <= 8192)
// N < 256 (fp4mm_kernel): 128 x 128 tiles, N128 MMAs, two 128-column
// accumulators, 5-stage ring of 36 KB, four epilogue warps.
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "ptx.cuh"
#include "rowstore.cuh"

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
// code tiles; the SF512 images then hold 4 scales per 128 K (one image per 128 K).
// RT = rows per packed tile (128, or 256 for the wide kernel's B operand): a
// T8x32 tile of RT rows (K-chunk stride RT x 16 bytes) and, per K step, RT / 128
// SF512 images back to back (rows 128.. in the second, the TMEM scale columns
// SFB + 4.. of an N = 256 MMA).
template <bool MX, int RT>
__global__ void __launch_bounds__(256) pack_operand(const uint8_t* __restrict__ codes,
                                                     const uint8_t* __restrict__ scales, int64_t rows, int64_t K,
                                                     int64_t kp, uint8_t* __restrict__ codes_t,
                                                     uint8_t* __restrict__ sf_t) {
  constexpr int NI = RT / 128;  // SF512 images per K step
  const int64_t nb = kp / 16;
  const int64_t tiles = ceil_div(rows, RT);
  const int64_t total = tiles * RT * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = t % nb;
    const int64_t r = t / nb;
    const int64_t tile = r / RT;
    const int rr = static_cast<int>(r % RT);
    uint2 c = make_uint2(0u, 0u);
    uint8_t s = 0;
    if (r < rows && b * 16 < K) {
      c = *reinterpret_cast<const uint2*>(codes + r * (K / 2) + b * 8);
      s = MX ? scales[r * (K / 32) + b / 2] : scales[r * (K / 16) + b];
    }
    // T8x32 with RT rows and kp columns: 32-wide K chunks of RT x 16 bytes, K-chunk-major
    const int64_t kk = b * 16;
    *reinterpret_cast<uint2*>(codes_t + tile * (RT * kp / 2) + (kk >> 5) * (RT * 16) + (rr >> 3) * 128 +
                              (rr & 7) * 16 + ((kk & 31) >> 1)) = c;
    const int kb = MX ? static_cast<int>(b / 2) : static_cast<int>(b);  // scale block index
    if (!MX || (b & 1) == 0)
      sf_t[tile * (kp / 64) * NI * 512 + (kb >> 2) * NI * 512 + (rr >> 7) * 512 + sf512_off(rr & 127, kb & 3)] = s;
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


// ---------------------------------------------------------------------------
// Wide kernel (N >= 256): 128 x 256 output tiles on M128 N256 K64 MMAs.
// With operands streaming from shared memory an M128 MMA costs ~47-65 ns for
// any N <= 128 but ~72 ns at N = 256 (scripts/probe_mma.py,
// profiles/r02_pipe_probe.txt), so N = 256 doubles the work per instruction
// and per A-panel byte. One 256-column accumulator (two would leave no TMEM
// for the scale factors): eight epilogue warps (two per lane quadrant, 128
// columns each) pull it into registers and release it at once, then store
// while the next tile's MMAs run.
namespace wide {
// STG: the epilogue writes C through a swizzled shared-memory stage
// (rowstore.cuh; full 128-byte row segments per store instruction instead of
// one 16-byte store per row and lane), which costs one ring stage. It pays
// when the main loop per tile is short (K <= 8192: 16K x 16K x 4K 0.744 ->
// 0.625 ms) and costs ~6 % at long K (4K x 4K x 16K), so both are built.
constexpr int BN = 256;
constexpr int A_CODES = TILE * BK / 2;                 // 16 KB
constexpr int B_CODES = 2 * TILE * BK / 2;             // 32 KB (one 256-row T8x32 slab)
constexpr int A_SF = (BK / 64) * 512, B_SF = 2 * A_SF; // NVFP4 (MXFP4 uses half)
constexpr int STAGE = A_CODES + B_CODES + A_SF + B_SF;
constexpr int NUM_EPI = 8;
constexpr int NUM_THREADS = 32 * (2 + NUM_EPI);
constexpr int SF_COLS = 12 * (BK / 64);                // per stage: A 4, B 8 columns per K step
constexpr uint32_t T_ACC = 0, T_SF = 256;
template <bool STG>
struct L {
  static constexpr int NST = STG ? 3 : 4;
  static constexpr int EPI_STG = NST * STAGE;         // 32 rows x 32 fp32 per epilogue warp
  static constexpr int BAR0 = EPI_STG + (STG ? NUM_EPI * 32 * 32 * 4 : 0);
  static constexpr int NUM_BARS = 2 * NST + 2;
  static constexpr int SMEM = BAR0 + NUM_BARS * 8 + 16;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(T_SF + SF_COLS * NST <= 512, "TMEM columns");
};

template <bool MX, bool STG>
__global__ void __launch_bounds__(NUM_THREADS, 1) fp4mm_wide_kernel(const GemmParams p) {
  constexpr int NST = L<STG>::NST, EPI_STG = L<STG>::EPI_STG, BAR0 = L<STG>::BAR0, NUM_BARS = L<STG>::NUM_BARS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR0);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* acc_full = bars + 2 * NST;
  uint64_t* acc_empty = bars + 2 * NST + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR0 + NUM_BARS * 8);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int64_t tiles_m = ceil_div(p.M, BM), tiles_n = ceil_div(p.N, BN);
  const int64_t n_tiles = tiles_m * tiles_n;
  const int slabs = static_cast<int>(p.kp / BK);
  constexpr int ASF = MX ? A_SF / 2 : A_SF, BSF = MX ? B_SF / 2 : B_SF;  // scale bytes per slab

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 32 * NUM_EPI);
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
          mbar_expect_tx(&full[st], A_CODES + B_CODES + ASF + BSF);
          bulk_g2s(dst, p.a_codes + tm * (TILE * p.kp / 2) + s * A_CODES, A_CODES, &full[st]);
          bulk_g2s(dst + A_CODES, p.b_codes + tn * (2 * TILE * p.kp / 2) + s * B_CODES, B_CODES, &full[st]);
          bulk_g2s(dst + A_CODES + B_CODES, p.a_sf + tm * (p.kp / 64) * 512 + s * ASF, ASF, &full[st]);
          bulk_g2s(dst + A_CODES + B_CODES + A_SF, p.b_sf + tn * (p.kp / 64) * 1024 + s * BSF, BSF, &full[st]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint64_t t_a = desc_template(TILE * 16, 128);      // K-major T8x32, 128 rows
    constexpr uint64_t t_b = desc_template(2 * TILE * 16, 128);  // K-major T8x32, 256 rows
    constexpr uint64_t t_sf = desc_template(0, 128);
    constexpr uint32_t id = idesc_nvf4(BM, BN);
    const uint32_t s0 = smem_u32(smem);
    int it = 0, k = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
      if (k >= 1) mbar_wait(acc_empty, (k - 1) & 1);
      tc_fence_after();
      for (int s = 0; s < slabs; ++s, ++it) {
        const int st = it % NST;
        mbar_wait(&full[st], (it / NST) & 1);
        tc_fence_after();
        const uint32_t a_c = s0 + st * STAGE, b_c = a_c + A_CODES, a_s = b_c + B_CODES, b_s = a_s + A_SF;
        const uint32_t sfa = tmem + T_SF + SF_COLS * st, sfb = sfa + 4 * (BK / 64);
        if (elect_one()) {
          if constexpr (MX) {
            // one A image and two B images (rows 0-127, 128-255) per 128 K; K step ks
            // starts at byte 2 (ks % 2) of each row's 32-bit scale cell
#pragma unroll
            for (int h = 0; h < BK / 128; ++h) {
              tmem_cp_32x128_x4(sfa + 4 * h, desc_at(t_sf, a_s + 512 * h));
              tmem_cp_32x128_x4(sfb + 8 * h, desc_at(t_sf, b_s + 1024 * h));
              tmem_cp_32x128_x4(sfb + 8 * h + 4, desc_at(t_sf, b_s + 1024 * h + 512));
            }
#pragma unroll
            for (int ks = 0; ks < BK / 64; ++ks) {
              const uint32_t sid = 2u * (ks & 1);
              const uint32_t h = ks >> 1;
              mma_mxf4_ss(tmem + T_ACC, desc_at(t_a, a_c + ks * 4096), desc_at(t_b, b_c + ks * 8192),
                          idesc_mxf4(BM, BN, sid), (sfa + 4 * h) | (sid << 30), (sfb + 8 * h) | (sid << 30),
                          (s > 0 || ks > 0));
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < BK / 64; ++ks) {
              tmem_cp_32x128_x4(sfa + 4 * ks, desc_at(t_sf, a_s + ks * 512));
              tmem_cp_32x128_x4(sfb + 8 * ks, desc_at(t_sf, b_s + ks * 1024));
              tmem_cp_32x128_x4(sfb + 8 * ks + 4, desc_at(t_sf, b_s + ks * 1024 + 512));
            }
#pragma unroll
            for (int ks = 0; ks < BK / 64; ++ks)
              mma_nvf4_ss(tmem + T_ACC, desc_at(t_a, a_c + ks * 4096), desc_at(t_b, b_c + ks * 8192), id,
                          sfa + 4 * ks, sfb + 8 * ks, (s > 0 || ks > 0));
          }
          tc_commit(&empty[st]);
          if (s == slabs - 1) tc_commit(acc_full);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..9)
    const int quad = warp & 3;        // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2; // columns [128 half, 128 half + 128)
    const int row_in = quad * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(quad * 32) << 16) + T_ACC + half * 128;
    int k = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
      const int64_t tm = t % tiles_m, tn = t / tiles_m;
      mbar_wait(acc_full, k & 1);
      tc_fence_after();
      float v[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32f(t_lane + c, v + c);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(acc_empty);
      const int64_t row = tm * BM + row_in;
      const int64_t col0 = tn * BN + half * 128;
      if (STG && col0 + 128 <= p.N && (p.ldc % 4) == 0) {
        const int64_t r0 = tm * BM + quad * 32;
        const int64_t left = p.M - r0;
        uint8_t* stg = smem + EPI_STG + (warp - 2) * (32 * 32 * 4);
#pragma unroll
        for (int c = 0; c < 128; c += 32)
          warp_store_rows<32>(stg, lane, v + c, 1.f, 0, reinterpret_cast<uint8_t*>(p.c + r0 * p.ldc + col0 + c),
                              p.ldc * 4, static_cast<int>(left < 32 ? left : 32));
        continue;
      }
      if (row < p.M) {
        float* dst = p.c + row * p.ldc + col0;
        if (col0 + 128 <= p.N && (p.ldc % 4) == 0) {
#pragma unroll
          for (int e = 0; e < 128; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        } else {
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (col0 + e < p.N) dst[e] = v[e];
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
}  // namespace wide

int grid_for(int64_t work) {
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace gemm

// the wide kernel (B packed in 256-row tiles) runs when N >= 256
static bool fp4mm_wide(int64_t N) { return N >= 256; }

int64_t fp4mm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const int64_t kp = ceil_div(K, gemm::BK) * gemm::BK;
  auto op = [&](int64_t rows, int64_t rt) { return ceil_div(rows, rt) * rt * (kp / 2 + (kp / 64) * 4); };
  return op(M, TILE) + op(N, fp4mm_wide(N) ? 2 * TILE : TILE) + 1024;
}

cudaError_t launch_fp4mm(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
                         const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, uint8_t* ws,
                         cudaStream_t st, bool mx) {
  using namespace gemm;
  const bool wd = fp4mm_wide(N);
  const int64_t rtb = wd ? 2 * TILE : TILE;  // rows per packed B tile
  const int64_t kp = ceil_div(K, BK) * BK;
  const int64_t a_codes_b = ceil_div(M, TILE) * (TILE * kp / 2), a_sf_b = ceil_div(M, TILE) * (kp / 64) * 512;
  const int64_t b_codes_b = ceil_div(N, rtb) * (rtb * kp / 2);
  uint8_t* ac = ws;
  uint8_t* as = ac + a_codes_b;
  uint8_t* bc = as + a_sf_b;
  uint8_t* bs = bc + b_codes_b;
  const int ga = grid_for(ceil_div(M, TILE) * TILE * (kp / 16)), gb = grid_for(ceil_div(N, rtb) * rtb * (kp / 16));
  if (mx) {
    pack_operand<true, TILE><<<ga, 256, 0, st>>>(a_codes, a_scales, M, K, kp, ac, as);
    if (wd) pack_operand<true, 2 * TILE><<<gb, 256, 0, st>>>(b_codes, b_scales, N, K, kp, bc, bs);
    else pack_operand<true, TILE><<<gb, 256, 0, st>>>(b_codes, b_scales, N, K, kp, bc, bs);
  } else {
    pack_operand<false, TILE><<<ga, 256, 0, st>>>(a_codes, a_scales, M, K, kp, ac, as);
    if (wd) pack_operand<false, 2 * TILE><<<gb, 256, 0, st>>>(b_codes, b_scales, N, K, kp, bc, bs);
    else pack_operand<false, TILE><<<gb, 256, 0, st>>>(b_codes, b_scales, N, K, kp, bc, bs);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GemmParams p{ac, as, bc, bs, c, M, N, ldc, kp};
  if (wd) {
    const bool stg = kp <= 8192;
    auto kern = mx ? (stg ? wide::fp4mm_wide_kernel<true, true> : wide::fp4mm_wide_kernel<true, false>)
                   : (stg ? wide::fp4mm_wide_kernel<false, true> : wide::fp4mm_wide_kernel<false, false>);
    const int smem = stg ? wide::L<true>::SMEM : wide::L<false>::SMEM;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int64_t tiles = ceil_div(M, BM) * ceil_div(N, wide::BN);
    const int grid = static_cast<int>(tiles < sms ? tiles : sms);
    kern<<<grid, wide::NUM_THREADS, smem, st>>>(p);
    return cudaGetLastError();
  }
  auto kern = mx ? fp4mm_kernel<true> : fp4mm_kernel<false>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  kern<<<grid, NUM_THREADS, SMEM, st>>>(p);
  return cudaGetLastError();
}

}  // namespace aq
