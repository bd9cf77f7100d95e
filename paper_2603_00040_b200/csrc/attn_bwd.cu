// K6 / K7 / K8: NVFP4 Attn-QAT backward on tcgen05 (sm_100a).
//
// Follows flash_backward (attnqat/flash.py:317-390):
//   D   = rowsum(dO . O_ref), O_ref = O' (CORRECT / NO_FAKE_QUANT_P) or O
//                                                    (flash.py:333-351)   [K6]
//   per key tile j (dK_j, dV_j stationary in TMEM), over query tiles i:
//     S  = Q^F K^F^T / sqrt(d)      FP4 block-scaled MMA, the forward's exact
//                                   instruction sequence (flash.py:372-377)
//     P  = exp(S - L)               shared code with the forward (flash.py:379)
//     P^F = NVFP4(P) if the variant fake-quantizes P     (flash.py:380)
//     dV += P^F^T dO                bf16 MMA            (flash.py:381)
//     dP = dO V^F^T                 bf16 MMA            (flash.py:382)
//     dS = (dP - D) . P / sqrt(d)   unquantized P        (flash.py:383)
//     dQ += dS K^F                  bf16 MMA, tile staged in SMEM and added to
//                                   an fp32 HBM accumulator with one bulk
//                                   reduce-add per (i, j)  (flash.py:384)
//     dK += dS^T Q^F                bf16 MMA            (flash.py:385)      [K7]
//   fp32 dQ accumulator -> output dtype                                      [K8]
//
// CTA = one (head, 128-key tile). 8 compute warps: thread = (query row,
// 64-key half) for S/P/dP/dS, = (row, d/2 columns) for the dQ drain, = (key
// row, d/2 columns) for the dK/dV epilogue. Warp 8 is the producer (1-D bulk
// copies of pre-tiled operands), warp 9 issues the MMAs from one thread.
// TMEM: R1 [0,128) = S_i then dQ_i; dK [128, 128+D); dV [256, 256+D);
// R2 [384, 448) = dP, one 64-key half at a time; scale factors at 448+.
// SMEM: K / K^F / V^F tiles (constant), Q codes (2 stages), Q^F + dO (1
// stage), P^F and dS bf16 tiles (reused as the 64 KB fp32 dQ staging tile).
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "pquant.cuh"
#include "ptx.cuh"

namespace aq {

namespace bwd {

constexpr int NCW = 8;                       // compute warps
constexpr int NUM_THREADS = 32 * (NCW + 2);
constexpr int PRODUCER = NCW, MMA = NCW + 1;
constexpr int HALF = TILE / 2;               // keys per compute thread

template <int D>
struct Smem {
  static constexpr int K_CODES = 0;
  static constexpr int K_SF = K_CODES + TILE * D / 2;
  static constexpr int K_H = K_SF + (D / 64) * 512;
  static constexpr int V_H = K_H + TILE * D * 2;
  static constexpr int QC0 = V_H + TILE * D * 2;                  // Q codes + SF, 2 stages
  static constexpr int QC_BYTES = TILE * D / 2 + (D / 64) * 512;
  static constexpr int Q_H = QC0 + 2 * QC_BYTES;
  static constexpr int DO_H = Q_H + TILE * D * 2;
  static constexpr int P_H = DO_H + TILE * D * 2;                 // P^F bf16 [query][key]
  static constexpr int DS_H = P_H + TILE * TILE * 2;               // dS bf16 [query][key]
  // the fp32 dQ staging tile (128 x D x 4 B <= 64 KB) overlays P^F + dS
  static constexpr int BARS = P_H + 2 * TILE * TILE * 2;
  static constexpr int NUM_BARS = 24;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int TOTAL = TMEM_SLOT + 16;
  static constexpr int K_BYTES = TILE * D / 2 + (D / 64) * 512 + 2 * TILE * D * 2;
  static constexpr int QD_BYTES = 2 * TILE * D * 2;
  static_assert(TOTAL <= 227 * 1024, "shared memory");
};

constexpr uint32_t T_R1 = 0, T_DK = 128, T_DV = 256, T_R2 = 384, T_QSF = 448, T_KSF = 464;

enum Bar {
  B_K = 0, B_QC_FULL = 1, B_QC_EMPTY = 3, B_QD_FULL = 5, B_QD_EMPTY, B_S_FULL, B_S_EMPTY, B_DP_FULL,
  B_DP_EMPTY = B_DP_FULL + 2, B_DS_FULL = B_DP_EMPTY + 2, B_DQ_FULL, B_DQ_EMPTY, B_MMA_I, B_PF_FREE,
  B_STAGE_FREE, B_DONE
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1) attn_bwd_kernel(const BwdParams p) {
  using L = Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::TMEM_SLOT);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int kt = blockIdx.x;
  const int64_t head = blockIdx.y;
  const int k0 = kt * TILE;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const int64_t offset = p.n_k - p.n_q;
  // first query tile with any visible key of this key tile (flash.py:127-128, 366-368)
  int i_begin = 0;
  if (p.causal) {
    const int64_t need = k0 - offset - (TILE - 1);  // q0 >= need
    i_begin = need > 0 ? static_cast<int>(ceil_div(need, TILE)) : 0;
  }
  const int ni = q_tiles > i_begin ? q_tiles - i_begin : 0;

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_K], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[B_QC_FULL + s], 1);
      mbar_init(&bars[B_QC_EMPTY + s], 1);
      mbar_init(&bars[B_DP_FULL + s], 1);
      mbar_init(&bars[B_DP_EMPTY + s], 128);
    }
    mbar_init(&bars[B_QD_FULL], 1);
    mbar_init(&bars[B_QD_EMPTY], 1);
    mbar_init(&bars[B_S_FULL], 1);
    mbar_init(&bars[B_S_EMPTY], 32 * NCW);
    mbar_init(&bars[B_DS_FULL], 32 * NCW);
    mbar_init(&bars[B_DQ_FULL], 1);
    mbar_init(&bars[B_DQ_EMPTY], 32 * NCW);
    mbar_init(&bars[B_MMA_I], 1);
    mbar_init(&bars[B_PF_FREE], 1);
    mbar_init(&bars[B_STAGE_FREE], 32 * NCW);
    mbar_init(&bars[B_DONE], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == PRODUCER) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      const int64_t kidx = head * k_tiles + kt;
      mbar_expect_tx(&bars[B_K], L::K_BYTES);
      bulk_g2s(smem + L::K_CODES, p.k_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, &bars[B_K]);
      bulk_g2s(smem + L::K_SF, p.k_sf + kidx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[B_K]);
      bulk_g2s(smem + L::K_H, p.k_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[B_K]);
      bulk_g2s(smem + L::V_H, p.v_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[B_K]);
      // Q codes run up to two tiles ahead; Q^F + dO are single-buffered
      int iq = 0, id = 0;
      while (id < ni) {
        if (iq < ni && iq <= id + 1) {
          const int s = iq & 1;
          if (iq >= 2) mbar_wait(&bars[B_QC_EMPTY + s], ((iq >> 1) - 1) & 1);
          const int64_t qidx = head * q_tiles + i_begin + iq;
          uint8_t* dst = smem + L::QC0 + s * L::QC_BYTES;
          mbar_expect_tx(&bars[B_QC_FULL + s], L::QC_BYTES);
          bulk_g2s(dst, p.q_codes + qidx * fp4_tile_bytes(D), TILE * D / 2, &bars[B_QC_FULL + s]);
          bulk_g2s(dst + TILE * D / 2, p.q_sf + qidx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[B_QC_FULL + s]);
          ++iq;
          continue;
        }
        if (id > 0) mbar_wait(&bars[B_QD_EMPTY], (id - 1) & 1);
        const int64_t qidx = head * q_tiles + i_begin + id;
        mbar_expect_tx(&bars[B_QD_FULL], L::QD_BYTES);
        bulk_g2s(smem + L::Q_H, p.q_h + qidx * h_tile_bytes(D), TILE * D * 2, &bars[B_QD_FULL]);
        bulk_g2s(smem + L::DO_H, p.do_h + qidx * h_tile_bytes(D), TILE * D * 2, &bars[B_QD_FULL]);
        ++id;
      }
    }
  } else if (warp == MMA) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      const uint32_t id_s = idesc_nvf4(128, 128);
      const uint32_t id_dp = idesc_f16(128, HALF, 1, 0, 0);  // dO (K-major) x V^F half (K-major)
      const uint32_t id_kv = idesc_f16(128, D, 1, 1, 1);     // P^F^T / dS^T (MN) x dO / Q^F (MN)
      const uint32_t id_dq = idesc_f16(128, D, 1, 0, 1);     // dS (K-major) x K^F (MN)
      const uint32_t k_codes = smem_u32(smem + L::K_CODES);
      const uint32_t k_h = smem_u32(smem + L::K_H), v_h = smem_u32(smem + L::V_H);
      const uint32_t q_h = smem_u32(smem + L::Q_H), do_h = smem_u32(smem + L::DO_H);
      const uint32_t p_h = smem_u32(smem + L::P_H), ds_h = smem_u32(smem + L::DS_H);
      mbar_wait(&bars[B_K], 0);
      tc_fence_after();
      for (int ks = 0; ks < D / 64; ++ks)
        tmem_cp_32x128_x4(tmem + T_KSF + 4 * ks, smem_desc(smem_u32(smem + L::K_SF + ks * 512), 0, 128));
      for (int ii = 0; ii < ni; ++ii) {
        const uint32_t ph = ii & 1;
        const int s = ii & 1;
        const uint32_t qc = smem_u32(smem + L::QC0 + s * L::QC_BYTES);
        mbar_wait(&bars[B_QC_FULL + s], (ii >> 1) & 1);
        if (ii > 0) mbar_wait(&bars[B_DQ_EMPTY], (ii - 1) & 1);  // R1 drained
        tc_fence_after();
        for (int ks = 0; ks < D / 64; ++ks)
          tmem_cp_32x128_x4(tmem + T_QSF + 4 * ks, smem_desc(qc + TILE * D / 2 + ks * 512, 0, 128));
        // S = Q K^T (FP4, same instruction sequence as the forward)
        for (int ks = 0; ks < D / 64; ++ks)
          mma_nvf4_ss(tmem + T_R1, smem_desc(qc + ks * 2 * 2048, 2048, 128),
                      smem_desc(k_codes + ks * 2 * 2048, 2048, 128), id_s, tmem + T_QSF + 4 * ks,
                      tmem + T_KSF + 4 * ks, ks > 0);
        tc_commit(&bars[B_S_FULL]);
        tc_commit(&bars[B_QC_EMPTY + s]);
        // dP = dO V^F^T, one 64-key half at a time into R2
        mbar_wait(&bars[B_QD_FULL], ph);
        for (int h = 0; h < 2; ++h) {
          if (ii > 0 || h > 0) mbar_wait(&bars[B_DP_EMPTY + (h ^ 1)], h ? ph : (ph ^ 1));
          tc_fence_after();
          for (int ks = 0; ks < D / 16; ++ks)
            mma_f16_ss(tmem + T_R2, smem_desc(do_h + ks * 2 * 2048, 2048, 128),
                       smem_desc(v_h + h * 8 * 128 + ks * 2 * 2048, 2048, 128), id_dp, ks > 0);
          tc_commit(&bars[B_DP_FULL + h]);
        }
        // dQ_i = dS K^F first (R1: S was read before dS exists) so its drain
        // overlaps dV += P^F^T dO and dK += dS^T Q^F
        mbar_wait(&bars[B_DS_FULL], ph);
        tc_fence_after();
        for (int ks = 0; ks < TILE / 16; ++ks)
          mma_f16_ss(tmem + T_R1, smem_desc(ds_h + ks * 2 * 2048, 2048, 128),
                     smem_desc(k_h + ks * 2 * 128, 128, 2048), id_dq, ks > 0);
        tc_commit(&bars[B_DQ_FULL]);
        for (int ks = 0; ks < TILE / 16; ++ks)
          mma_f16_ss(tmem + T_DV, smem_desc(p_h + ks * 2 * 128, 128, 2048),
                     smem_desc(do_h + ks * 2 * 128, 128, 2048), id_kv, (ii > 0 || ks > 0));
        tc_commit(&bars[B_PF_FREE]);   // P^F buffer free (dQ staging, half 0)
        for (int ks = 0; ks < TILE / 16; ++ks)
          mma_f16_ss(tmem + T_DK, smem_desc(ds_h + ks * 2 * 128, 128, 2048),
                     smem_desc(q_h + ks * 2 * 128, 128, 2048), id_kv, (ii > 0 || ks > 0));
        tc_commit(&bars[B_QD_EMPTY]);
        tc_commit(&bars[B_MMA_I]);     // dS buffer free (dQ staging, half 1)
      }
      tc_commit(&bars[B_DONE]);
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int row = 32 * (warp & 3) + lane;
    const int half = warp >> 2;
    const int kb = half * HALF;   // first key (in tile) of this thread
    const uint32_t t_lane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const float sl2 = p.scale_log2;
    uint8_t* p_h = smem + L::P_H;
    uint8_t* ds_h = smem + L::DS_H;
    for (int ii = 0; ii < ni; ++ii) {
      const uint32_t ph = ii & 1;
      const int64_t q = static_cast<int64_t>(i_begin + ii) * TILE + row;
      const bool qvalid = q < p.n_q;
      const float L2 = qvalid ? p.lse[head * p.n_q + q] * 1.44269504088896340736f : 0.f;
      const float Dq = p.delta[head * (q_tiles * TILE) + q];
      int64_t kmax = p.n_k - 1;
      if (p.causal) kmax = min(kmax, q + offset);
      const int64_t lim = qvalid ? kmax - (k0 + kb) : -1;  // visible keys: c <= lim
      float pr[HALF];
      mbar_wait(&bars[B_S_FULL], ph);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < HALF; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + T_R1 + kb + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) pr[c0 + e] = __uint_as_float(r[e]);
      }
      tc_fence_before();
      mbar_arrive(&bars[B_S_EMPTY]);
      // P = exp(S - L) exactly as the forward computes it
      p_from_s<HALF / 2>(pr, kb, sl2, L2);
      if (lim < HALF - 1) {
#pragma unroll
        for (int c = 0; c < HALF; ++c) pr[c] = (c <= lim) ? pr[c] : 0.f;
      }
      // the previous tile's dQ staging must have been consumed by its bulk reduce
      if (ii > 0) mbar_wait(&bars[B_STAGE_FREE], (ii - 1) & 1);
      // P^F (or P) -> bf16 [query][key] T8x8
#pragma unroll
      for (int blk = 0; blk < HALF / 16; ++blk) {
        uint4 w[2];
        if (p.fq_p) {
          const PBlock qb = quantize_p16(pr + blk * 16);
          __half2 c[4];
          const __half sh = __float2half_rn(qb.sv);
          const __half2 s2 = __halves2half2(sh, sh);
#pragma unroll
          for (int h8 = 0; h8 < 2; ++h8) {
            e2m1x8_to_h2(qb.codes[h8], c);
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(__hmul2(c[e], s2));
              o[e] = pack_bf16(f.x, f.y);
            }
            w[h8] = make_uint4(o[0], o[1], o[2], o[3]);
          }
        } else {
#pragma unroll
          for (int h8 = 0; h8 < 2; ++h8) {
            const float* v = pr + blk * 16 + h8 * 8;
            w[h8] = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                               pack_bf16(v[6], v[7]));
          }
        }
        *reinterpret_cast<uint4*>(p_h + t8x8_off(row, kb + blk * 16)) = w[0];
        *reinterpret_cast<uint4*>(p_h + t8x8_off(row, kb + blk * 16 + 8)) = w[1];
      }
      // dS = (dP - D) . P / sqrt(d) -> bf16
      mbar_wait(&bars[B_DP_FULL + half], ph);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < HALF; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + T_R2 + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int c8 = 0; c8 < 32; c8 += 8) {
          float ds[8];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float2 dd = __fmul2_rn(
                __fadd2_rn(make_float2(__uint_as_float(r[c8 + e]), __uint_as_float(r[c8 + e + 1])),
                           make_float2(-Dq, -Dq)),
                make_float2(pr[c0 + c8 + e] * p.inv_sqrt_d, pr[c0 + c8 + e + 1] * p.inv_sqrt_d));
            ds[e] = dd.x;
            ds[e + 1] = dd.y;
          }
          *reinterpret_cast<uint4*>(ds_h + t8x8_off(row, kb + c0 + c8)) =
              make_uint4(pack_bf16(ds[0], ds[1]), pack_bf16(ds[2], ds[3]), pack_bf16(ds[4], ds[5]),
                         pack_bf16(ds[6], ds[7]));
        }
      }
      tc_fence_before();
      mbar_arrive(&bars[B_DP_EMPTY + half]);
      fence_async_smem();
      mbar_arrive(&bars[B_DS_FULL]);
      // dQ_i: TMEM -> registers, free R1, stage in SMEM once every MMA of
      // this tile is done with P^F / dS, then one bulk reduce-add into HBM
      mbar_wait(&bars[B_DQ_FULL], ph);
      tc_fence_after();
      constexpr int DH = D / 2;
      float dq[DH];
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + T_R1 + half * DH + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) dq[c0 + e] = __uint_as_float(r[e]);
      }
      tc_fence_before();
      mbar_arrive(&bars[B_DQ_EMPTY]);
      // stage this warpgroup's d/2 columns as a contiguous [128][d/2] fp32
      // block (P^F buffer for half 0 once dV is done, dS buffer for half 1
      // once dK is done); dq_acc tiles are [2][128][d/2] with 16-byte chunks
      // XOR-swizzled by (row & 7) (undone by K8), so the 16-byte stores are
      // bank-conflict free and one bulk reduce-add moves each half
      mbar_wait(&bars[half ? B_MMA_I : B_PF_FREE], ph);
      uint8_t* sbase = smem + (half ? L::DS_H : L::P_H);
      uint8_t* srow = sbase + row * (DH * 4);
#pragma unroll
      for (int c4 = 0; c4 < DH / 4; ++c4) {
        const int chunk = c4 ^ (row & 7);
        *reinterpret_cast<float4*>(srow + chunk * 16) =
            make_float4(dq[4 * c4], dq[4 * c4 + 1], dq[4 * c4 + 2], dq[4 * c4 + 3]);
      }
      fence_async_smem();
      named_bar_sync(1 + half, 128);
      if ((threadIdx.x & 127) == 0) {
        float* dst = p.dq_acc + ((head * q_tiles + i_begin + ii) * 2 + half) * static_cast<int64_t>(TILE) * DH;
        bulk_s2g_add_f32(dst, sbase, TILE * DH * 4);
        bulk_commit();
        bulk_wait_read0();
      }
      named_bar_sync(1 + half, 128);
      mbar_arrive(&bars[B_STAGE_FREE]);
    }
    if ((threadIdx.x & 127) == 0) bulk_wait0();
    // epilogue: dK, dV rows (thread = key row, d/2 columns)
    if (ni > 0) {
      mbar_wait(&bars[B_DONE], 0);
      tc_fence_after();
    }
    const int64_t key = k0 + row;
    constexpr int DH = D / 2;
    for (int which = 0; which < 2; ++which) {
      void* dst = which ? p.dv : p.dk;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t r[32];
        if (ni > 0) {
          tmem_ld32(t_lane + (which ? T_DV : T_DK) + half * DH + c0, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = 0u;  // no visible query: zero gradient
        }
        if (key < p.n_k) {
          const int64_t base = (head * p.n_k + key) * D + half * DH + c0;
          if (p.g_dt == 0) {
            float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + base);
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              d4[e / 4] = make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), __uint_as_float(r[e + 2]),
                                      __uint_as_float(r[e + 3]));
          } else {
            uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + base);
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint32_t h[4];
#pragma unroll
              for (int k2 = 0; k2 < 4; ++k2) {
                const float a = __uint_as_float(r[e + 2 * k2]), b = __uint_as_float(r[e + 2 * k2 + 1]);
                if (p.g_dt == 1) {
                  h[k2] = pack_bf16(a, b);
                } else {
                  const __half2 hv = __floats2half2_rn(a, b);
                  h[k2] = *reinterpret_cast<const uint32_t*>(&hv);
                }
              }
              d4[e / 8] = make_uint4(h[0], h[1], h[2], h[3]);
            }
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

// K6: D = rowsum(dO . O_ref) (fp32), dO -> bf16 T8x8 tiles (pad rows zero),
// dQ accumulator [heads][n_pad][d] zeroed. One thread per 8 columns of a row.
__global__ void __launch_bounds__(256) bwd_pre_kernel(const void* d_o, int do_dt, const void* o_ref, int o_dt,
                                                      int64_t heads, int64_t n_q, int d, float* delta, uint8_t* do_h,
                                                      float* dq_acc) {
  const int per_row = d / 8;
  const int64_t q_tiles = ceil_div(n_q, TILE);
  const int64_t rows = heads * q_tiles * TILE;
  const int64_t total = rows * per_row;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(t % per_row);
    const int64_t rp = t / per_row;
    const int64_t h = rp / (q_tiles * TILE);
    const int64_t q = rp % (q_tiles * TILE);
    const bool valid = q < n_q;
    float g[8], o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      g[e] = 0.f;
      o[e] = 0.f;
    }
    if (valid) {
      const int64_t base = (h * n_q + q) * d + c8 * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (do_dt == 1) g[e] = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(d_o)[base + e]);
        else if (do_dt == 2) g[e] = __half2float(reinterpret_cast<const __half*>(d_o)[base + e]);
        else g[e] = reinterpret_cast<const float*>(d_o)[base + e];
        if (o_dt == 1) o[e] = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(o_ref)[base + e]);
        else if (o_dt == 2) o[e] = __half2float(reinterpret_cast<const __half*>(o_ref)[base + e]);
        else o[e] = reinterpret_cast<const float*>(o_ref)[base + e];
      }
    }
    float4* z = reinterpret_cast<float4*>(dq_acc + rp * d + c8 * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = fmaf(g[e], o[e], acc);
    // reduce across the per_row (8 or 16) consecutive lanes of this row
    for (int off = per_row / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (c8 == 0) delta[rp] = acc;
    const int64_t tile = h * q_tiles + q / TILE;
    const uint4 w = make_uint4(pack_bf16(g[0], g[1]), pack_bf16(g[2], g[3]), pack_bf16(g[4], g[5]),
                               pack_bf16(g[6], g[7]));
    *reinterpret_cast<uint4*>(do_h + tile * h_tile_bytes(d) + t8x8_off(static_cast<int>(q % TILE), c8 * 8)) = w;
  }
}

// K8: fp32 dQ accumulator, per 128-query tile two [128][d/2] column halves
// with 16-byte chunks of row q XOR-swizzled by q & 7 -> [heads][n_q][d].
__global__ void __launch_bounds__(256) dq_convert_kernel(const float* src, void* dst, int dt, int64_t heads,
                                                         int64_t n_q, int d) {
  const int64_t n_pad = ceil_div(n_q, TILE) * TILE;
  const int64_t total = heads * n_q * d / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = i * 4;
    const int64_t h = e / (n_q * d), rem = e % (n_q * d);
    const int64_t q = rem / d;
    const int col = static_cast<int>(rem % d), hf = col / (d / 2), c4 = (col % (d / 2)) / 4;
    const int64_t tile = h * (n_pad / TILE) + q / TILE;
    const float4 v = *reinterpret_cast<const float4*>(
        src + ((tile * 2 + hf) * TILE + (q % TILE)) * (d / 2) + ((c4 ^ static_cast<int>(q & 7)) * 4));
    if (dt == 0) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + e) = v;
    } else if (dt == 1) {
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(dst) + e) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
    } else {
      const __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(dst) + e) =
          make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
  }
}

template <int D>
cudaError_t launch(const BwdParams& p, cudaStream_t st) {
  using L = Smem<D>;
  auto kern = attn_bwd_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(ceil_div(p.n_k, TILE)), static_cast<unsigned>(p.heads));
  kern<<<grid, NUM_THREADS, L::TOTAL, st>>>(p);
  return cudaGetLastError();
}

static int grid_for(int64_t work) {
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace bwd

cudaError_t launch_attn_bwd(const BwdParams& p, cudaStream_t st) {
  if (p.d == 64) return bwd::launch<64>(p, st);
  if (p.d == 128) return bwd::launch<128>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_pre(const void* d_o, int do_dt, const void* o_ref, int o_dt, int64_t heads, int64_t n_q,
                           int d, float* delta, uint8_t* do_h, float* dq_acc, cudaStream_t st) {
  const int64_t rows = heads * ceil_div(n_q, TILE) * TILE;
  // per_row threads of a row must sit in one warp: 256-thread blocks, d/8 in {8, 16}
  bwd::bwd_pre_kernel<<<bwd::grid_for(rows * (d / 8)), 256, 0, st>>>(d_o, do_dt, o_ref, o_dt, heads, n_q, d, delta,
                                                                     do_h, dq_acc);
  return cudaGetLastError();
}

cudaError_t launch_dq_convert(const float* dq_acc, void* dq, int g_dt, int64_t heads, int64_t n_q, int d,
                              cudaStream_t st) {
  bwd::dq_convert_kernel<<<bwd::grid_for(heads * n_q * d / 4), 256, 0, st>>>(dq_acc, dq, g_dt, heads, n_q, d);
  return cudaGetLastError();
}

}  // namespace aq
