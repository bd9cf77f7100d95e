// K6 / K7: NVFP4 Attn-QAT backward on tcgen05 (sm_100a).
//
// Follows flash_backward (attnqat/flash.py:317-390):
//   D   = rowsum(dO . O_ref), O_ref = O' (CORRECT / NO_FAKE_QUANT_P) or O
//                                                    (flash.py:333-351)   [K6]
//   S  = Q^F K^F^T / sqrt(d)      FP4 block-scaled MMA, the forward's exact
//                                 instruction sequence (flash.py:372-377)
//   P  = exp(S - L)               shared code with the forward (flash.py:379)
//   P^F = NVFP4(P) if the variant fake-quantizes P     (flash.py:380)
//   dV += P^F^T dO                bf16 MMA            (flash.py:381)
//   dP = dO V^F^T                 bf16 MMA            (flash.py:382)
//   dS = (dP - D) . P / sqrt(d)   unquantized P        (flash.py:383)
//   dQ += dS K^F                  bf16 MMA            (flash.py:384)
//   dK += dS^T Q^F                bf16 MMA            (flash.py:385)
//
// Two roles, each owning its accumulators in TMEM for the whole reduction, so
// no gradient goes through atomics or an fp32 HBM accumulator and every
// gradient is deterministic:
//  * KV role: CTA = (head, 128-key tile); dK, dV stationary while it loops
//    over query tiles (the reference's key-outer loop, flash.py:360-365);
//  * Q role:  CTA = (head, 128-query tile); dQ stationary while it loops over
//    key tiles, recomputing S, P, dP, dS (dQ does not need P^F).
// Both run in one launch (attn_bwd_kernel). Each CTA: compute warps (thread =
// query row x KPT keys, Cfg<D>), one producer warp (1-D bulk copies of
// pre-tiled operands), one MMA warp (warp-uniform schedule; one elected lane
// issues tcgen05.cp / mma / commit).
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "pquant.cuh"
#include "ptx.cuh"

namespace aq {

namespace bwd {

// Tuning aid (-DAQ_BWD_PROFILE): cycle sums per compute-warp segment, lane 0
// of every compute warp; [0..7] KV role, [8..13] Q role, [14] KV tiles, [15] Q tiles.
__device__ unsigned long long g_bprof[16];
#ifdef AQ_BWD_PROFILE
// per-CTA timeline (globaltimer ns): [0] entry, [1] first S in registers
// (compute warp 0), [2] tile loop done, [3] exit, [4] smid | role << 16 | tiles << 32
constexpr int kTimelineCtas = 32768;
__device__ unsigned long long g_btl[kTimelineCtas][5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int64_t tl_cta() { return static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x; }
#define AQ_TL(slot) do { if (threadIdx.x == 0 && tl_cta() < kTimelineCtas) g_btl[tl_cta()][slot] = gtimer(); } while (0)
#else
#define AQ_TL(slot) do { } while (0)
#endif
#ifdef AQ_BWD_PROFILE
#define AQ_BPROF(...) __VA_ARGS__
#else
#define AQ_BPROF(...)
#endif

// Compute warps: 4 TMEM row groups x NKG key groups. 16 warps hide more
// latency but cap registers at 96/thread: d=64 gains 9%, d=128 loses 2%
// (spills), so the count is per head dim.
template <int D>
struct Cfg {
  static constexpr int NCW = D == 64 ? 16 : 8;
  static constexpr int NKG = NCW / 4;
  static constexpr int KPT = TILE / NKG;     // keys per compute thread
  static constexpr int NUM_THREADS = 32 * (NCW + 2);
  static constexpr int PRODUCER = NCW, MMA = NCW + 1;
};
// The KV role computes dP_i as one N=128 product into the S columns once S_i
// is in registers (S_{i+1} follows once dP_i is). Until round 2 it ran two N=64
// halves in a 64-column buffer; with operands streaming from shared memory an
// N=64 bf16 MMA costs as long as an N=128 one (~49 vs ~50 ns per K16 step,
// scripts/probe_mma.py), so the halves doubled dP's tensor time.
// AQ_BWD_PAIR=1: a KV CTA runs two key tiles of its head (see bwd_kv_tile).
// Measured at C4 it is 5 % slower (3.62 -> 3.82 ms): the paired CTAs' tile
// loops ran ~5 % slower per tile and the item switch was not hidden, so the
// default launch keeps one key tile per CTA (the item loop then runs once).
#ifndef AQ_BWD_PAIR
#define AQ_BWD_PAIR 0
#endif

// N consecutive fp32 columns of this warp's TMEM lanes
template <int N>
__device__ __forceinline__ void tmem_load_f(uint32_t taddr, float* v) {
  if constexpr (N % 32 == 0) {
#pragma unroll
    for (int c = 0; c < N; c += 32) tmem_ld32f(taddr + c, v + c);
    tmem_ld_wait();
  } else {
    static_assert(N == 16, "TMEM load width");
    uint32_t r[16];
    tmem_ld16(taddr, r);
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}
// 16-bit pair in the MMA operand format: fp16 (f16 = true, the PLAIN instance's
// fp16 mode) or bf16
__device__ __forceinline__ uint32_t pack16(float a, float b, bool f16) {
  if (f16) {
    const __half2 v = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
  }
  return pack_bf16(a, b);
}

// N consecutive fp32 values -> dst[base, base+N) in dtype dt (0 fp32, 1 bf16, 2 fp16)
template <int N>
__device__ __forceinline__ void store_run(void* dst, int64_t base, int dt, float* v, float mul = 1.f) {
  if (mul != 1.f) {  // per-tensor scale of the other operand (two-level NVFP4; 1 = reference)
#pragma unroll
    for (int e = 0; e < N; ++e) v[e] *= mul;
  }
  if (dt == 0) {
    float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + base);
#pragma unroll
    for (int e = 0; e < N; e += 4) d4[e / 4] = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
  } else {
    uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + base);
#pragma unroll
    for (int e = 0; e < N; e += 8) {
      uint32_t h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (dt == 1) {
          h[k] = pack_bf16(v[e + 2 * k], v[e + 2 * k + 1]);
        } else {
          const __half2 hv = __floats2half2_rn(v[e + 2 * k], v[e + 2 * k + 1]);
          h[k] = *reinterpret_cast<const uint32_t*>(&hv);
        }
      }
      d4[e / 8] = make_uint4(h[0], h[1], h[2], h[3]);
    }
  }
}

// dS = (dP - D) . P / sqrt(d) for a KPT-key run -> bf16 [query][key] T8x8
template <int KPT>
__device__ __forceinline__ void store_ds(uint8_t* ds_h, int row, int kb, const float* dp, const float* pr, float Dq,
                                         float inv_sqrt_d, bool f16 = false) {
#pragma unroll
  for (int c8 = 0; c8 < KPT; c8 += 8) {
    float ds[8];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float2 dd =
          __fmul2_rn(__fadd2_rn(make_float2(dp[c8 + e], dp[c8 + e + 1]), make_float2(-Dq, -Dq)),
                     make_float2(pr[c8 + e] * inv_sqrt_d, pr[c8 + e + 1] * inv_sqrt_d));
      ds[e] = dd.x;
      ds[e + 1] = dd.y;
    }
    *reinterpret_cast<uint4*>(ds_h + t8x8_off(row, kb + c8)) =
        make_uint4(pack16(ds[0], ds[1], f16), pack16(ds[2], ds[3], f16), pack16(ds[4], ds[5], f16),
                   pack16(ds[6], ds[7], f16));
  }
}

// ============================================================================ K7a: dK, dV
// PLAIN (quantized=False, flash.py:344-349): S from 16-bit Q / K tiles on
// kind::f16; the Q ring then carries bf16 Q tiles that serve both S and dK
// (no separate Q^F stage) and the stationary K is a bf16 tile; one dO stage
// keeps the layout inside 227 KB.
template <int D, bool PLAIN = false>
struct KvSmem {
  static constexpr int K_CODES = 0;                                // FP4 K (bf16 K tile for PLAIN)
  static constexpr int K_SF = K_CODES + TILE * D / 2;
  static constexpr int V_H = PLAIN ? TILE * D * 2 : K_SF + (D / 64) * 512;
  static constexpr int QC0 = V_H + TILE * D * 2;                  // Q codes + SF (bf16 Q for PLAIN), 2 stages
  static constexpr int QC_BYTES = PLAIN ? TILE * D * 2 : TILE * D / 2 + (D / 64) * 512;
  static constexpr int Q_H = QC0 + 2 * QC_BYTES;                  // Q^F, 1 stage (none for PLAIN)
  static constexpr int NDO = PLAIN ? 1 : 2;
  static constexpr int DO_H0 = Q_H + (PLAIN ? 0 : TILE * D * 2);   // dO, NDO stages
  static constexpr int P_H = DO_H0 + NDO * TILE * D * 2;          // P^F bf16 [query][key]
  static constexpr int DS_H = P_H + TILE * TILE * 2;               // dS bf16 [query][key]
  static constexpr int BARS = DS_H + TILE * TILE * 2;
  static constexpr int NUM_BARS = 24;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int TOTAL = TMEM_SLOT + 16;
  static constexpr int K_BYTES = TILE * D / 2 + (D / 64) * 512 + TILE * D * 2;
  static_assert(TOTAL <= 227 * 1024, "shared memory");
};

// TMEM: S and dP (one after the other) [0,128); dK [128,128+D); dV [256,256+D); SF 448+
constexpr uint32_t KV_T_S = 0, KV_T_DK = 128, KV_T_DV = 256, KV_T_QSF = 448, KV_T_KSF = 464;

enum KvBar {
  KV_B_K = 0, KV_B_QC_FULL = 1, KV_B_QC_EMPTY = 3, KV_B_DO_FULL = 5, KV_B_DO_EMPTY = 7, KV_B_QH_FULL = 9,
  KV_B_QH_EMPTY, KV_B_S_FULL, KV_B_S_EMPTY, KV_B_DP_FULL, KV_B_DP_EMPTY = KV_B_DP_FULL + 2,
  KV_B_PF_FULL = KV_B_DP_EMPTY + 2, KV_B_PF_FREE, KV_B_DS_FULL, KV_B_DS_FREE, KV_B_DONE, KV_B_V, KV_B_DV_DONE
};

// Schedule per query tile i (MMA warp, in issue order):
//   dP_i (N=128, into S's columns once S_i is read) | S_{i+1} (once dP_i is read) |
//   dV_i (once P^F_i is in SMEM) | dK_i (once dS_i is)
// so dP_i runs under the P / P^F computation and S_{i+1} under dS_i; the Q
// codes / dO / Q^F rings are released by the MMA that last reads them.
// A CTA may run a second key tile kt2 of the same head after kt (kt2 >= 0):
// every ring and barrier phase continues across the two items (g = tile count
// of the CTA); the second item's K / V are loaded once the first item's MMAs
// are done, and its first S / dP run while the compute warps store the first
// item's dK / dV, so the second item pays no launch gap and no ramp.
template <int D, bool MX, bool PLAIN>
__device__ __forceinline__ void bwd_kv_tile(const BwdParams& p, uint8_t* smem, int kt, int64_t head, int kt2 = -1) {
  using L = KvSmem<D, PLAIN>;
  constexpr int NDO = L::NDO;
  constexpr int NCW = Cfg<D>::NCW, NKG = Cfg<D>::NKG, KPT = Cfg<D>::KPT;
  constexpr int PRODUCER = Cfg<D>::PRODUCER, MMA = Cfg<D>::MMA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::TMEM_SLOT);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const int64_t offset = p.n_k - p.n_q;
  const int nit = kt2 >= 0 ? 2 : 1;
  // first query tile with any visible key of key tile t (flash.py:127-128, 366-368)
  auto first_q = [&](int t) {
    if (!p.causal) return 0;
    const int64_t need = static_cast<int64_t>(t) * TILE - offset - (TILE - 1);  // q0 >= need
    return need > 0 ? static_cast<int>(ceil_div(need, TILE)) : 0;
  };
  // per-item state (item 0 here; every role switches to item 1 in its own loop)
  int k0 = kt * TILE, i_begin = first_q(kt);
  int ni = q_tiles > i_begin ? q_tiles - i_begin : 0;
  int64_t kidx = head * k_tiles + kt;
  auto set_item = [&](int it) {
    const int t = it ? kt2 : kt;
    k0 = t * TILE;
    i_begin = first_q(t);
    ni = q_tiles > i_begin ? q_tiles - i_begin : 0;
    kidx = head * k_tiles + t;
  };
  if (threadIdx.x == 32 * PRODUCER) {
    mbar_init(&bars[KV_B_K], 1);
    mbar_init(&bars[KV_B_V], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[KV_B_QC_FULL + s], 1);
      mbar_init(&bars[KV_B_QC_EMPTY + s], 1);
      mbar_init(&bars[KV_B_DO_FULL + s], 1);
      mbar_init(&bars[KV_B_DO_EMPTY + s], 1);
      mbar_init(&bars[KV_B_DP_FULL + s], 1);
      mbar_init(&bars[KV_B_DP_EMPTY + s], 32 * NCW);
    }
    mbar_init(&bars[KV_B_QH_FULL], 1);
    mbar_init(&bars[KV_B_QH_EMPTY], 1);
    mbar_init(&bars[KV_B_S_FULL], 1);
    mbar_init(&bars[KV_B_S_EMPTY], 32 * NCW);
    mbar_init(&bars[KV_B_PF_FULL], 32 * NCW);
    mbar_init(&bars[KV_B_PF_FREE], 1);
    mbar_init(&bars[KV_B_DS_FULL], 32 * NCW);
    mbar_init(&bars[KV_B_DS_FREE], 1);
    mbar_init(&bars[KV_B_DONE], 1);
    mbar_init(&bars[KV_B_DV_DONE], 1);
    fence_mbar_init();
    // the stationary K / V^F tiles and the first query tile are requested
    // before the CTA-wide sync, so their latency overlaps TMEM allocation.
    // K (first S) and V^F (first dP) on separate barriers.
    if (PLAIN) {
      mbar_expect_tx(&bars[KV_B_K], TILE * D * 2);
      bulk_g2s(smem + L::K_CODES, p.k_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_K]);
    } else {
      mbar_expect_tx(&bars[KV_B_K], TILE * D / 2 + (D / 64) * 512);
      bulk_g2s(smem + L::K_CODES, p.k_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, &bars[KV_B_K]);
      bulk_g2s(smem + L::K_SF, p.k_sf + kidx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[KV_B_K]);
    }
    if (ni > 0) {
      const int64_t qidx = head * q_tiles + i_begin;
      mbar_expect_tx(&bars[KV_B_QC_FULL], L::QC_BYTES);
      if (PLAIN) {
        bulk_g2s(smem + L::QC0, p.q_h + qidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_QC_FULL]);
      } else {
        bulk_g2s(smem + L::QC0, p.q_codes + qidx * fp4_tile_bytes(D), TILE * D / 2, &bars[KV_B_QC_FULL]);
        bulk_g2s(smem + L::QC0 + TILE * D / 2, p.q_sf + qidx * sf_tile_bytes_qk(D), (D / 64) * 512,
                 &bars[KV_B_QC_FULL]);
      }
    }
    mbar_expect_tx(&bars[KV_B_V], TILE * D * 2);
    bulk_g2s(smem + L::V_H, p.v_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_V]);
    if (ni > 0) {
      const int64_t qidx = head * q_tiles + i_begin;
      mbar_expect_tx(&bars[KV_B_DO_FULL], TILE * D * 2);
      bulk_g2s(smem + L::DO_H0, p.do_h + qidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_DO_FULL]);
    }
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == PRODUCER) {
    // ------------------------------------------------------------ producer
    // (K, V^F and query tile 0 were requested before the CTA-wide sync)
    auto load_qc = [&](int t, int64_t qidx) {  // t: ring position (tile count of the CTA)
      const int s = t & 1;
      if (t >= 2) mbar_wait(&bars[KV_B_QC_EMPTY + s], ((t >> 1) - 1) & 1);
      if (elect_one()) {
        uint8_t* dst = smem + L::QC0 + s * L::QC_BYTES;
        mbar_expect_tx(&bars[KV_B_QC_FULL + s], L::QC_BYTES);
        if (PLAIN) {
          bulk_g2s(dst, p.q_h + qidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_QC_FULL + s]);
        } else {
          bulk_g2s(dst, p.q_codes + qidx * fp4_tile_bytes(D), TILE * D / 2, &bars[KV_B_QC_FULL + s]);
          bulk_g2s(dst + TILE * D / 2, p.q_sf + qidx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[KV_B_QC_FULL + s]);
        }
      }
      __syncwarp();
    };
    auto load_do = [&](int t, int64_t qidx) {
      const int s = t % NDO;
      if (t >= NDO) mbar_wait(&bars[KV_B_DO_EMPTY + s], ((t / NDO) - 1) & 1);
      if (elect_one()) {
        mbar_expect_tx(&bars[KV_B_DO_FULL + s], TILE * D * 2);
        bulk_g2s(smem + L::DO_H0 + s * TILE * D * 2, p.do_h + qidx * h_tile_bytes(D), TILE * D * 2,
                 &bars[KV_B_DO_FULL + s]);
      }
      __syncwarp();
    };
    int g = 0;
    for (int it = 0; it < nit; ++it) {
      if (it > 0) {
        set_item(it);
        // K / V^F of this item replace the previous item's once all its MMAs are done
        mbar_wait(&bars[KV_B_DONE], (it - 1) & 1);
        if (elect_one()) {
          if (PLAIN) {
            mbar_expect_tx(&bars[KV_B_K], TILE * D * 2);
            bulk_g2s(smem + L::K_CODES, p.k_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_K]);
          } else {
            mbar_expect_tx(&bars[KV_B_K], TILE * D / 2 + (D / 64) * 512);
            bulk_g2s(smem + L::K_CODES, p.k_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, &bars[KV_B_K]);
            bulk_g2s(smem + L::K_SF, p.k_sf + kidx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[KV_B_K]);
          }
          mbar_expect_tx(&bars[KV_B_V], TILE * D * 2);
          bulk_g2s(smem + L::V_H, p.v_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_V]);
        }
        __syncwarp();
      }
      for (int t = 0; t < ni; ++t, ++g) {
        // the next query tile: this item's, or the next item's first (the rings run on)
        if (t + 1 < ni) {
          load_qc(g + 1, head * q_tiles + i_begin + t + 1);
          load_do(g + 1, head * q_tiles + i_begin + t + 1);
        } else if (it + 1 < nit) {
          const int ib = first_q(kt2);
          if (ib < q_tiles) {
            load_qc(g + 1, head * q_tiles + ib);
            load_do(g + 1, head * q_tiles + ib);
          }
        }
        if (PLAIN) continue;  // the Q ring slot is the dK operand too
        if (g > 0) mbar_wait(&bars[KV_B_QH_EMPTY], (g - 1) & 1);
        const int64_t qidx = head * q_tiles + i_begin + t;
        if (elect_one()) {
          mbar_expect_tx(&bars[KV_B_QH_FULL], TILE * D * 2);
          bulk_g2s(smem + L::Q_H, p.q_h + qidx * h_tile_bytes(D), TILE * D * 2, &bars[KV_B_QH_FULL]);
        }
        __syncwarp();
      }
    }
  } else if (warp == MMA) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_nvf4(128, 128);
    // 16-bit operand format: bf16, or the PLAIN instance's p.plain_fmt (0 = fp16)
    const uint32_t f16f = PLAIN ? static_cast<uint32_t>(p.plain_fmt) : 1u;
    const uint32_t id_s16 = idesc_f16(128, 128, f16f, 0, 0);  // PLAIN: Q (K-major) x K (K-major)
    const uint32_t id_dp = idesc_f16(128, TILE, f16f, 0, 0);  // dO (K-major) x V^F (K-major)
    const uint32_t id_kv = idesc_f16(128, D, f16f, 1, 1);     // P^F^T / dS^T (MN) x dO / Q^F (MN)
    constexpr uint64_t t_fp4 = desc_template(2048, 128);        // FP4 codes, K-major T8x32
    constexpr uint64_t t_sf = desc_template(0, 128);
    constexpr uint64_t t_kmaj = desc_template(2048, 128);       // bf16 T8x8 read K-major
    constexpr uint64_t t_mn = desc_template(128, 2048);         // bf16 T8x8 read MN-major
    const uint32_t s0 = smem_u32(smem);
    const uint32_t k_codes = s0 + L::K_CODES, v_h = s0 + L::V_H;
    const uint32_t q_h = s0 + L::Q_H, p_h = s0 + L::P_H, ds_h = s0 + L::DS_H;
    auto issue_s = [&](int i) {
      const int s = i & 1;
      const uint32_t qc = s0 + L::QC0 + s * L::QC_BYTES;
      mbar_wait(&bars[KV_B_QC_FULL + s], (i >> 1) & 1);
      // the caller has waited for dP_{i-1} to be read (it shares S's columns)
      tc_fence_after();
      if (elect_one()) {
        // S = Q K^T (FP4, same instruction sequence as the forward)
        if constexpr (PLAIN) {
          for (int ks = 0; ks < D / 16; ++ks)
            mma_f16_ss(tmem + KV_T_S, desc_at(t_kmaj, qc + ks * 4096), desc_at(t_kmaj, k_codes + ks * 4096), id_s16,
                       ks > 0);
        } else if constexpr (MX) {
          tmem_cp_32x128_x4(tmem + KV_T_QSF, desc_at(t_sf, qc + TILE * D / 2));
          for (int ks = 0; ks < D / 64; ++ks) {
            const uint32_t sid = 2u * ks;
            mma_mxf4_ss(tmem + KV_T_S, desc_at(t_fp4, qc + ks * 4096), desc_at(t_fp4, k_codes + ks * 4096),
                        idesc_mxf4(128, 128, sid), (tmem + KV_T_QSF) | (sid << 30), (tmem + KV_T_KSF) | (sid << 30),
                        ks > 0);
          }
        } else {
          for (int ks = 0; ks < D / 64; ++ks)
            tmem_cp_32x128_x4(tmem + KV_T_QSF + 4 * ks, desc_at(t_sf, qc + TILE * D / 2 + ks * 512));
          for (int ks = 0; ks < D / 64; ++ks)
            mma_nvf4_ss(tmem + KV_T_S, desc_at(t_fp4, qc + ks * 4096), desc_at(t_fp4, k_codes + ks * 4096), id_s,
                        tmem + KV_T_QSF + 4 * ks, tmem + KV_T_KSF + 4 * ks, ks > 0);
        }
        tc_commit(&bars[KV_B_S_FULL]);
        if (!PLAIN) tc_commit(&bars[KV_B_QC_EMPTY + s]);  // PLAIN: released by dK
      }
      __syncwarp();
    };
    auto issue_dp = [&](int i, int h, uint32_t do_h) {
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < D / 16; ++ks)
          mma_f16_ss(tmem + KV_T_S, desc_at(t_kmaj, do_h + ks * 4096), desc_at(t_kmaj, v_h + h * 1024 + ks * 4096),
                     id_dp, ks > 0);
        tc_commit(&bars[KV_B_DP_FULL + h]);
      }
      __syncwarp();
    };
    int g = 0;  // tile count of the CTA: ring slots and barrier phases run on across items
    for (int it = 0; it < nit; ++it) {
      if (it > 0) set_item(it);
      mbar_wait(&bars[KV_B_K], it & 1);
      // S's columns: the previous item's last dP has been read (S_0 overwrites them)
      if (g > 0) mbar_wait(&bars[KV_B_DP_EMPTY], (g - 1) & 1);
      tc_fence_after();
      if (!PLAIN && elect_one()) {  // after the previous item's S MMAs in the pipe
        for (int ks = 0; ks < D / 64; ++ks)
          tmem_cp_32x128_x4(tmem + KV_T_KSF + 4 * ks, desc_at(t_sf, s0 + L::K_SF + ks * 512));
      }
      __syncwarp();
      if (ni > 0) issue_s(g);
      for (int ii = 0; ii < ni; ++ii, ++g) {
        const uint32_t ph = g & 1;
        const int s = g % NDO;
        const uint32_t do_h = s0 + L::DO_H0 + s * TILE * D * 2;
        mbar_wait(&bars[KV_B_DO_FULL + s], (g / NDO) & 1);
        // dP_i (N = 128) into S's columns once every compute warp holds S_i; S_{i+1}
        // once every compute warp holds dP_i
        if (ii == 0) mbar_wait(&bars[KV_B_V], it & 1);
        mbar_wait(&bars[KV_B_S_EMPTY], ph);
        issue_dp(g, 0, do_h);
        if (ii + 1 < ni) {
          mbar_wait(&bars[KV_B_DP_EMPTY], ph);
          issue_s(g + 1);
        }
        // dV += P^F^T dO (the item's first dV overwrites: the compute warps read the
        // previous item's dV before they produced this P^F)
        mbar_wait(&bars[KV_B_PF_FULL], ph);
        tc_fence_after();
        if (elect_one()) {
          for (int ks = 0; ks < TILE / 16; ++ks)
            mma_f16_ss(tmem + KV_T_DV, desc_at(t_mn, p_h + ks * 256), desc_at(t_mn, do_h + ks * 256), id_kv,
                       (ii > 0 || ks > 0));
          tc_commit(&bars[KV_B_PF_FREE]);
          tc_commit(&bars[KV_B_DO_EMPTY + s]);
          if (ii == ni - 1) tc_commit(&bars[KV_B_DV_DONE]);  // dV final: its epilogue overlaps the last dK
        }
        __syncwarp();
        // dK += dS^T Q^F (PLAIN: Q from its ring slot, already waited for by S_i)
        mbar_wait(&bars[KV_B_DS_FULL], ph);
        if (!PLAIN) mbar_wait(&bars[KV_B_QH_FULL], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t qf = PLAIN ? s0 + L::QC0 + (g & 1) * L::QC_BYTES : q_h;
          for (int ks = 0; ks < TILE / 16; ++ks)
            mma_f16_ss(tmem + KV_T_DK, desc_at(t_mn, ds_h + ks * 256), desc_at(t_mn, qf + ks * 256), id_kv,
                       (ii > 0 || ks > 0));
          tc_commit(&bars[KV_B_DS_FREE]);
          tc_commit(&bars[PLAIN ? KV_B_QC_EMPTY + (g & 1) : KV_B_QH_EMPTY]);
        }
        __syncwarp();
      }
      if (elect_one()) {
        if (ni == 0) tc_commit(&bars[KV_B_DV_DONE]);  // one DV_DONE / DONE phase per item
        tc_commit(&bars[KV_B_DONE]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ compute warps
    const int row = 32 * (warp & 3) + lane;
    const int kg = warp >> 2;
    const int kb = kg * KPT;      // first key (in tile) of this thread
    const uint32_t t_lane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const float sl2 = p.scale_log2;
    const bool f16 = PLAIN && p.plain_fmt == 0;  // fp16 operand tiles (PLAIN fp16 mode)
    uint8_t* p_h = smem + L::P_H;
    uint8_t* ds_h = smem + L::DS_H;
    AQ_BPROF(unsigned long long pr_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long tq_ = clock64();)
    // per-row L and D of the next query tile are loaded one tile ahead, so the
    // global-load latency never sits between S_FULL and the exponentials
    auto row_stats = [&](int t, float& l2, float& dq) {
      const int64_t qq = static_cast<int64_t>(i_begin + t) * TILE + row;
      l2 = (t < ni && qq < p.n_q) ? p.lse[head * p.n_q + qq] : 0.f;
      dq = t < ni ? p.delta[head * (q_tiles * TILE) + qq] : 0.f;
    };
    int g = 0;  // tile count of the CTA (barrier phases run on across items)
    for (int it = 0; it < nit; ++it) {
    if (it > 0) set_item(it);
    float L_next, D_next;
    row_stats(0, L_next, D_next);
    for (int ii = 0; ii < ni; ++ii, ++g) {
      const uint32_t ph = g & 1;
      const int64_t q = static_cast<int64_t>(i_begin + ii) * TILE + row;
      const bool qvalid = q < p.n_q;
      const float L2 = L_next * 1.44269504088896340736f;
      const float Dq = D_next;
      row_stats(ii + 1, L_next, D_next);
      int64_t kmax = p.n_k - 1;
      if (p.causal) kmax = min(kmax, q + offset);
      const int64_t lim = qvalid ? kmax - (k0 + kb) : -1;  // visible keys: c <= lim
      float pr[KPT];
      AQ_BPROF(tq_ = clock64();)
      mbar_wait(&bars[KV_B_S_FULL], ph);
      if (ii == 0 && it == 0) AQ_TL(1);
      tc_fence_after();
      tmem_load_f<KPT>(t_lane + KV_T_S + kb, pr);
      tc_fence_before();
      mbar_arrive(&bars[KV_B_S_EMPTY]);
      AQ_BPROF(long long tn_ = clock64(); pr_[0] += tn_ - tq_; tq_ = tn_;)
      // P = exp(S - L) exactly as the forward computes it
      p_from_s<KPT / 2>(pr, kb, sl2, L2);
      if (lim < KPT - 1) {
#pragma unroll
        for (int c = 0; c < KPT; ++c) pr[c] = (c <= lim) ? pr[c] : 0.f;
      }
      AQ_BPROF(tn_ = clock64(); pr_[1] += tn_ - tq_; tq_ = tn_;)
      if (g > 0) mbar_wait(&bars[KV_B_PF_FREE], (g - 1) & 1);
      AQ_BPROF(tn_ = clock64(); pr_[2] += tn_ - tq_; tq_ = tn_;)
      // P^F (or P) -> bf16 [query][key] T8x8
      if (!PLAIN && MX && p.fq_p) {  // MXFP4 P^F: 32-key UE8M0 blocks, dequantized exactly to bf16
#pragma unroll
        for (int b32 = 0; b32 < KPT / 32; ++b32) {
          uint32_t cd[4], sc;
          quantize_p32_mx(pr + 32 * b32, cd, sc);
          // byte-permute lookups of the E2M1 values' bf16 bytes (as for NVFP4
          // below), then an exact bf16x2 multiply by the power-of-two scale
          const __nv_bfloat16 sb = __float2bfloat16_rn(__int_as_float(static_cast<int>(sc << 23)));
          const __nv_bfloat162 s2 = __halves2bfloat162(sb, sb);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t o[4];
#pragma unroll
            for (int q4 = 0; q4 < 2; ++q4) {
              const uint32_t sel = (cd[g] >> (16 * q4)) & 0xFFFFu;
              const uint32_t lo = __byte_perm(0xC0800000u, 0xC0804000u, sel);
              const uint32_t hi = __byte_perm(0x3F3F3F00u, 0x40404040u, sel);
              uint32_t v01 = __byte_perm(lo, hi, 0x5140), v23 = __byte_perm(lo, hi, 0x7362);
              const __nv_bfloat162 p01 = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v01), s2);
              const __nv_bfloat162 p23 = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v23), s2);
              o[2 * q4] = *reinterpret_cast<const uint32_t*>(&p01);
              o[2 * q4 + 1] = *reinterpret_cast<const uint32_t*>(&p23);
            }
            *reinterpret_cast<uint4*>(p_h + t8x8_off(row, kb + 32 * b32 + 8 * g)) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
      }
if (PLAIN || !(MX && p.fq_p)) {
#pragma unroll
      for (int blk = 0; blk < KPT / 16; ++blk) {
        uint4 w[2];
        if (!PLAIN && p.fq_p) {
          const PBlock qb = quantize_p16_s(pr + blk * 16, p.p_r);
          if (p.pf_codes != nullptr && qvalid) {  // instrument (flash.py:386-387): the recomputed P^F
            const int64_t n16 = ceil_div(p.n_k, 16);
            const int64_t gb = (k0 + kb) / 16 + blk;
            if (gb < n16) {
              *reinterpret_cast<uint2*>(p.pf_codes + (head * p.n_q + q) * (n16 * 8) + gb * 8) =
                  make_uint2(qb.codes[0], qb.codes[1]);
              p.pf_scales[(head * p.n_q + q) * n16 + gb] = static_cast<uint8_t>(qb.scale);
            }
          }
          // P^F in bf16 straight from the codes: byte-permute lookups of the
          // E2M1 values' bf16 bytes, then one exact bf16x2 multiply by the
          // decoded scale (code x E4M3 has <= 5 significant bits)
          const __nv_bfloat16 sb = __float2bfloat16_rn(qb.sv);
          const __nv_bfloat162 s2 = __halves2bfloat162(sb, sb);
#pragma unroll
          for (int h8 = 0; h8 < 2; ++h8) {
            uint32_t o[4];
#pragma unroll
            for (int q4 = 0; q4 < 2; ++q4) {
              const uint32_t sel = (qb.codes[h8] >> (16 * q4)) & 0xFFFFu;
              const uint32_t lo = __byte_perm(0xC0800000u, 0xC0804000u, sel);  // low bytes of 0,.5,1,1.5 | 2,3,4,6
              const uint32_t hi = __byte_perm(0x3F3F3F00u, 0x40404040u, sel);  // high bytes
              uint32_t v01 = __byte_perm(lo, hi, 0x5140), v23 = __byte_perm(lo, hi, 0x7362);
              const __nv_bfloat162 p01 = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v01), s2);
              const __nv_bfloat162 p23 = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v23), s2);
              o[2 * q4] = *reinterpret_cast<const uint32_t*>(&p01);
              o[2 * q4 + 1] = *reinterpret_cast<const uint32_t*>(&p23);
            }
            w[h8] = make_uint4(o[0], o[1], o[2], o[3]);
          }
        } else {
#pragma unroll
          for (int h8 = 0; h8 < 2; ++h8) {
            const float* v = pr + blk * 16 + h8 * 8;
            w[h8] = make_uint4(pack16(v[0], v[1], f16), pack16(v[2], v[3], f16), pack16(v[4], v[5], f16),
                               pack16(v[6], v[7], f16));
          }
        }
        *reinterpret_cast<uint4*>(p_h + t8x8_off(row, kb + blk * 16)) = w[0];
        *reinterpret_cast<uint4*>(p_h + t8x8_off(row, kb + blk * 16 + 8)) = w[1];
      }
      }
      fence_async_smem();
      mbar_arrive(&bars[KV_B_PF_FULL]);
      AQ_BPROF(tn_ = clock64(); pr_[3] += tn_ - tq_; tq_ = tn_;)
      // dS = (dP - D) . P / sqrt(d) -> bf16
      mbar_wait(&bars[KV_B_DP_FULL], ph);
      tc_fence_after();
      float dp[KPT];
      tmem_load_f<KPT>(t_lane + KV_T_S + kb, dp);
      tc_fence_before();
      mbar_arrive(&bars[KV_B_DP_EMPTY]);
      AQ_BPROF(tn_ = clock64(); pr_[4] += tn_ - tq_; tq_ = tn_;)
      if (g > 0) mbar_wait(&bars[KV_B_DS_FREE], (g - 1) & 1);
      AQ_BPROF(tn_ = clock64(); pr_[5] += tn_ - tq_; tq_ = tn_;)
      store_ds<KPT>(ds_h, row, kb, dp, pr, Dq, p.inv_sqrt_d, f16);
      fence_async_smem();
      mbar_arrive(&bars[KV_B_DS_FULL]);
      AQ_BPROF(tn_ = clock64(); pr_[6] += tn_ - tq_; tq_ = tn_;)
    }
    AQ_BPROF(if (lane == 0) { for (int e = 0; e < 7; ++e) { atomicAdd(&g_bprof[e], pr_[e]); pr_[e] = 0; } atomicAdd(&g_bprof[14], static_cast<unsigned long long>(ni)); })
    AQ_TL(2);
    // epilogue: dV rows as soon as the last dV MMA is done (while the last dK
    // MMA runs), then dK rows (thread = key row, D/NKG columns); the next
    // item's S / dP run meanwhile
    const int64_t key = k0 + row;
    constexpr int DH = D / NKG;
#pragma unroll
    for (int w2 = 0; w2 < 2; ++w2) {
      const int which = 1 - w2;
      if (ni > 0) {
        mbar_wait(&bars[which ? KV_B_DV_DONE : KV_B_DONE], it & 1);
        tc_fence_after();
      }
      float gr[DH];
      if (ni > 0) {
        tmem_load_f<DH>(t_lane + (which ? KV_T_DV : KV_T_DK) + kg * DH, gr);
      } else {
#pragma unroll
        for (int e = 0; e < DH; ++e) gr[e] = 0.f;  // no visible query: zero gradient
      }
      if (key < p.n_k)
        store_run<DH>(which ? p.dv : p.dk, (head * p.n_k + key) * D + kg * DH, p.g_dt, gr, which ? p.dv_mul : p.dk_mul);
    }
    }  // items
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================================ K7b: dQ
// PLAIN: bf16 Q tile stationary; the K ring carries bf16 K tiles that serve S
// and dQ (no separate K^F ring).
template <int D, bool PLAIN = false>
struct QSmem {
  static constexpr int Q_CODES = 0;                                  // FP4 Q (bf16 Q tile for PLAIN)
  static constexpr int Q_SF = Q_CODES + TILE * D / 2;
  static constexpr int DO_H = PLAIN ? TILE * D * 2 : Q_SF + (D / 64) * 512;
  // per-operand rings over key tiles, each released by the MMA that last reads it:
  // K codes + scale factors (S), V^F (dP), K^F (dQ)
  static constexpr int KC_BYTES = PLAIN ? TILE * D * 2 : TILE * D / 2 + (D / 64) * 512;
  static constexpr int KC0 = DO_H + TILE * D * 2;
  static constexpr int VH0 = KC0 + 2 * KC_BYTES;
  static constexpr int KH0 = VH0 + 2 * TILE * D * 2;
  static constexpr int DS_H = KH0 + (PLAIN ? 0 : 2 * TILE * D * 2);  // dS bf16 [query][key]
  static constexpr int BARS = DS_H + TILE * TILE * 2;
  static constexpr int NUM_BARS = 24;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int TOTAL = TMEM_SLOT + 16;
  static constexpr int Q_BYTES = TILE * D / 2 + (D / 64) * 512 + TILE * D * 2;
  static_assert(TOTAL <= 227 * 1024, "shared memory");
};

// TMEM: S [0,128); dP [128,256); dQ [256,256+D); Q SF 384+, K SF 392 + 8 * stage
constexpr uint32_t Q_T_S = 0, Q_T_DP = 128, Q_T_DQ = 256, Q_T_QSF = 384, Q_T_KSF = 392;

enum QBar {
  Q_B_Q = 0, Q_B_KC_FULL = 1, Q_B_KC_EMPTY = 3, Q_B_VH_FULL = 5, Q_B_VH_EMPTY = 7, Q_B_KH_FULL = 9,
  Q_B_KH_EMPTY = 11, Q_B_S_FULL = 13, Q_B_S_EMPTY, Q_B_DP_FULL, Q_B_DP_EMPTY, Q_B_DS_FULL, Q_B_DS_EMPTY, Q_B_DONE,
  Q_B_DOH
};

// MMA issue order: S_0 dP_0 | S_1 dP_1 dQ_0 | S_2 dP_2 dQ_1 | ... so S_{j+1} and
// dP_{j+1} run while the compute warps turn S_j / dP_j into dS_j.
template <int D, bool MX, bool PLAIN>
__device__ __forceinline__ void bwd_q_tile(const BwdParams& p, uint8_t* smem, int qt, int64_t head) {
  using L = QSmem<D, PLAIN>;
  constexpr int NCW = Cfg<D>::NCW, NKG = Cfg<D>::NKG, KPT = Cfg<D>::KPT;
  constexpr int PRODUCER = Cfg<D>::PRODUCER, MMA = Cfg<D>::MMA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::TMEM_SLOT);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int q0 = qt * TILE;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const int64_t offset = p.n_k - p.n_q;
  int nt = k_tiles;  // key tiles with any visible key for this query tile
  if (p.causal) {
    const int64_t last = min(static_cast<int64_t>(q0 + TILE - 1), p.n_q - 1) + offset;
    nt = last < 0 ? 0 : min(nt, static_cast<int>(last / TILE) + 1);
  }

  const int64_t qidx0 = head * q_tiles + qt;
  if (threadIdx.x == 32 * PRODUCER) {
    mbar_init(&bars[Q_B_Q], 1);
    mbar_init(&bars[Q_B_DOH], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[Q_B_KC_FULL + s], 1);
      mbar_init(&bars[Q_B_KC_EMPTY + s], 1);
      mbar_init(&bars[Q_B_VH_FULL + s], 1);
      mbar_init(&bars[Q_B_VH_EMPTY + s], 1);
      mbar_init(&bars[Q_B_KH_FULL + s], 1);
      mbar_init(&bars[Q_B_KH_EMPTY + s], 1);
    }
    mbar_init(&bars[Q_B_S_FULL], 1);
    mbar_init(&bars[Q_B_S_EMPTY], 32 * NCW);
    mbar_init(&bars[Q_B_DP_FULL], 1);
    mbar_init(&bars[Q_B_DP_EMPTY], 32 * NCW);
    mbar_init(&bars[Q_B_DS_FULL], 32 * NCW);
    mbar_init(&bars[Q_B_DS_EMPTY], 1);
    mbar_init(&bars[Q_B_DONE], 1);
    fence_mbar_init();
    // stationary Q codes / dO and key tile 0 requested before the CTA-wide sync
    if (PLAIN) {
      mbar_expect_tx(&bars[Q_B_Q], TILE * D * 2);
      bulk_g2s(smem + L::Q_CODES, p.q_h + qidx0 * h_tile_bytes(D), TILE * D * 2, &bars[Q_B_Q]);
    } else {
      mbar_expect_tx(&bars[Q_B_Q], TILE * D / 2 + (D / 64) * 512);
      bulk_g2s(smem + L::Q_CODES, p.q_codes + qidx0 * fp4_tile_bytes(D), TILE * D / 2, &bars[Q_B_Q]);
      bulk_g2s(smem + L::Q_SF, p.q_sf + qidx0 * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[Q_B_Q]);
    }
    if (nt > 0) {
      const int64_t kidx = head * k_tiles;
      mbar_expect_tx(&bars[Q_B_KC_FULL], L::KC_BYTES);
      if (PLAIN) {
        bulk_g2s(smem + L::KC0, p.k_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[Q_B_KC_FULL]);
      } else {
        bulk_g2s(smem + L::KC0, p.k_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, &bars[Q_B_KC_FULL]);
        bulk_g2s(smem + L::KC0 + TILE * D / 2, p.k_sf + kidx * sf_tile_bytes_qk(D), (D / 64) * 512,
                 &bars[Q_B_KC_FULL]);
      }
    }
    mbar_expect_tx(&bars[Q_B_DOH], TILE * D * 2);
    bulk_g2s(smem + L::DO_H, p.do_h + qidx0 * h_tile_bytes(D), TILE * D * 2, &bars[Q_B_DOH]);
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == PRODUCER) {
    // ------------------------------------------------------------ producer
    // (Q codes, dO and key tile 0's codes were requested before the CTA-wide sync)
    for (int j = 0; j < nt; ++j) {
      const int st = j & 1;
      const uint32_t pe = ((j >> 1) - 1) & 1;
      const int64_t kidx = head * k_tiles + j;
      if (j >= 2) mbar_wait(&bars[Q_B_KC_EMPTY + st], pe);
      if (j > 0 && elect_one()) {
        uint8_t* dst = smem + L::KC0 + st * L::KC_BYTES;
        mbar_expect_tx(&bars[Q_B_KC_FULL + st], L::KC_BYTES);
        if (PLAIN) {
          bulk_g2s(dst, p.k_h + kidx * h_tile_bytes(D), TILE * D * 2, &bars[Q_B_KC_FULL + st]);
        } else {
          bulk_g2s(dst, p.k_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, &bars[Q_B_KC_FULL + st]);
          bulk_g2s(dst + TILE * D / 2, p.k_sf + kidx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[Q_B_KC_FULL + st]);
        }
      }
      __syncwarp();
      if (j >= 2) mbar_wait(&bars[Q_B_VH_EMPTY + st], pe);
      if (elect_one()) {
        mbar_expect_tx(&bars[Q_B_VH_FULL + st], TILE * D * 2);
        bulk_g2s(smem + L::VH0 + st * TILE * D * 2, p.v_h + kidx * h_tile_bytes(D), TILE * D * 2,
                 &bars[Q_B_VH_FULL + st]);
      }
      __syncwarp();
      if (PLAIN) continue;  // the K ring slot is the dQ operand too
      if (j >= 2) mbar_wait(&bars[Q_B_KH_EMPTY + st], pe);
      if (elect_one()) {
        mbar_expect_tx(&bars[Q_B_KH_FULL + st], TILE * D * 2);
        bulk_g2s(smem + L::KH0 + st * TILE * D * 2, p.k_h + kidx * h_tile_bytes(D), TILE * D * 2,
                 &bars[Q_B_KH_FULL + st]);
      }
      __syncwarp();
    }
  } else if (warp == MMA) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_nvf4(128, 128);
    const uint32_t f16f = PLAIN ? static_cast<uint32_t>(p.plain_fmt) : 1u;
    const uint32_t id_s16 = idesc_f16(128, 128, f16f, 0, 0);  // PLAIN: Q (K-major) x K (K-major)
    const uint32_t id_dp = idesc_f16(128, 128, f16f, 0, 0);  // dO (K-major) x V^F (K-major)
    const uint32_t id_dq = idesc_f16(128, D, f16f, 0, 1);    // dS (K-major) x K^F (MN-major)
    constexpr uint64_t t_fp4 = desc_template(2048, 128);
    constexpr uint64_t t_sf = desc_template(0, 128);
    constexpr uint64_t t_kmaj = desc_template(2048, 128);
    constexpr uint64_t t_mn = desc_template(128, 2048);
    const uint32_t s0 = smem_u32(smem);
    const uint32_t q_codes = s0 + L::Q_CODES, do_h = s0 + L::DO_H, ds_h = s0 + L::DS_H;
    mbar_wait(&bars[Q_B_Q], 0);
    tc_fence_after();
    if (!PLAIN && elect_one()) {
      for (int ks = 0; ks < D / 64; ++ks)
        tmem_cp_32x128_x4(tmem + Q_T_QSF + 4 * ks, desc_at(t_sf, s0 + L::Q_SF + ks * 512));
    }
    __syncwarp();
    auto issue_s_dp = [&](int j) {
      const int st = j & 1;
      const uint32_t pf = (j >> 1) & 1;
      const uint32_t kc = s0 + L::KC0 + st * L::KC_BYTES;
      mbar_wait(&bars[Q_B_KC_FULL + st], pf);
      if (j > 0) mbar_wait(&bars[Q_B_S_EMPTY], (j - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        if constexpr (PLAIN) {
          for (int ks = 0; ks < D / 16; ++ks)
            mma_f16_ss(tmem + Q_T_S, desc_at(t_kmaj, q_codes + ks * 4096), desc_at(t_kmaj, kc + ks * 4096), id_s16,
                       ks > 0);
        } else if constexpr (MX) {
          tmem_cp_32x128_x4(tmem + Q_T_KSF + 8 * st, desc_at(t_sf, kc + TILE * D / 2));
          for (int ks = 0; ks < D / 64; ++ks) {
            const uint32_t sid = 2u * ks;
            mma_mxf4_ss(tmem + Q_T_S, desc_at(t_fp4, q_codes + ks * 4096), desc_at(t_fp4, kc + ks * 4096),
                        idesc_mxf4(128, 128, sid), (tmem + Q_T_QSF) | (sid << 30),
                        (tmem + Q_T_KSF + 8 * st) | (sid << 30), ks > 0);
          }
        } else {
          for (int ks = 0; ks < D / 64; ++ks)
            tmem_cp_32x128_x4(tmem + Q_T_KSF + 8 * st + 4 * ks, desc_at(t_sf, kc + TILE * D / 2 + ks * 512));
          for (int ks = 0; ks < D / 64; ++ks)
            mma_nvf4_ss(tmem + Q_T_S, desc_at(t_fp4, q_codes + ks * 4096), desc_at(t_fp4, kc + ks * 4096), id_s,
                        tmem + Q_T_QSF + 4 * ks, tmem + Q_T_KSF + 8 * st + 4 * ks, ks > 0);
        }
        tc_commit(&bars[Q_B_S_FULL]);
        if (!PLAIN) tc_commit(&bars[Q_B_KC_EMPTY + st]);  // PLAIN: released by dQ
      }
      __syncwarp();
      mbar_wait(&bars[Q_B_VH_FULL + st], pf);
      if (j > 0) mbar_wait(&bars[Q_B_DP_EMPTY], (j - 1) & 1);
      else mbar_wait(&bars[Q_B_DOH], 0);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t vh = s0 + L::VH0 + st * TILE * D * 2;
        for (int ks = 0; ks < D / 16; ++ks)
          mma_f16_ss(tmem + Q_T_DP, desc_at(t_kmaj, do_h + ks * 4096), desc_at(t_kmaj, vh + ks * 4096), id_dp, ks > 0);
        tc_commit(&bars[Q_B_DP_FULL]);
        tc_commit(&bars[Q_B_VH_EMPTY + st]);
      }
      __syncwarp();
    };
    if (nt > 0) issue_s_dp(0);
    for (int j = 0; j < nt; ++j) {
      if (j + 1 < nt) issue_s_dp(j + 1);
      const int st = j & 1;
      mbar_wait(&bars[Q_B_DS_FULL], j & 1);
      if (!PLAIN) mbar_wait(&bars[Q_B_KH_FULL + st], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t kh = PLAIN ? s0 + L::KC0 + st * L::KC_BYTES : s0 + L::KH0 + st * TILE * D * 2;
        for (int ks = 0; ks < TILE / 16; ++ks)
          mma_f16_ss(tmem + Q_T_DQ, desc_at(t_kmaj, ds_h + ks * 4096), desc_at(t_mn, kh + ks * 256), id_dq,
                     (j > 0 || ks > 0));
        tc_commit(&bars[Q_B_DS_EMPTY]);
        tc_commit(&bars[PLAIN ? Q_B_KC_EMPTY + st : Q_B_KH_EMPTY + st]);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bars[Q_B_DONE]);
    __syncwarp();
  } else {
    // ------------------------------------------------------------ compute warps
    const int row = 32 * (warp & 3) + lane;
    const int kg = warp >> 2;
    const int kb = kg * KPT;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const float sl2 = p.scale_log2;
    const bool f16 = PLAIN && p.plain_fmt == 0;
    const int64_t q = q0 + row;
    const bool qvalid = q < p.n_q;
    const float L2 = qvalid ? p.lse[head * p.n_q + q] * 1.44269504088896340736f : 0.f;
    const float Dq = p.delta[head * (q_tiles * TILE) + q];
    int64_t kmax = p.n_k - 1;
    if (p.causal) kmax = min(kmax, q + offset);
    uint8_t* ds_h = smem + L::DS_H;
    AQ_BPROF(unsigned long long pr_[6] = {0, 0, 0, 0, 0, 0}; long long tq_ = clock64();)
    for (int j = 0; j < nt; ++j) {
      const uint32_t ph = j & 1;
      const int64_t lim = qvalid ? kmax - (static_cast<int64_t>(j) * TILE + kb) : -1;
      float pr[KPT];
      AQ_BPROF(tq_ = clock64();)
      mbar_wait(&bars[Q_B_S_FULL], ph);
      if (j == 0) AQ_TL(1);
      tc_fence_after();
      tmem_load_f<KPT>(t_lane + Q_T_S + kb, pr);
      tc_fence_before();
      mbar_arrive(&bars[Q_B_S_EMPTY]);
      AQ_BPROF(long long tn_ = clock64(); pr_[0] += tn_ - tq_; tq_ = tn_;)
      p_from_s<KPT / 2>(pr, kb, sl2, L2);
      if (lim < KPT - 1) {
#pragma unroll
        for (int c = 0; c < KPT; ++c) pr[c] = (c <= lim) ? pr[c] : 0.f;
      }
      AQ_BPROF(tn_ = clock64(); pr_[1] += tn_ - tq_; tq_ = tn_;)
      mbar_wait(&bars[Q_B_DP_FULL], ph);
      tc_fence_after();
      float dp[KPT];
      tmem_load_f<KPT>(t_lane + Q_T_DP + kb, dp);
      tc_fence_before();
      mbar_arrive(&bars[Q_B_DP_EMPTY]);
      AQ_BPROF(tn_ = clock64(); pr_[2] += tn_ - tq_; tq_ = tn_;)
      if (j > 0) mbar_wait(&bars[Q_B_DS_EMPTY], (j - 1) & 1);
      AQ_BPROF(tn_ = clock64(); pr_[3] += tn_ - tq_; tq_ = tn_;)
      store_ds<KPT>(ds_h, row, kb, dp, pr, Dq, p.inv_sqrt_d, f16);
      fence_async_smem();
      mbar_arrive(&bars[Q_B_DS_FULL]);
      AQ_BPROF(tn_ = clock64(); pr_[4] += tn_ - tq_; tq_ = tn_;)
    }
    AQ_BPROF(if (lane == 0) { for (int e = 0; e < 5; ++e) atomicAdd(&g_bprof[8 + e], pr_[e]); atomicAdd(&g_bprof[15], static_cast<unsigned long long>(nt)); })
    AQ_TL(2);
    // epilogue: dQ rows (thread = query row, D/NKG columns), written once in the output dtype
    if (nt > 0) {
      mbar_wait(&bars[Q_B_DONE], 0);
      tc_fence_after();
    }
    constexpr int DH = D / NKG;
    float g[DH];
    if (nt > 0) {
      tmem_load_f<DH>(t_lane + Q_T_DQ + kg * DH, g);
    } else {
#pragma unroll
      for (int e = 0; e < DH; ++e) g[e] = 0.f;
    }
    if (qvalid) store_run<DH>(p.dq, (head * p.n_q + q) * D + kg * DH, p.g_dt, g, p.dq_mul);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// K7: one launch for both roles. blockIdx.y = head, blockIdx.x = rank within
// the head in longest-first order: with causal masking key tile kt visits
// q_tiles - kt query tiles and query tile qt visits qt + 1 key tiles, so the
// ranks alternate KV tile 0, Q tile T-1, KV tile 1, Q tile T-2, ... Items of
// one head run together and share its operands in L2 (head-fastest order
// is 18% slower at C4); KV and Q items share no barriers.
// MX: the MXFP4 instance (S recomputed on kind::mxf4 block32, P^F in 32-key
// UE8M0 blocks dequantized exactly to bf16; everything else is shared).
// PLAIN: quantized=False (16-bit S recompute, P unquantized; flash.py:344-349).
// KV items pair up when the key and query tilings match and the tile count is even
__host__ __device__ __forceinline__ bool pair_kv(const BwdParams& p, int kv_tiles, int q_tiles) {
  return AQ_BWD_PAIR && kv_tiles == q_tiles && p.n_q == p.n_k && (kv_tiles & 1) == 0;
}

template <int D, bool MX, bool PLAIN = false>
__global__ void __launch_bounds__(Cfg<D>::NUM_THREADS, 1) attn_bwd_kernel(const BwdParams p, int kv_tiles, int q_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int64_t head = blockIdx.y;
  const int r = blockIdx.x;
  if (pair_kv(p, kv_tiles, q_tiles)) {
    // KV CTAs run key tiles (c, T-1-c): T+1 query tiles each under causal masking
    // (T non-causal); order KV pair 0, Q tile T-1, KV pair 1, Q tile T-2, ...
    const int h = kv_tiles / 2;
    AQ_TL(0);
    if (r < 2 * h && (r & 1) == 0) bwd_kv_tile<D, MX, PLAIN>(p, smem, r >> 1, head, kv_tiles - 1 - (r >> 1));
    else bwd_q_tile<D, MX, PLAIN>(p, smem, q_tiles - 1 - (r < 2 * h ? (r >> 1) : r - h), head);
#ifdef AQ_BWD_PROFILE
    if (threadIdx.x == 0 && tl_cta() < kTimelineCtas) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      g_btl[tl_cta()][3] = gtimer();
      g_btl[tl_cta()][4] = smid | (static_cast<unsigned long long>(r < 2 * h && (r & 1) == 0) << 16);
    }
#endif
    return;
  }
  const int m = min(kv_tiles, q_tiles);
  int kv = -1, qt = -1;
  if (r < 2 * m) {
    if (r & 1) qt = q_tiles - 1 - (r >> 1);
    else kv = r >> 1;
  } else if (kv_tiles > q_tiles) {
    kv = r - m;
  } else {
    qt = q_tiles - 1 - (r - m);
  }
  AQ_TL(0);
  if (kv >= 0) bwd_kv_tile<D, MX, PLAIN>(p, smem, kv, head);
  else bwd_q_tile<D, MX, PLAIN>(p, smem, qt, head);
#ifdef AQ_BWD_PROFILE
  if (threadIdx.x == 0 && tl_cta() < kTimelineCtas) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_btl[tl_cta()][3] = gtimer();
    g_btl[tl_cta()][4] = smid | (static_cast<unsigned long long>(kv >= 0) << 16);
  }
#endif
}

// K6: D = rowsum(dO . O_ref) (fp32) and dO -> bf16 T8x8 tiles (pad rows zero).
// A warp owns 8 consecutive rows (one T8x8 core row group): lane = (row % 8,
// column group c8 = lane / 8 + 4 i), so every 16-byte tile store of a warp
// fills four contiguous 128-byte runs; the row sum is closed with two
// shuffles over the four lanes that share a row.
template <int D>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const void* d_o, int do_dt, const void* o_ref, int o_dt,
                                                      int64_t heads, int64_t n_q, float* delta, uint8_t* do_h,
                                                      float delta_mul, int tile_f16) {
  constexpr int NCG = D / 8;  // 16-byte column groups per row
  const int64_t q_tiles = ceil_div(n_q, TILE);
  const int64_t row_groups = heads * q_tiles * (TILE / 8);
  const int lane = threadIdx.x % 32;
  const int r8 = lane % 8, cg = lane / 8;
  for (int64_t wg = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; wg < row_groups;
       wg += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const int64_t rp = wg * 8 + r8;              // padded row over all heads
    const int64_t h = rp / (q_tiles * TILE);
    const int64_t q = rp % (q_tiles * TILE);
    const bool valid = q < n_q;
    const int64_t base_row = (h * n_q + q) * D;
    const int64_t tile = h * q_tiles + q / TILE;
    uint8_t* tdst = do_h + tile * h_tile_bytes(D);
    float acc = 0.f;
    // bf16 dO and O_ref (the autograd path): all of this lane's 16-byte loads are
    // issued before any tile store, so they are in flight together (the stores
    // could alias the inputs as far as the compiler knows)
    const bool bf = do_dt == 1 && o_dt == 1;
    uint4 gw[NCG / 4], ow[NCG / 4];
    if (bf && valid) {
#pragma unroll
      for (int i = 0; i < NCG / 4; ++i) {
        const int64_t base = base_row + (cg + 4 * i) * 8;
        gw[i] = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(d_o) + base);
        ow[i] = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(o_ref) + base);
      }
    }
#pragma unroll
    for (int i = 0; i < NCG / 4; ++i) {
      const int c8 = cg + 4 * i;
      float g[8], o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) g[e] = o[e] = 0.f;
      if (valid && bf) {
        const uint32_t gg[4] = {gw[i].x, gw[i].y, gw[i].z, gw[i].w}, oo[4] = {ow[i].x, ow[i].y, ow[i].z, ow[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          g[2 * e] = __uint_as_float(gg[e] << 16);
          g[2 * e + 1] = __uint_as_float(gg[e] & 0xFFFF0000u);
          o[2 * e] = __uint_as_float(oo[e] << 16);
          o[2 * e + 1] = __uint_as_float(oo[e] & 0xFFFF0000u);
        }
      } else if (valid) {
        const int64_t base = base_row + c8 * 8;
        if (do_dt == 1) {
          const uint4 w = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(d_o) + base);
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            g[2 * e] = __uint_as_float(ww[e] << 16);
            g[2 * e + 1] = __uint_as_float(ww[e] & 0xFFFF0000u);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            g[e] = do_dt == 2 ? __half2float(reinterpret_cast<const __half*>(d_o)[base + e])
                              : reinterpret_cast<const float*>(d_o)[base + e];
        }
        if (o_dt == 1) {
          const uint4 w = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(o_ref) + base);
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            o[2 * e] = __uint_as_float(ww[e] << 16);
            o[2 * e + 1] = __uint_as_float(ww[e] & 0xFFFF0000u);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = o_dt == 2 ? __half2float(reinterpret_cast<const __half*>(o_ref)[base + e])
                             : reinterpret_cast<const float*>(o_ref)[base + e];
        }
      }
      // D from the dO the dP MMA sees: round dO to the tile format first, so
      // dP - D cancels exactly where the softmax is sharp (dP ~ D) instead of
      // exposing dO's 16-bit rounding (round-2 fix; D = rowsum(dO . O_ref))
#pragma unroll
      for (int e = 0; e < 8; ++e)
        g[e] = tile_f16 ? __half2float(__float2half_rn(g[e])) : __bfloat162float(__float2bfloat16_rn(g[e]));
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(g[e], o[e], acc);
      *reinterpret_cast<uint4*>(tdst + t8x8_off(static_cast<int>(q % TILE), c8 * 8)) =
          make_uint4(pack16(g[0], g[1], tile_f16), pack16(g[2], g[3], tile_f16), pack16(g[4], g[5], tile_f16),
                     pack16(g[6], g[7], tile_f16));
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    if (cg == 0) delta[rp] = acc * delta_mul;  // D / t_v (1 = reference), see BwdParams::inv_sqrt_d
  }
}

template <int D>
cudaError_t launch(const BwdParams& p, cudaStream_t st) {
  auto kern = p.plain ? attn_bwd_kernel<D, false, true> : p.mx ? attn_bwd_kernel<D, true> : attn_bwd_kernel<D, false>;
  constexpr int smem_q = KvSmem<D>::TOTAL > QSmem<D>::TOTAL ? KvSmem<D>::TOTAL : QSmem<D>::TOTAL;
  constexpr int smem_p = KvSmem<D, true>::TOTAL > QSmem<D, true>::TOTAL ? KvSmem<D, true>::TOTAL : QSmem<D, true>::TOTAL;
  const int smem = p.plain ? smem_p : smem_q;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int kv_tiles = static_cast<int>(ceil_div(p.n_k, TILE)), q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int gx = pair_kv(p, kv_tiles, q_tiles) ? kv_tiles / 2 + q_tiles : kv_tiles + q_tiles;
  kern<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(p.heads)), Cfg<D>::NUM_THREADS, smem, st>>>(
      p, kv_tiles, q_tiles);
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

// per-CTA timeline of the last profiled launch (-DAQ_BWD_PROFILE builds; else returns 5)
extern "C" int aq_debug_bwd_timeline(unsigned long long* out, int ctas) {
#ifdef AQ_BWD_PROFILE
  if (ctas > bwd::kTimelineCtas) ctas = bwd::kTimelineCtas;
  return cudaMemcpyFromSymbol(out, bwd::g_btl, sizeof(unsigned long long) * 5 * ctas) == cudaSuccess ? 0 : 5;
#else
  (void)out;
  (void)ctas;
  return 5;
#endif
}

extern "C" int aq_debug_bwd_profile(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, bwd::g_bprof, sizeof(bwd::g_bprof)) != cudaSuccess) return 5;
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(bwd::g_bprof, z, sizeof(z)) != cudaSuccess) return 5;
  }
  return 0;
}

cudaError_t launch_bwd_pre(const void* d_o, int do_dt, const void* o_ref, int o_dt, int64_t heads, int64_t n_q,
                           int d, float* delta, uint8_t* do_h, cudaStream_t st, float delta_mul, int tile_f16) {
  const int64_t rows = heads * ceil_div(n_q, TILE) * TILE;
  const int g = bwd::grid_for(rows * 4);  // 4 threads per row
  if (d == 128)
    bwd::bwd_pre_kernel<128><<<g, 256, 0, st>>>(d_o, do_dt, o_ref, o_dt, heads, n_q, delta, do_h, delta_mul, tile_f16);
  else if (d == 64)
    bwd::bwd_pre_kernel<64><<<g, 256, 0, st>>>(d_o, do_dt, o_ref, o_dt, heads, n_q, delta, do_h, delta_mul, tile_f16);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace aq
