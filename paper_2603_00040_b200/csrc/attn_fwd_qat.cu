// K11: NVFP4 training forward, split-pass (sm_100a).
//
// flash_forward_training (attnqat/flash.py:176-246): O = P^F V^F, O' = P V^F
// and L for each 128-row query tile, on K5's two-stream structure
// (attn_fwd_infer.cu): warpgroup A runs pass 1 of item k+1 -- S tiles,
// online (m, l), L -- while warpgroup B runs pass 2 of item k -- S again,
// P = exp(S - L), P^F, P^ = P l for O' -- and its epilogue, so the MUFU-bound
// exp-sum of one group overlaps the ALU / shared-memory-bound quantization of
// the other on every SMSP. In K4 (attn_fwd.cu) all softmax warps run the same
// phase at the same time and the two halves of the work never overlap.
//
// TMEM: training keeps O and O' (256 columns) in TMEM beside the scale
// factors, so the two streams cannot both have K5's 128-column S buffer.
// Group B (the heavier pass) keeps one, which its MMA warp refills as soon as
// B has loaded the previous tile. Group A gets a 64-column buffer and runs
// pass 1 on half tiles: its two column halves (warps 0-3: keys 0-63, warps
// 4-7: keys 64-127 of every tile, K4's CS = 2 split) take turns in it, N = 64
// MMAs (K rows 64.. at +1024 B in each T8x32 chunk, their scale factors at
// column +2). The halves drift half a tile apart, so each half's S MMA runs
// while the other half computes. The K scale factors of each stream live in
// one TMEM slot: a stream's next tile is issued only after its previous S
// tile was loaded, i.e. after the MMA that read the slot completed.
// Same arithmetic as K4: identical S MMAs, pass-1 code and (m, l) merge order
// (CS = 2), p_from_s / quantize_p16_s, P^ = fp16(P * l), O' MMA order and
// epilogue scaling -- so O, O' and L are bit-identical to K4, and O, L to K5.
//
// MXFP4: the same pipeline on kind::mxf4 (the MX template flag).
// Item order: K5's static snake, or (p.item_ctr, causal) K4's dynamic banded
// queue, claimed by producer A and published through a shared-memory ring.
// AQ_FWD_DEBUG bits (timing experiments only): 1 skips the O' MMAs, 2 the P^
// stores, 4 the V^F loads.
//
// Warps: 0-7 group A, 8-23 group B, 24 producer A (Q + K), 25 producer B
// (K + V^T + scale factors + fp16 V^F), 26 MMA A, 27 MMA B.
// TMEM: S_A [0,64), S_B [64,192), O [192,320), O' [320,448), scale factors 448+.
#include <cstdint>
#include <cuda_runtime.h>

// inline mbarrier waits: the warp roles run under different setmaxnreg limits
#ifndef AQ_WAIT_MODE
#define AQ_WAIT_MODE 3
#endif
#include "attn.h"
#include "layouts.cuh"
#include "pquant.cuh"
#include "ptx.cuh"
#include "rowstore.cuh"

#ifndef AQ_QAT_REGB
#define AQ_QAT_REGB 56
#endif
// how many S_B tiles MMA B may issue ahead of the PV MMAs
#ifndef AQ_QAT_SLEAD
#define AQ_QAT_SLEAD 1
#endif

namespace aq {
namespace fwdq {

// Tuning aid (-DAQ_FWDQ_PROFILE, enabled by AQ_FWD_DEBUG bit 32): cycle sums of
// the softmax groups' waits, from lane 0 of every warp (aq_debug_fwdq_profile).
__device__ unsigned long long g_qprof[16];
#ifdef AQ_FWDQ_PROFILE
#define AQ_QPROF(...) __VA_ARGS__
#else
#define AQ_QPROF(...)
#endif

template <int D>
struct Cfg {
  static constexpr int CS = 2, CSB = 4;                   // column splits of pass 1 / pass 2
  static constexpr int CW = TILE / CS, CWB = TILE / CSB;  // key columns per softmax thread
  static constexpr int NSW = 4 * CS, NSWB = 4 * CSB;      // warps per group
  static constexpr int WA = 0, WB = NSW, PROD_A = NSW + NSWB, PROD_B = PROD_A + 1, MMA_A = PROD_B + 1,
                       MMA_B = MMA_A + 1;
  static constexpr int NUM_THREADS = 32 * (MMA_B + 1);    // 896
  // registers (setmaxnreg): launch 72 x 896; producer / MMA warpgroup 40,
  // group B (32 keys per thread) REG_B, group A (64 live scores) the rest
  static constexpr int POOL = (65536 / NUM_THREADS) / 8 * 8 * NUM_THREADS;
  static constexpr int REG_P = 40, REG_B = AQ_QAT_REGB,
                       REG_A = ((POOL - 128 * REG_P - 32 * NSWB * REG_B) / (32 * NSW)) / 8 * 8;
  static_assert(128 * REG_P + 32 * NSWB * REG_B + 32 * NSW * REG_A <= POOL, "register pool");
  // Q slots, ring depths (A: K; B: K and V separately, so B's next K tile does
  // not wait for a 41 KB V stage to drain), P buffers
  static constexpr int NQ = 2, NSA = 2, NSBK = 2, NSB = 2, NP = 2;
  // TMEM: S_A (half tiles) 64, S_B 128, O 128, O' 128, scale factors 64
  static constexpr uint32_t T_SA = 0, T_SB = 64, T_O = 192, T_OP = 320;
  static constexpr uint32_t T_QSF = 448, T_KSFA = T_QSF + 8 * NQ, T_KSFB = T_KSFA + 8, T_PSF = T_KSFB + 8,
                            T_VSF = T_PSF + 8 * NP;
  static_assert(T_VSF + 8 * NSB <= 512, "TMEM columns");
  static constexpr int QC_BYTES = TILE * D / 2, QSF_BYTES = (D / 64) * 512, Q_BYTES = QC_BYTES + QSF_BYTES;
  static constexpr int Q0 = 0;                                         // NQ Q slots
  static constexpr int KA0 = Q0 + NQ * Q_BYTES, KA_BYTES = Q_BYTES;    // ring A: K codes + SF
  static constexpr int KBK0 = KA0 + NSA * KA_BYTES;                    // ring BK: K codes + SF
  static constexpr int KB0 = KBK0 + NSBK * KA_BYTES;                   // ring BV: V^T + SF + V^F
  static constexpr int KB_V = 0, KB_VSF = KB_V + TILE * D / 2, KB_VH = KB_VSF + 1024;
  static constexpr int KB_BYTES = KB_VH + TILE * D * 2;
  static constexpr int P0 = KB0 + NSB * KB_BYTES;                      // P^F codes + SF + P^ fp16
  static constexpr int PB_SF = TILE * TILE / 2, PB_H = PB_SF + 1024, P_BYTES = PB_H + TILE * TILE * 2;
  static constexpr int ML = P0 + NP * P_BYTES;                         // pass-1 (m, l) partials [CS][2][TILE]
  static constexpr int LB = ML + CS * 2 * TILE * 4;                    // (L, l) handoff [NQ][2][TILE]
  static constexpr int BARS = LB + NQ * 2 * TILE * 4;
  static constexpr int NUM_BARS = 48;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int NIQ = 4;                                        // dynamic-schedule item ring
  static constexpr int IQ = TMEM_SLOT + 16;
  static constexpr int USED = IQ + NIQ * 8;
  static constexpr int TOTAL = USED > 120 * 1024 ? USED : 120 * 1024;
  static_assert(USED <= 227 * 1024, "shared memory");
  // barriers
  static constexpr int B_Q_FULL = 0, B_Q_EMPTY = NQ, B_L_FULL = 2 * NQ, B_L_EMPTY = 3 * NQ, B_O_FULL = 4 * NQ,
                       B_O_EMPTY = B_O_FULL + 1, B_SA_FULL = B_O_EMPTY + 1, B_SA_EMPTY = B_SA_FULL + 2,
                       B_SB_FULL = B_SA_EMPTY + 2, B_SB_EMPTY = B_SB_FULL + 1, B_KA_FULL = B_SB_EMPTY + 1,
                       B_KA_EMPTY = B_KA_FULL + NSA, B_KB_FULL = B_KA_EMPTY + NSA, B_KB_EMPTY = B_KB_FULL + NSB,
                       B_KBK_FULL = B_KB_EMPTY + NSB, B_KBK_EMPTY = B_KBK_FULL + NSBK,
                       B_P_FULL = B_KBK_EMPTY + NSBK, B_P_EMPTY = B_P_FULL + NP, B_QSF = B_P_EMPTY + NP,
                       B_IQ_FULL = B_QSF + NQ, B_IQ_EMPTY = B_IQ_FULL + NIQ, B_END = B_IQ_EMPTY + NIQ;
  static_assert(B_END <= NUM_BARS, "barriers");
};

struct Item {
  int64_t head;
  int qt, nt;
};

// K5's item order (attn_fwd_infer.cu): causal rows longest first across heads,
// boustrophedon over the persistent CTAs.
__device__ __forceinline__ Item work_item(const FwdParams& p, int64_t w64, int q_tiles, int k_tiles) {
  Item it;
  int w = static_cast<int>(w64);
  const int heads = static_cast<int>(p.heads);
  if (p.causal && p.item_ctr) {
    // dynamic schedule (K4's banded order, attn_fwd.cu): bands of item_band
    // query tiles longest first, head-major inside a band, so the CTAs in
    // flight share each head's K / V^T / V^F tiles in L2
    const int band = min(p.item_band, q_tiles), full = q_tiles / band;
    int b, r, bs;
    if (w < full * band * heads) {
      b = w / (band * heads);
      r = w - b * (band * heads);
      bs = band;
    } else {
      b = full;
      r = w - full * band * heads;
      bs = q_tiles - full * band;
    }
    it.head = r / bs;
    it.qt = q_tiles - 1 - (b * band + r % bs);
    const int64_t last =
        static_cast<int64_t>(min(it.qt * TILE + TILE - 1, static_cast<int>(p.n_q) - 1)) + (p.n_k - p.n_q);
    it.nt = min(k_tiles, static_cast<int>(last / TILE) + 1);
    return it;
  }
  if (p.causal) {
    const int G = gridDim.x, r = w / G;
    if ((r & 1) && (r + 1) * G <= heads * q_tiles) w = r * G + (G - 1 - (w - r * G));
    it.qt = q_tiles - 1 - w / heads;
    it.head = w % heads;
    const int64_t last =
        static_cast<int64_t>(min(it.qt * TILE + TILE - 1, static_cast<int>(p.n_q) - 1)) + (p.n_k - p.n_q);
    it.nt = min(k_tiles, static_cast<int>(last / TILE) + 1);  // flash.py:127-128, 154
  } else {
    it.qt = w % q_tiles;
    it.head = w / q_tiles;
    it.nt = k_tiles;
  }
  return it;
}

// MX: the MXFP4 instance (codec.py:123-203): S and PV on kind::mxf4 block32
// with one scale-factor image per 128 K (IDs 0 / 2 per K = 64 step), P in
// 32-key UE8M0 blocks -- K4's MX instance on this pipeline.
template <int D, bool MX = false>
__global__ void __launch_bounds__(Cfg<D>::NUM_THREADS, 1) attn_fwd_qat_kernel(const FwdParams p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::TMEM_SLOT);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const int64_t n_items = p.heads * q_tiles;
  constexpr int GRP = 32 * C::NSW;    // threads of group A
  constexpr int GRPB = 32 * C::NSWB;  // threads of group B

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NQ; ++s) {
      mbar_init(&bars[C::B_Q_FULL + s], 1);
      mbar_init(&bars[C::B_Q_EMPTY + s], 1);
      mbar_init(&bars[C::B_L_FULL + s], GRP);
      mbar_init(&bars[C::B_L_EMPTY + s], GRPB);
      mbar_init(&bars[C::B_QSF + s], 1);
    }
    mbar_init(&bars[C::B_O_FULL], 1);
    mbar_init(&bars[C::B_O_EMPTY], GRPB);
    for (int h = 0; h < 2; ++h) {  // one pair per column half of group A
      mbar_init(&bars[C::B_SA_FULL + h], 1);
      mbar_init(&bars[C::B_SA_EMPTY + h], GRP / 2);
    }
    mbar_init(&bars[C::B_SB_FULL], 1);
    mbar_init(&bars[C::B_SB_EMPTY], GRPB);
    for (int s = 0; s < C::NSA; ++s) {
      mbar_init(&bars[C::B_KA_FULL + s], 1);
      mbar_init(&bars[C::B_KA_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NSBK; ++s) {
      mbar_init(&bars[C::B_KBK_FULL + s], 1);
      mbar_init(&bars[C::B_KBK_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NSB; ++s) {
      mbar_init(&bars[C::B_KB_FULL + s], 1);
      mbar_init(&bars[C::B_KB_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NP; ++s) {
      mbar_init(&bars[C::B_P_FULL + s], GRPB);
      mbar_init(&bars[C::B_P_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NIQ; ++s) {
      mbar_init(&bars[C::B_IQ_FULL + s], 1);
      mbar_init(&bars[C::B_IQ_EMPTY + s], C::MMA_B);  // every warp but producer A
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t s0 = smem_u32(smem);

  // Work items: static (blockIdx.x + k * gridDim.x) or, with p.item_ctr
  // (causal), claimed by producer A from a global counter and published
  // through an NIQ-slot ring that every other warp reads (as in K4 / K5).
  const bool dyn = p.item_ctr != nullptr;
  int64_t* iq = reinterpret_cast<int64_t*>(smem + C::IQ);
  auto next_item = [&](int kk) -> int64_t {
    if (!dyn) {
      const int64_t w = blockIdx.x + static_cast<int64_t>(kk) * gridDim.x;
      return w < n_items ? w : -1;
    }
    const int s = kk % C::NIQ;
    mbar_wait(&bars[C::B_IQ_FULL + s], (kk / C::NIQ) & 1);
    const int64_t w = iq[s];
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[C::B_IQ_EMPTY + s]);
    return w;
  };

  if (warp >= C::PROD_A) {
    setmaxnreg_dec<C::REG_P>();
    if (warp == C::PROD_A) {
      // ---------------------------------------------------------- producer A: Q + K for pass 1
      int it = 0, k = 0;
      int claim = 0;  // lane 0: the next claimed item (dynamic)
      if (dyn && lane == 0) claim = static_cast<int>(gridDim.x) + atomicAdd(p.item_ctr, 1);
      for (;; ++k) {
        int64_t w;
        if (!dyn) {
          w = blockIdx.x + static_cast<int64_t>(k) * gridDim.x;
          if (w >= n_items) break;
        } else {
          w = k == 0 ? static_cast<int64_t>(blockIdx.x) : static_cast<int64_t>(__shfl_sync(~0u, claim, 0));
          if (k > 0 && lane == 0 && w < n_items) claim = static_cast<int>(gridDim.x) + atomicAdd(p.item_ctr, 1);
          const int s = k % C::NIQ;
          if (k >= C::NIQ) mbar_wait(&bars[C::B_IQ_EMPTY + s], ((k / C::NIQ) - 1) & 1);
          if (lane == 0) {
            iq[s] = w < n_items ? w : -1;
            mbar_arrive(&bars[C::B_IQ_FULL + s]);
          }
          __syncwarp();
          if (w >= n_items) break;
        }
        const Item item = work_item(p, w, q_tiles, k_tiles);
        const int qs = k % C::NQ;
        if (k >= C::NQ) mbar_wait(&bars[C::B_Q_EMPTY + qs], ((k / C::NQ) - 1) & 1);
        const int64_t qidx = item.head * q_tiles + item.qt;
        if (elect_one()) {
          uint64_t* fb = &bars[C::B_Q_FULL + qs];
          mbar_expect_tx(fb, C::Q_BYTES);
          bulk_g2s(smem + C::Q0 + qs * C::Q_BYTES, p.q_codes + qidx * fp4_tile_bytes(D), C::QC_BYTES, fb);
          bulk_g2s(smem + C::Q0 + qs * C::Q_BYTES + C::QC_BYTES, p.q_sf + qidx * sf_tile_bytes_qk(D), C::QSF_BYTES, fb);
        }
        __syncwarp();
        for (int j = 0; j < item.nt; ++j, ++it) {
          const int st = it % C::NSA;
          if (it >= C::NSA) mbar_wait(&bars[C::B_KA_EMPTY + st], ((it / C::NSA) - 1) & 1);
          const int64_t kidx = item.head * k_tiles + j;
          if (elect_one()) {
            uint64_t* fb = &bars[C::B_KA_FULL + st];
            uint8_t* sb = smem + C::KA0 + st * C::KA_BYTES;
            mbar_expect_tx(fb, C::KA_BYTES);
            bulk_g2s(sb, p.k_codes + kidx * fp4_tile_bytes(D), C::QC_BYTES, fb);
            bulk_g2s(sb + C::QC_BYTES, p.k_sf + kidx * sf_tile_bytes_qk(D), C::QSF_BYTES, fb);
          }
          __syncwarp();
        }
      }
    } else if (warp == C::PROD_B) {
      // ---------------------------------------------------------- producer B: K + V for pass 2
      int it = 0, k = 0;
      for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
        const Item item = work_item(p, w, q_tiles, k_tiles);
        for (int j = 0; j < item.nt; ++j, ++it) {
          const int64_t kidx0 = item.head * k_tiles + j;
          // K of this tile (S_B) first: its ring drains as soon as the S MMA completes
          const int sk = it % C::NSBK;
          if (it >= C::NSBK) mbar_wait(&bars[C::B_KBK_EMPTY + sk], ((it / C::NSBK) - 1) & 1);
          if (elect_one()) {
            uint64_t* fb = &bars[C::B_KBK_FULL + sk];
            uint8_t* kb = smem + C::KBK0 + sk * C::KA_BYTES;
            mbar_expect_tx(fb, C::KA_BYTES);
            bulk_g2s(kb, p.k_codes + kidx0 * fp4_tile_bytes(D), C::QC_BYTES, fb);
            bulk_g2s(kb + C::QC_BYTES, p.k_sf + kidx0 * sf_tile_bytes_qk(D), C::QSF_BYTES, fb);
          }
          __syncwarp();
          const int st = it % C::NSB;
          if (it >= C::NSB) mbar_wait(&bars[C::B_KB_EMPTY + st], ((it / C::NSB) - 1) & 1);
          const int64_t kidx = item.head * k_tiles + j;
          if (elect_one()) {
            uint64_t* fb = &bars[C::B_KB_FULL + st];
            uint8_t* sb = smem + C::KB0 + st * C::KB_BYTES;
            mbar_expect_tx(fb, (p.debug & 4) ? C::KB_VH : C::KB_BYTES);
            bulk_g2s(sb + C::KB_V, p.v_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, fb);
            bulk_g2s(sb + C::KB_VSF, p.v_sf + kidx * kSfTileBytesV, 1024, fb);
            if (!(p.debug & 4)) bulk_g2s(sb + C::KB_VH, p.v_h + kidx * h_tile_bytes(D), TILE * D * 2, fb);
          }
          __syncwarp();
        }
      }
    } else {
      constexpr uint64_t t_k = desc_template(2048, 128);    // Q / K / P^F codes (K-major T8x32)
      constexpr uint64_t t_v = desc_template(D * 16, 128);  // V^T codes (K-major T8x32, D rows)
      constexpr uint64_t t_sf = desc_template(0, 128);      // SF512 images
      constexpr uint64_t t_ph = desc_template(2048, 128);   // P^ fp16 (K-major T8x8)
      constexpr uint64_t t_vh = desc_template(128, 2048);   // V^F fp16 (MN-major T8x8)
      constexpr uint32_t id_s = idesc_nvf4(128, 128);
      constexpr uint32_t id_h = idesc_nvf4(128, 64);
      constexpr uint32_t id_pv = idesc_nvf4(128, D);
      constexpr uint32_t id_op = idesc_f16(128, D, 0u, /*a_mn*/ 0, /*b_mn*/ 1);
      if (warp == C::MMA_A) {
        // -------------------------------------------------------- MMA A: pass-1 half tiles
        int it = 0, k = 0, u0 = 0, u1 = 0;
        for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
          const int nt = work_item(p, w, q_tiles, k_tiles).nt;
          const int qs = k % C::NQ;
          const uint32_t qb = s0 + C::Q0 + qs * C::Q_BYTES;
          mbar_wait(&bars[C::B_Q_FULL + qs], (k / C::NQ) & 1);
          tc_fence_after();
          if (elect_one()) {  // Q scale factors in TMEM, for MMA B too
            for (int ks = 0; ks < (MX ? 1 : D / 64); ++ks)
              tmem_cp_32x128_x4(tmem + C::T_QSF + 8 * qs + 4 * ks, desc_at(t_sf, qb + C::QC_BYTES + ks * 512));
            tc_commit(&bars[C::B_QSF + qs]);
          }
          __syncwarp();
          for (int j = 0; j < nt; ++j, ++it) {
            const int st = it % C::NSA;
            const uint32_t kb = s0 + C::KA0 + st * C::KA_BYTES;
            mbar_wait(&bars[C::B_KA_FULL + st], (it / C::NSA) & 1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              // the buffer's previous user: the other half (h = 0: half 1 of the previous tile)
              if (h == 0 && u1 > 0) mbar_wait(&bars[C::B_SA_EMPTY + 1], (u1 - 1) & 1);
              if (h == 1) mbar_wait(&bars[C::B_SA_EMPTY], (u0 - 1) & 1);
              tc_fence_after();
              if (elect_one()) {
                if (h == 0) {  // the slot's previous reader (half 1 of the last tile) has completed
#pragma unroll
                  for (int ks = 0; ks < (MX ? 1 : D / 64); ++ks)
                    tmem_cp_32x128_x4(tmem + C::T_KSFA + 4 * ks, desc_at(t_sf, kb + C::QC_BYTES + ks * 512));
                }
#pragma unroll
                for (int ks = 0; ks < D / 64; ++ks) {
                  if constexpr (MX) {
                    const uint32_t sid = 2u * ks;
                    mma_mxf4_ss(tmem + C::T_SA, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096 + h * 1024),
                                idesc_mxf4(128, 64, sid), (tmem + C::T_QSF + 8 * qs) | (sid << 30),
                                (tmem + C::T_KSFA + 2 * h) | (sid << 30), ks > 0);
                  } else {
                    mma_nvf4_ss(tmem + C::T_SA, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096 + h * 1024),
                                id_h, tmem + C::T_QSF + 8 * qs + 4 * ks, tmem + C::T_KSFA + 4 * ks + 2 * h, ks > 0);
                  }
                }
                tc_commit(&bars[C::B_SA_FULL + h]);
                if (h == 1) tc_commit(&bars[C::B_KA_EMPTY + st]);
              }
              __syncwarp();
              if (h == 0) ++u0; else ++u1;
            }
          }
        }
      } else if (warp == C::MMA_B) {
        // -------------------------------------------------------- MMA B: pass-2 S tiles + PV + O'
        int it = 0, k = 0, su = 0, pc = 0;
        for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
          const int nt = work_item(p, w, q_tiles, k_tiles).nt;
          const int qs = k % C::NQ;
          const uint32_t qb = s0 + C::Q0 + qs * C::Q_BYTES;
          // the Q slot and its TMEM scale factors were staged by MMA A
          mbar_wait(&bars[C::B_QSF + qs], (k / C::NQ) & 1);
          tc_fence_after();
          for (int ns = 0, np = 0; np < nt;) {
            if (ns < nt && ns <= np + AQ_QAT_SLEAD) {
              const int sk = (it + ns) % C::NSBK;
              mbar_wait(&bars[C::B_KBK_FULL + sk], ((it + ns) / C::NSBK) & 1);
              if (su > 0) mbar_wait(&bars[C::B_SB_EMPTY], (su - 1) & 1);  // also: the K SF slot's reader completed
              ++su;
              tc_fence_after();
              const uint32_t kb = s0 + C::KBK0 + sk * C::KA_BYTES;
              if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < (MX ? 1 : D / 64); ++ks)
                  tmem_cp_32x128_x4(tmem + C::T_KSFB + 4 * ks, desc_at(t_sf, kb + C::QC_BYTES + ks * 512));
#pragma unroll
                for (int ks = 0; ks < D / 64; ++ks) {
                  if constexpr (MX) {
                    const uint32_t sid = 2u * ks;
                    mma_mxf4_ss(tmem + C::T_SB, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096),
                                idesc_mxf4(128, 128, sid), (tmem + C::T_QSF + 8 * qs) | (sid << 30),
                                (tmem + C::T_KSFB) | (sid << 30), ks > 0);
                  } else {
                    mma_nvf4_ss(tmem + C::T_SB, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096), id_s,
                                tmem + C::T_QSF + 8 * qs + 4 * ks, tmem + C::T_KSFB + 4 * ks, ks > 0);
                  }
                }
                tc_commit(&bars[C::B_SB_FULL]);
                tc_commit(&bars[C::B_KBK_EMPTY + sk]);
                if (ns == nt - 1) tc_commit(&bars[C::B_Q_EMPTY + qs]);  // last read of this Q slot
              }
              __syncwarp();
              ++ns;
              continue;
            }
            const int pj = np++;
            const int pb = pc % C::NP;
            const int st = (it + pj) % C::NSB;
            if (pj == 0 && k > 0) mbar_wait(&bars[C::B_O_EMPTY], (k - 1) & 1);  // previous epilogue read O, O'
            mbar_wait(&bars[C::B_KB_FULL + st], ((it + pj) / C::NSB) & 1);     // V^T, V^F of this tile landed
            mbar_wait(&bars[C::B_P_FULL + pb], (pc / C::NP) & 1);
            ++pc;
            tc_fence_after();
            const uint32_t sb = s0 + C::KB0 + st * C::KB_BYTES;
            const uint32_t pbase = s0 + C::P0 + pb * C::P_BYTES;
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < (MX ? 1 : 2); ++ks) {
                tmem_cp_32x128_x4(tmem + C::T_PSF + 8 * pb + 4 * ks, desc_at(t_sf, pbase + C::PB_SF + ks * 512));
                tmem_cp_32x128_x4(tmem + C::T_VSF + 8 * st + 4 * ks, desc_at(t_sf, sb + C::KB_VSF + ks * 512));
              }
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                if constexpr (MX) {
                  const uint32_t sid = 2u * ks;
                  mma_mxf4_ss(tmem + C::T_O, desc_at(t_k, pbase + ks * 4096),
                              desc_at(t_v, sb + C::KB_V + ks * 2 * (D * 16)), idesc_mxf4(128, D, sid),
                              (tmem + C::T_PSF + 8 * pb) | (sid << 30), (tmem + C::T_VSF + 8 * st) | (sid << 30),
                              (pj > 0 || ks > 0));
                } else {
                  mma_nvf4_ss(tmem + C::T_O, desc_at(t_k, pbase + ks * 4096),
                              desc_at(t_v, sb + C::KB_V + ks * 2 * (D * 16)), id_pv, tmem + C::T_PSF + 8 * pb + 4 * ks,
                              tmem + C::T_VSF + 8 * st + 4 * ks, (pj > 0 || ks > 0));
                }
              }
#pragma unroll
              for (int ks = 0; ks < ((p.debug & 1) ? 0 : TILE / 16); ++ks)
                mma_f16_ss(tmem + C::T_OP, desc_at(t_ph, pbase + C::PB_H + ks * 4096),
                           desc_at(t_vh, sb + C::KB_VH + ks * 256), id_op, (pj > 0 || ks > 0));
              tc_commit(&bars[C::B_P_EMPTY + pb]);
              tc_commit(&bars[C::B_KB_EMPTY + st]);
            }
            __syncwarp();
          }
          it += nt;
          if (elect_one()) tc_commit(&bars[C::B_O_FULL]);
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax groups
    const bool grp_a = warp < C::WB;
    const int gw = grp_a ? warp - C::WA : warp - C::WB;  // warp within its group
    const int row = 32 * (gw & 3) + lane;                // TMEM lane == query row
    const uint32_t t_lane = tmem + (static_cast<uint32_t>((gw & 3) * 32) << 16);
    const float sl2 = p.scale_log2;
    float* ml = reinterpret_cast<float*>(smem + C::ML);
    float* lb = reinterpret_cast<float*>(smem + C::LB);
    int su = 0, k = 0;
    AQ_QPROF(long long qpa[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; const long long qstart_all = clock64();)
    // per-group wait sums into g_qprof: A [0] S_A, [1] L_EMPTY, [2] total, [3] tiles;
    // B [8] S_B, [9] L_FULL, [10] P_EMPTY, [11] O_FULL, [13] tiles, [14] total
    auto qdump = [&](bool ga) {
      AQ_QPROF(if ((p.debug & 32) && lane == 0) {
        const long long tot = clock64() - qstart_all;
        if (ga) {
          atomicAdd(&g_qprof[0], static_cast<unsigned long long>(qpa[0]));
          atomicAdd(&g_qprof[1], static_cast<unsigned long long>(qpa[1]));
          atomicAdd(&g_qprof[2], static_cast<unsigned long long>(tot));
          atomicAdd(&g_qprof[3], static_cast<unsigned long long>(qpa[3]));
        } else {
          for (int e = 4; e < 10; ++e) atomicAdd(&g_qprof[e + 4], static_cast<unsigned long long>(qpa[e]));
          atomicAdd(&g_qprof[14], static_cast<unsigned long long>(tot));
        }
      })
      (void)ga;
    };
    if (grp_a) {
      setmaxnreg_inc<C::REG_A>();
      constexpr int CW = C::CW;
      const int half = gw >> 2;
      const int cbase = half * CW;
      float x[CW];
      for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
        const Item item = work_item(p, w, q_tiles, k_tiles);
        const int nt = item.nt;
        const int64_t grow = static_cast<int64_t>(item.qt) * TILE + row;
        int64_t kmax = p.n_k - 1;
        if (p.causal) kmax = min(kmax, grow + (p.n_k - p.n_q));
        const int qs = k % C::NQ;
        // ---------------- pass 1: online (m, l) over 64 columns (K4 / K5's code and merge order)
        float m = -INFINITY, l = 0.f;
        for (int jj = 0; jj < nt; ++jj) {
          // this half's 64 keys of the tile, from the shared half-tile buffer
          AQ_QPROF(long long t0 = clock64();)
          mbar_wait(&bars[C::B_SA_FULL + half], su & 1);
          AQ_QPROF(qpa[0] += clock64() - t0; qpa[3] += 1;)
          ++su;
          tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < CW; c0 += 32) tmem_ld32f(t_lane + C::T_SA + c0, x + c0);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&bars[C::B_SA_EMPTY + half]);
          const int64_t lim = kmax - (static_cast<int64_t>(jj) * TILE + cbase);
          if (lim < CW - 1) {
#pragma unroll
            for (int c = 0; c < CW; ++c) x[c] = (c <= lim) ? x[c] : -INFINITY;
          }
          auto expsum = [&](float base) {
            float2 acc[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a] = make_float2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < CW / 2; ++i) {
              const float2 t = __ffma2_rn(make_float2(x[2 * i], x[2 * i + 1]), make_float2(sl2, sl2),
                                          make_float2(-base, -base));
              const float2 e = use_poly_p1(cbase / 2 + i) ? ex2_pair<true>(t) : ex2_pair<false>(t);
              acc[i & 3] = __fadd2_rn(acc[i & 3], e);
            }
            const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
            const float2 s4 = __fadd2_rn(s01, s23);
            return s4.x + s4.y;
          };
          float sum = expsum(m == -INFINITY ? 0.f : m);
          // a rebase needs a term above 2^8 (sum > 240 or inf): same m sequence as K4 / K5
          if (!(sum <= 240.0f) || m == -INFINITY) {
            float mx[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) mx[a] = x[a];
#pragma unroll
            for (int c = 8; c < CW; ++c) mx[c & 7] = fmaxf(mx[c & 7], x[c]);
            const float mloc = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                     fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
            if (mloc > m + 8.0f) {
              l = (m == -INFINITY) ? 0.f : l * ex2(m - mloc);
              m = mloc;
              sum = expsum(m);
            }
          }
          l += sum;
        }
        ml[(half * 2 + 0) * TILE + row] = m;
        ml[(half * 2 + 1) * TILE + row] = l;
        named_bar_sync(1, GRP);
        float mt = -INFINITY;
#pragma unroll
        for (int h = 0; h < C::CS; ++h) mt = fmaxf(mt, ml[(h * 2) * TILE + row]);
        float lt = 0.f;
#pragma unroll
        for (int h = 0; h < C::CS; ++h) lt += ml[(h * 2 + 1) * TILE + row] * ex2(ml[(h * 2) * TILE + row] - mt);
        named_bar_sync(1, GRP);
        // natural-log L as the reference stores it (flash.py:217); group B
        // rebuilds L2 = fl(L) * log2(e) like K4 and the backward
        const float L_nat = (mt + __log2f(lt)) * 0.69314718055994530942f;
        if (half == 0 && grow < p.n_q) p.lse[item.head * p.n_q + grow] = L_nat;
        AQ_QPROF(long long t1 = clock64();)
        if (k >= C::NQ) mbar_wait(&bars[C::B_L_EMPTY + qs], ((k / C::NQ) - 1) & 1);
        AQ_QPROF(qpa[1] += clock64() - t1;)
        if (half == 0) {
          lb[(qs * 2 + 0) * TILE + row] = L_nat;
          lb[(qs * 2 + 1) * TILE + row] = lt;
        }
        mbar_arrive(&bars[C::B_L_FULL + qs]);
      }
      qdump(true);
    } else {
      setmaxnreg_dec<C::REG_B>();
      constexpr int CW = C::CWB;  // 32 keys per thread
      const int half = gw >> 2;   // column quarter of this warp
      const int cbase = half * CW;
      float x[CW];
      int pc = 0;
      for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
        const Item item = work_item(p, w, q_tiles, k_tiles);
        const int nt = item.nt;
        const int64_t grow = static_cast<int64_t>(item.qt) * TILE + row;
        int64_t kmax = p.n_k - 1;
        if (p.causal) kmax = min(kmax, grow + (p.n_k - p.n_q));
        const int qs = k % C::NQ;
        float L2 = 0.f, l_scale = 0.f;
        // ---------------- pass 2: P, P^F (NVFP4 over 16-key blocks), P^ for O'
        for (int jj = 0; jj < nt; ++jj) {
          AQ_QPROF(long long t0 = clock64();)
          mbar_wait(&bars[C::B_SB_FULL], su & 1);
          AQ_QPROF(qpa[4] += clock64() - t0; qpa[9] += 1;)
          ++su;
          tc_fence_after();
          tmem_ld32f(t_lane + C::T_SB + cbase, x);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&bars[C::B_SB_EMPTY]);
          if (jj == 0) {  // after the first S load, so MMA B can refill the buffer meanwhile
            AQ_QPROF(long long t1 = clock64();)
            mbar_wait(&bars[C::B_L_FULL + qs], (k / C::NQ) & 1);
            AQ_QPROF(qpa[5] += clock64() - t1;)
            L2 = lb[(qs * 2 + 0) * TILE + row] * 1.44269504088896340736f;
            l_scale = lb[(qs * 2 + 1) * TILE + row];  // P^ = exp(S - m) = P * l
            mbar_arrive(&bars[C::B_L_EMPTY + qs]);
          }
          const int64_t lim = kmax - (static_cast<int64_t>(jj) * TILE + cbase);
          p_from_s<CW / 2>(x, cbase, sl2, L2);
          if (lim < CW - 1) {
#pragma unroll
            for (int c = 0; c < CW; ++c) x[c] = (c <= lim) ? x[c] : 0.f;
          }
          const int pb = pc % C::NP;
          AQ_QPROF(long long t2 = clock64();)
          if (pc >= C::NP) mbar_wait(&bars[C::B_P_EMPTY + pb], ((pc / C::NP) - 1) & 1);
          AQ_QPROF(qpa[6] += clock64() - t2;)
          ++pc;
          uint8_t* pbase = smem + C::P0 + pb * C::P_BYTES;
          uint8_t* psf = pbase + C::PB_SF;
          if constexpr (MX) {  // one 32-key UE8M0 block
            uint32_t cd[4], sc;
            quantize_p32_mx(x, cd, sc);
            *reinterpret_cast<uint4*>(pbase + t8x32_off(row, cbase, TILE)) = make_uint4(cd[0], cd[1], cd[2], cd[3]);
            psf[sf512_off(row, cbase / 32)] = static_cast<uint8_t>(sc);
          } else {
            const PBlock qa = quantize_p16_s(x, p.p_r);
            const PBlock qb = quantize_p16_s(x + 16, p.p_r);
            *reinterpret_cast<uint4*>(pbase + t8x32_off(row, cbase, TILE)) =
                make_uint4(qa.codes[0], qa.codes[1], qb.codes[0], qb.codes[1]);
            *reinterpret_cast<uint16_t*>(psf + sf512_off(row, cbase / 16)) =
                static_cast<uint16_t>(qa.scale | (qb.scale << 8));
          }
          uint8_t* ph = pbase + C::PB_H;
#pragma unroll
          for (int c8 = 0; c8 < ((p.debug & 2) ? 0 : CW / 8); ++c8) {
            uint32_t h[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 ph2 = __fmul2_rn(make_float2(x[c8 * 8 + 2 * e], x[c8 * 8 + 2 * e + 1]),
                                            make_float2(l_scale, l_scale));
              const __half2 v = __floats2half2_rn(ph2.x, ph2.y);
              h[e] = *reinterpret_cast<const uint32_t*>(&v);
            }
            *reinterpret_cast<uint4*>(ph + t8x8_off(row, cbase + c8 * 8)) = make_uint4(h[0], h[1], h[2], h[3]);
          }
          if (!MX && p.pf_codes != nullptr && grow < p.n_q) {  // instrument: this row's P^F of the tile
            const int64_t n16 = ceil_div(p.n_k, 16);
            const int64_t c0 = static_cast<int64_t>(jj) * TILE + cbase;
            uint8_t* dc = p.pf_codes + (item.head * p.n_q + grow) * (n16 * 8);
            uint8_t* dsc = p.pf_scales + (item.head * p.n_q + grow) * n16;
#pragma unroll
            for (int b = 0; b < CW / 16; ++b) {
              const int64_t blk = c0 / 16 + b;
              if (blk < n16) {
                *reinterpret_cast<uint2*>(dc + blk * 8) =
                    *reinterpret_cast<const uint2*>(pbase + t8x32_off(row, cbase + 16 * b, TILE));
                dsc[blk] = psf[sf512_off(row, cbase / 16 + b)];
              }
            }
          }
          fence_async_smem();
          mbar_arrive(&bars[C::B_P_FULL + pb]);
        }
        // ---------------- epilogue: D / 4 columns of O, then of O' * 1/l
        AQ_QPROF(long long t3 = clock64();)
        mbar_wait(&bars[C::B_O_FULL], k & 1);
        AQ_QPROF(qpa[7] += clock64() - t3;)
        tc_fence_after();
        constexpr int DW = D / C::CSB;
        const float inv_l = 1.f / l_scale;
#pragma unroll
        for (int out = 0; out < 2; ++out) {
          float o[DW];
          if constexpr (DW >= 32) {
#pragma unroll
            for (int c = 0; c < DW; c += 32) tmem_ld32f(t_lane + (out ? C::T_OP : C::T_O) + half * DW + c, o + c);
          } else {
            uint32_t r16[16];
            tmem_ld16(t_lane + (out ? C::T_OP : C::T_O) + half * DW, r16);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __uint_as_float(r16[c]);
          }
          tmem_ld_wait();
          if (out == 1) {  // both accumulators read: the next item's PV MMAs may start
            tc_fence_before();
            mbar_arrive(&bars[C::B_O_EMPTY]);
          }
          void* dst = out ? p.o_hp : p.o;
          if (dst != nullptr && grow < p.n_q) {
            const int dt = out ? p.o_hp_dt : p.o_dt;
            const float mul = out ? inv_l * p.ohp_mul : p.o_mul;  // per-tensor scales (1 = reference)
            store_row<DW>(reinterpret_cast<uint8_t*>(dst) + ((item.head * p.n_q + grow) * D + half * DW) * (dt == 0 ? 4 : 2),
                          o, mul, dt);
          }
        }
      }
      qdump(false);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool MX = false>
cudaError_t launch(const FwdParams& p, cudaStream_t st) {
  using C = Cfg<D>;
  auto kern = attn_fwd_qat_kernel<D, MX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::TOTAL);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = p.heads * ceil_div(p.n_q, TILE);
  const int grid = static_cast<int>(items < sms ? items : sms);
  if (p.item_ctr) {
    e = cudaMemsetAsync(p.item_ctr, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, C::NUM_THREADS, C::TOTAL, st>>>(p);
  return cudaGetLastError();
}

}  // namespace fwdq

// [0] group A S_A wait, [1] A L_EMPTY wait, [2] A total, [3] A tiles (warp-tiles),
// [8] B S_B wait, [9] B L_FULL wait, [10] B P_EMPTY wait, [11] B O_FULL wait, [13] B tiles, [14] B total
extern "C" int aq_debug_fwdq_profile(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, fwdq::g_qprof, sizeof(fwdq::g_qprof)) != cudaSuccess) return 5;
  if (reset) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(fwdq::g_qprof, z, sizeof(z)) != cudaSuccess) return 5;
  }
  return 0;
}

cudaError_t launch_attn_fwd_qat(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return fwdq::launch<64>(p, st);
  if (p.d == 128) return fwdq::launch<128>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_attn_fwd_qat_mx(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return fwdq::launch<64, true>(p, st);
  if (p.d == 128) return fwdq::launch<128, true>(p, st);
  return cudaErrorInvalidValue;
}

}  // namespace aq
