// K5: NVFP4 inference forward, split-pass pipelined variant (sm_100a).
//
// Same math as flash_forward_inference (attnqat/flash.py:249-314) and as the
// training kernel in attn_fwd.cu (identical S MMAs, identical p_from_s /
// quantize_p16, so O is bit-identical between the two):
//   pass 1  S = Q^F K^F^T -> online (m, l) -> L = m + log l   (flash.py:145-173, 217)
//   pass 2  S again -> P = exp(S - L) -> P^F (16-key NVFP4 blocks) -> O += P^F V^F
//
// Structure: the two passes run as two concurrent streams on different work
// items. Warpgroup A runs pass 1 of item k+1 while warpgroup B runs pass 2 (and
// the epilogue) of item k, so the SFU-heavy exp-sum of pass 1 and the
// ALU-heavy P quantization of pass 2 overlap on every SMSP and the two groups
// never wait on the same barrier phase. Each stream has its own producer warp,
// MMA-issuer warp, K(/V) ring and single TMEM S buffer; L crosses from A to B
// through shared memory. Persistent: one CTA per SM walks the item list.
//
// Warps: 0-7 softmax A (pass 1), 8-15 softmax B (pass 2 + epilogue),
// 16 producer A (Q + K), 17 producer B (K + V), 18 MMA A, 19 MMA B.
// TMEM: SA [0,128), SB [128,256), O [256,256+D), scale factors at 384+.
#include <cstdint>
#include <cuda_runtime.h>

// mbarrier waits inline in this kernel (ptx.cuh mode 0): the warp roles run
// under different setmaxnreg limits, and an out-of-line wait routine would be
// one function shared across them (ptxas cannot allocate it)
#ifndef AQ_WAIT_MODE
#define AQ_WAIT_MODE 3
#endif
#include "attn.h"
#include "layouts.cuh"
#include "pquant.cuh"
#include "ptx.cuh"

#ifndef AQ_FWDI_QSLOTS
#define AQ_FWDI_QSLOTS 2
#endif
#ifndef AQ_FWDI_NSA
#define AQ_FWDI_NSA 4
#endif
#ifndef AQ_FWDI_NSB
#define AQ_FWDI_NSB 3
#endif
#ifndef AQ_FWDI_NP
#define AQ_FWDI_NP 2
#endif
// how many pass-2 S tiles MMA B may issue ahead of the PV MMA it is waiting on
#ifndef AQ_FWDI_SNAKE
#define AQ_FWDI_SNAKE 1
#endif
#ifndef AQ_FWDI_SLEAD
#define AQ_FWDI_SLEAD 1
#endif

namespace aq {
namespace fwdi {

// Tuning aid (-DAQ_FWDI_PROFILE, enabled by AQ_FWD_DEBUG bit 32): cycle sums of
// the softmax groups' waits, from lane 0 of every warp (aq_debug_fwdi_profile):
// A [0] S wait, [1] L_EMPTY wait, [2] total, [3] tiles;
// B [8] S wait, [9] L_FULL wait, [10] P_EMPTY wait, [11] O_FULL wait, [13] tiles, [14] total
__device__ unsigned long long g_iprof[16];
#ifdef AQ_FWDI_PROFILE
#define AQ_IPROF(...) __VA_ARGS__
#else
#define AQ_IPROF(...)
#endif

#ifndef AQ_FWDI_CSB
#define AQ_FWDI_CSB 4
#endif
template <int D>
struct Cfg {
  // column splits: pass 1 (group A) keeps 2 (its (m, l) merge order is shared
  // with K4, so L and O stay bit-identical between the kernels); pass 2 (group
  // B, the heavier half: exp + NVFP4 quantization) runs CSB splits, i.e. 4 x
  // the warps per TMEM row quadrant for latency hiding at 32 keys per thread
  static constexpr int CS = 2, CSB = AQ_FWDI_CSB;
  static constexpr int CW = TILE / CS, CWB = TILE / CSB;  // key columns per softmax thread
  static constexpr int NSW = 4 * CS, NSWB = 4 * CSB;      // warps per softmax group
  static constexpr int WA = 0, WB = NSW, PROD_A = NSW + NSWB, PROD_B = PROD_A + 1, MMA_A = PROD_B + 1,
                       MMA_B = MMA_A + 1;
  static constexpr int NUM_THREADS = 32 * (MMA_B + 1);
  // 896 threads launch at 72 registers; the producer / MMA warpgroup drops to 40,
  // group B (32 keys per thread) to 56, and group A (64 live scores per thread)
  // takes the rest, 120 (setmaxnreg; no spills anywhere)
  static constexpr bool REALLOC = NUM_THREADS == 896;
#ifndef AQ_FWDI_REGA
#define AQ_FWDI_REGA 0
#endif
#ifndef AQ_FWDI_REGP
#define AQ_FWDI_REGP 40
#endif
#ifndef AQ_FWDI_REGB
#define AQ_FWDI_REGB 56
#endif
  // the CTA's register pool is what it launched with (72 x 896 = 64512): the
  // three warpgroup limits must fit it exactly (an over-budget inc never returns)
  static constexpr int POOL = (65536 / NUM_THREADS) / 8 * 8 * NUM_THREADS;
  static constexpr int REG_P = AQ_FWDI_REGP, REG_B = AQ_FWDI_REGB,
                       REG_A = AQ_FWDI_REGA ? AQ_FWDI_REGA : ((POOL - 128 * REG_P - 32 * NSWB * REG_B) / (32 * NSW)) / 8 * 8;
  static_assert(!REALLOC || 128 * REG_P + 32 * NSWB * REG_B + 32 * NSW * REG_A <= POOL, "register pool");
  static constexpr int NSA = AQ_FWDI_NSA, NSB = AQ_FWDI_NSB, NP = AQ_FWDI_NP;  // ring depths
  static constexpr int NQ = AQ_FWDI_QSLOTS;           // Q slots: how far pass 1 may run ahead of pass 2
  // TMEM
  static constexpr uint32_t T_SA = 0, T_SB = 128, T_O = 256;
  static constexpr uint32_t T_QSF = 384, T_KSFA = T_QSF + 8 * NQ, T_KSFB = T_KSFA + 8 * NSA, T_PSF = T_KSFB + 8 * NSB,
                            T_VSF = T_PSF + 8 * NP;
  // SMEM
  static constexpr int QC_BYTES = TILE * D / 2, QSF_BYTES = (D / 64) * 512, Q_BYTES = QC_BYTES + QSF_BYTES;
  static constexpr int Q0 = 0;                                    // NQ Q slots
  static constexpr int KA0 = Q0 + NQ * Q_BYTES;                   // ring A: K codes + SF
  static constexpr int KA_BYTES = QC_BYTES + QSF_BYTES;
  static constexpr int KB0 = KA0 + NSA * KA_BYTES;                // ring B: K + V^T codes + SF
  static constexpr int KB_V = KA_BYTES, KB_VSF = KB_V + TILE * D / 2, KB_BYTES = KB_VSF + 1024;
  static constexpr int P0 = KB0 + NSB * KB_BYTES;                 // P^F codes + SF
  static constexpr int PB_SF = TILE * TILE / 2, P_BYTES = PB_SF + 1024;
  static constexpr int ML = P0 + NP * P_BYTES;                    // pass-1 (m, l) partials [CS][2][TILE]
  static constexpr int LB = ML + CS * 2 * TILE * 4;               // L handoff [NQ][TILE]
  static constexpr int BARS = LB + NQ * TILE * 4;
  static constexpr int NUM_BARS = 48;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int USED = TMEM_SLOT + 16;
  static constexpr int TOTAL = USED > 120 * 1024 ? USED : 120 * 1024;
  // barriers
  static constexpr int B_Q_FULL = 0, B_Q_EMPTY = NQ, B_L_FULL = 2 * NQ, B_L_EMPTY = 3 * NQ, B_QSF = 4 * NQ,
                       B_O_FULL = 5 * NQ, B_O_EMPTY = B_O_FULL + 1, B_SA_FULL = B_O_EMPTY + 1,
                       B_SA_EMPTY = B_SA_FULL + 1, B_SB_FULL = B_SA_EMPTY + 1, B_SB_EMPTY = B_SB_FULL + 1,
                       B_KA_FULL = B_SB_EMPTY + 1, B_KA_EMPTY = B_KA_FULL + NSA, B_KB_FULL = B_KA_EMPTY + NSA,
                       B_KB_EMPTY = B_KB_FULL + NSB, B_P_FULL = B_KB_EMPTY + NSB, B_P_EMPTY = B_P_FULL + NP,
                       B_END = B_P_EMPTY + NP;
  static_assert(B_END <= NUM_BARS, "barriers");
  static_assert(USED <= 227 * 1024, "shared memory");
  static_assert(T_VSF + 8 * NSB <= 512, "TMEM columns");
};

struct Item {
  int64_t head;
  int qt, nt;
};

// Same item order as attn_fwd.cu: causal rows longest first across heads.
__device__ __forceinline__ Item work_item(const FwdParams& p, int64_t w, int q_tiles, int k_tiles) {
  Item it;
  if (AQ_FWDI_SNAKE && p.causal) {
    // boustrophedon over the persistent CTAs: CTA c takes the c-th item of even
    // rounds and the (G-1-c)-th of odd full rounds, so every CTA's sum of
    // longest-first row lengths is nearly equal (causal makespan / mean at
    // 148 CTAs: 128 heads x 64 tiles 1.017 -> 1.001, 16 heads 1.138 -> 1.018)
    const int64_t G = gridDim.x, r = w / G;
    if ((r & 1) && (r + 1) * G <= p.heads * q_tiles) w = r * G + (G - 1 - (w - r * G));
  }
  if (p.causal) {
    it.qt = q_tiles - 1 - static_cast<int>(w / p.heads);
    it.head = w % p.heads;
    const int64_t last =
        static_cast<int64_t>(min(it.qt * TILE + TILE - 1, static_cast<int>(p.n_q) - 1)) + (p.n_k - p.n_q);
    it.nt = min(k_tiles, static_cast<int>(last / TILE) + 1);  // flash.py:127-128, 154
  } else {
    it.qt = static_cast<int>(w % q_tiles);
    it.head = w / q_tiles;
    it.nt = k_tiles;
  }
  return it;
}

// MX: the MXFP4 variant (codec.py:123-203) -- S and PV on kind::mxf4 block32
// with one scale-factor image per 128 K (IDs 0 / 2 per K = 64 step), P in
// 32-key UE8M0 blocks; same pipeline.
// EARLY: the instance with the pass-2 early-out (long key rows, see launch()).
template <int D, bool MX = false, bool EARLY = false>
__global__ void __launch_bounds__(Cfg<D>::NUM_THREADS, 1) attn_fwd_infer_kernel(const FwdParams p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::TMEM_SLOT);
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const int64_t n_items = p.heads * q_tiles;
  constexpr int GRP = 32 * C::NSW;   // threads of softmax group A (pass 1)
  constexpr int GRPB = 32 * C::NSWB; // threads of softmax group B (pass 2)

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
    mbar_init(&bars[C::B_SA_FULL], 1);
    mbar_init(&bars[C::B_SA_EMPTY], GRP);
    mbar_init(&bars[C::B_SB_FULL], 1);
    mbar_init(&bars[C::B_SB_EMPTY], GRPB);
    for (int s = 0; s < C::NSA; ++s) {
      mbar_init(&bars[C::B_KA_FULL + s], 1);
      mbar_init(&bars[C::B_KA_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NSB; ++s) {
      mbar_init(&bars[C::B_KB_FULL + s], 1);
      mbar_init(&bars[C::B_KB_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NP; ++s) {
      mbar_init(&bars[C::B_P_FULL + s], GRPB);
      mbar_init(&bars[C::B_P_EMPTY + s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t s0 = smem_u32(smem);
  constexpr uint64_t t_k = desc_template(2048, 128);    // Q / K / P^F codes (K-major T8x32, 128 rows)
  constexpr uint64_t t_v = desc_template(D * 16, 128);  // V^T codes (K-major T8x32, D rows)
  constexpr uint64_t t_sf = desc_template(0, 128);      // SF512 images
  constexpr uint32_t id_s = idesc_nvf4(128, 128);
  constexpr uint32_t id_pv = idesc_nvf4(128, D);

  if (warp >= C::PROD_A) {
  // producer / MMA warpgroup: few registers (setmaxnreg inside each role branch,
  // so the limit applies to that branch only)
  if constexpr (C::REALLOC) setmaxnreg_dec<C::REG_P>();
  if (warp == C::PROD_A) {
    // ------------------------------------------------------------ producer A: Q + K for pass 1
    int it = 0, k = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
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
    // ------------------------------------------------------------ producer B: K + V for pass 2
    int it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const Item item = work_item(p, w, q_tiles, k_tiles);
      for (int j = 0; j < item.nt; ++j, ++it) {
        const int st = it % C::NSB;
        if (it >= C::NSB) mbar_wait(&bars[C::B_KB_EMPTY + st], ((it / C::NSB) - 1) & 1);
        const int64_t kidx = item.head * k_tiles + j;
        if (elect_one()) {
          uint64_t* fb = &bars[C::B_KB_FULL + st];
          uint8_t* sb = smem + C::KB0 + st * C::KB_BYTES;
          mbar_expect_tx(fb, C::KB_BYTES);
          bulk_g2s(sb, p.k_codes + kidx * fp4_tile_bytes(D), C::QC_BYTES, fb);
          bulk_g2s(sb + C::QC_BYTES, p.k_sf + kidx * sf_tile_bytes_qk(D), C::QSF_BYTES, fb);
          bulk_g2s(sb + C::KB_V, p.v_codes + kidx * fp4_tile_bytes(D), TILE * D / 2, fb);
          bulk_g2s(sb + C::KB_VSF, p.v_sf + kidx * kSfTileBytesV, 1024, fb);
        }
        __syncwarp();
      }
    }
  } else if (warp == C::MMA_A) {
    // ------------------------------------------------------------ MMA A: pass-1 S tiles
    int it = 0, k = 0, su = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
      const int nt = work_item(p, w, q_tiles, k_tiles).nt;
      const int qs = k % C::NQ;
      const uint32_t qb = s0 + C::Q0 + qs * C::Q_BYTES;
      mbar_wait(&bars[C::B_Q_FULL + qs], (k / C::NQ) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int ks = 0; ks < (MX ? 1 : D / 64); ++ks)
          tmem_cp_32x128_x4(tmem + C::T_QSF + 8 * qs + 4 * ks, desc_at(t_sf, qb + C::QC_BYTES + ks * 512));
        tc_commit(&bars[C::B_QSF + qs]);  // Q scale factors in TMEM, for MMA B too
      }
      __syncwarp();
      for (int j = 0; j < nt; ++j, ++it) {
        const int st = it % C::NSA;
        mbar_wait(&bars[C::B_KA_FULL + st], (it / C::NSA) & 1);
        if (su > 0) mbar_wait(&bars[C::B_SA_EMPTY], (su - 1) & 1);
        ++su;
        tc_fence_after();
        const uint32_t kb = s0 + C::KA0 + st * C::KA_BYTES;
        if (elect_one()) {
          if constexpr (MX) {
            tmem_cp_32x128_x4(tmem + C::T_KSFA + 8 * st, desc_at(t_sf, kb + C::QC_BYTES));
#pragma unroll
            for (int ks = 0; ks < D / 64; ++ks) {
              const uint32_t sid = 2u * ks;
              mma_mxf4_ss(tmem + C::T_SA, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096),
                          idesc_mxf4(128, 128, sid), (tmem + C::T_QSF + 8 * qs) | (sid << 30),
                          (tmem + C::T_KSFA + 8 * st) | (sid << 30), ks > 0);
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < D / 64; ++ks)
              tmem_cp_32x128_x4(tmem + C::T_KSFA + 8 * st + 4 * ks, desc_at(t_sf, kb + C::QC_BYTES + ks * 512));
#pragma unroll
            for (int ks = 0; ks < D / 64; ++ks)
              mma_nvf4_ss(tmem + C::T_SA, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096), id_s,
                          tmem + C::T_QSF + 8 * qs + 4 * ks, tmem + C::T_KSFA + 8 * st + 4 * ks, ks > 0);
          }
          tc_commit(&bars[C::B_SA_FULL]);
          tc_commit(&bars[C::B_KA_EMPTY + st]);
        }
        __syncwarp();
      }
    }
  } else if (warp == C::MMA_B) {
    // ------------------------------------------------------------ MMA B: pass-2 S tiles + PV
    int it = 0, k = 0, su = 0, pc = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
      const int nt = work_item(p, w, q_tiles, k_tiles).nt;
      const int qs = k % C::NQ;
      const uint32_t qb = s0 + C::Q0 + qs * C::Q_BYTES;
      // the Q slot and its TMEM scale factors were staged by MMA A
      mbar_wait(&bars[C::B_QSF + qs], (k / C::NQ) & 1);
      tc_fence_after();
      for (int ns = 0, np = 0; np < nt;) {
        if (ns < nt && ns <= np + AQ_FWDI_SLEAD) {
          const int st = (it + ns) % C::NSB;
          mbar_wait(&bars[C::B_KB_FULL + st], ((it + ns) / C::NSB) & 1);
          if (su > 0) mbar_wait(&bars[C::B_SB_EMPTY], (su - 1) & 1);
          ++su;
          tc_fence_after();
          const uint32_t kb = s0 + C::KB0 + st * C::KB_BYTES;
          if (elect_one()) {
            if constexpr (MX) {
              tmem_cp_32x128_x4(tmem + C::T_KSFB + 8 * st, desc_at(t_sf, kb + C::QC_BYTES));
#pragma unroll
              for (int ks = 0; ks < D / 64; ++ks) {
                const uint32_t sid = 2u * ks;
                mma_mxf4_ss(tmem + C::T_SB, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096),
                            idesc_mxf4(128, 128, sid), (tmem + C::T_QSF + 8 * qs) | (sid << 30),
                            (tmem + C::T_KSFB + 8 * st) | (sid << 30), ks > 0);
              }
            } else {
#pragma unroll
              for (int ks = 0; ks < D / 64; ++ks)
                tmem_cp_32x128_x4(tmem + C::T_KSFB + 8 * st + 4 * ks, desc_at(t_sf, kb + C::QC_BYTES + ks * 512));
#pragma unroll
              for (int ks = 0; ks < D / 64; ++ks)
                mma_nvf4_ss(tmem + C::T_SB, desc_at(t_k, qb + ks * 4096), desc_at(t_k, kb + ks * 4096), id_s,
                            tmem + C::T_QSF + 8 * qs + 4 * ks, tmem + C::T_KSFB + 8 * st + 4 * ks, ks > 0);
            }
            tc_commit(&bars[C::B_SB_FULL]);
            if (ns == nt - 1) tc_commit(&bars[C::B_Q_EMPTY + qs]);  // last read of this Q slot
          }
          __syncwarp();
          ++ns;
          continue;
        }
        const int pj = np++;
        const int pb = pc % C::NP;
        const int st = (it + pj) % C::NSB;
        if (pj == 0 && k > 0) mbar_wait(&bars[C::B_O_EMPTY], (k - 1) & 1);  // previous epilogue read O
        mbar_wait(&bars[C::B_P_FULL + pb], (pc / C::NP) & 1);
        ++pc;
        tc_fence_after();
        const uint32_t sb = s0 + C::KB0 + st * C::KB_BYTES;
        const uint32_t pbase = s0 + C::P0 + pb * C::P_BYTES;
        if (elect_one()) {
          if constexpr (MX) {
            tmem_cp_32x128_x4(tmem + C::T_PSF + 8 * pb, desc_at(t_sf, pbase + C::PB_SF));
            tmem_cp_32x128_x4(tmem + C::T_VSF + 8 * st, desc_at(t_sf, sb + C::KB_VSF));
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t sid = 2u * ks;
              mma_mxf4_ss(tmem + C::T_O, desc_at(t_k, pbase + ks * 4096),
                          desc_at(t_v, sb + C::KB_V + ks * 2 * (D * 16)), idesc_mxf4(128, D, sid),
                          (tmem + C::T_PSF + 8 * pb) | (sid << 30), (tmem + C::T_VSF + 8 * st) | (sid << 30),
                          (pj > 0 || ks > 0));
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              tmem_cp_32x128_x4(tmem + C::T_PSF + 8 * pb + 4 * ks, desc_at(t_sf, pbase + C::PB_SF + ks * 512));
              tmem_cp_32x128_x4(tmem + C::T_VSF + 8 * st + 4 * ks, desc_at(t_sf, sb + C::KB_VSF + ks * 512));
            }
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
              mma_nvf4_ss(tmem + C::T_O, desc_at(t_k, pbase + ks * 4096),
                          desc_at(t_v, sb + C::KB_V + ks * 2 * (D * 16)), id_pv, tmem + C::T_PSF + 8 * pb + 4 * ks,
                          tmem + C::T_VSF + 8 * st + 4 * ks, (pj > 0 || ks > 0));
          }
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
  } else {
    // ------------------------------------------------------------ softmax groups
    const bool grp_a = warp >= C::WA && warp < C::WA + C::NSW;
    const int gw = grp_a ? warp - C::WA : warp - C::WB;  // warp within its group
    const int row = 32 * (gw & 3) + lane;            // TMEM lane == query row
    const int half = gw >> 2;
    constexpr int CW = C::CW;
    const int cbase = half * CW;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>((gw & 3) * 32) << 16);
    const float sl2 = p.scale_log2;
    const float p_r = p.p_r;  // 1 / t_p (1 = the reference's P^F)
    float x[CW];
    int su = 0, pc = 0, k = 0;
    AQ_IPROF(long long ipa[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; const long long istart = clock64();)
    auto idump = [&](bool ga) {
      AQ_IPROF(if ((p.debug & 32) && lane == 0) {
        const long long tot = clock64() - istart;
        if (ga) {
          atomicAdd(&g_iprof[0], static_cast<unsigned long long>(ipa[0]));
          atomicAdd(&g_iprof[1], static_cast<unsigned long long>(ipa[1]));
          atomicAdd(&g_iprof[2], static_cast<unsigned long long>(tot));
          atomicAdd(&g_iprof[3], static_cast<unsigned long long>(ipa[3]));
        } else {
          for (int e = 4; e < 10; ++e) atomicAdd(&g_iprof[e + 4], static_cast<unsigned long long>(ipa[e]));
          atomicAdd(&g_iprof[14], static_cast<unsigned long long>(tot));
        }
      })
      (void)ga;
    };
    int chk_wait = 0, chk_pen = 0;  // early-out back-off (warp-uniform)
    const bool early_out = EARLY && (p.debug & 64) == 0;  // AQ_FWD_DEBUG bit 64 disables it (A/B timing)
    float* ml = reinterpret_cast<float*>(smem + C::ML);
    float* lb = reinterpret_cast<float*>(smem + C::LB);
    if (grp_a) {
      if constexpr (C::REALLOC) setmaxnreg_inc<C::REG_A>();
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const Item item = work_item(p, w, q_tiles, k_tiles);
        const int nt = item.nt;
        const int64_t grow = static_cast<int64_t>(item.qt) * TILE + row;
        int64_t kmax = p.n_k - 1;
        if (p.causal) kmax = min(kmax, grow + (p.n_k - p.n_q));
        const int qs = k % C::NQ;
          // ---------------- pass 1: online (m, l) over this thread's 64 columns
          // (log2 domain). Same code and merge order as the CS=2 column split of
          // the training kernel (attn_fwd.cu), so L (hence P, P^F and O) is
          // bit-identical between the two forward kernels.
          float m = -INFINITY, l = 0.f;
          for (int jj = 0; jj < nt; ++jj) {
            AQ_IPROF(long long t0 = clock64();)
            mbar_wait(&bars[C::B_SA_FULL], su & 1);
            AQ_IPROF(ipa[0] += clock64() - t0; ipa[3] += 1;)
            ++su;
            tc_fence_after();
  #pragma unroll
            for (int c0 = 0; c0 < CW; c0 += 32) tmem_ld32f(t_lane + C::T_SA + cbase + c0, x + c0);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&bars[C::B_SA_EMPTY]);
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
  #ifdef AQ_DBG_NOEXP1
                const float2 e = t;
  #else
                const float2 e = use_poly_p1(cbase / 2 + i) ? ex2_pair<true>(t) : ex2_pair<false>(t);
  #endif
                acc[i & 3] = __fadd2_rn(acc[i & 3], e);
              }
              const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
              const float2 s4 = __fadd2_rn(s01, s23);
              return s4.x + s4.y;
            };
            float sum = expsum(m == -INFINITY ? 0.f : m);
            // A rebase needs a term above 2^8, hence sum > 240 (or inf): only then (and
            // while no column is visible yet) is the tile max needed. Same m sequence,
            // hence the same bits, as taking the max of every tile.
            if (!(sum <= 240.0f) || m == -INFINITY) {
              float mx[8];
  #pragma unroll
              for (int a = 0; a < 8; ++a) mx[a] = x[a];
  #pragma unroll
              for (int c = 8; c < CW; ++c) mx[c & 7] = fmaxf(mx[c & 7], x[c]);
              const float mloc = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                       fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
              if (mloc > m + 8.0f) {  // first visible tile, or a much larger max: rebase
                l = (m == -INFINITY) ? 0.f : l * ex2(m - mloc);
                m = mloc;
                sum = expsum(m);
              }
            }
            l += sum;
          }
          // merge the column-split partials of each row
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
          // rebuilds L2 = fl(L) * log2(e) exactly like the backward does
          const float L_nat = (mt + __log2f(lt)) * 0.69314718055994530942f;
          if (half == 0 && grow < p.n_q) p.lse[item.head * p.n_q + grow] = L_nat;
          AQ_IPROF(long long t1 = clock64();)
          if (k >= C::NQ) mbar_wait(&bars[C::B_L_EMPTY + qs], ((k / C::NQ) - 1) & 1);
          AQ_IPROF(ipa[1] += clock64() - t1;)
          if (half == 0) lb[qs * TILE + row] = L_nat;
          mbar_arrive(&bars[C::B_L_FULL + qs]);
      }
      idump(true);
    } else {
      if constexpr (C::REALLOC) setmaxnreg_dec<C::REG_B>();
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++k) {
        const Item item = work_item(p, w, q_tiles, k_tiles);
        const int nt = item.nt;
        const int64_t grow = static_cast<int64_t>(item.qt) * TILE + row;
        int64_t kmax = p.n_k - 1;
        if (p.causal) kmax = min(kmax, grow + (p.n_k - p.n_q));
        const int qs = k % C::NQ;
          // ---------------- pass 2: P, P^F, O (CSB column splits of CWB keys per thread)
          constexpr int CW = C::CWB;
          const int half = gw >> 2;  // column split of this thread (pass 2)
          const int cbase = half * CW;
          AQ_IPROF(long long t1 = clock64();)
          mbar_wait(&bars[C::B_L_FULL + qs], (k / C::NQ) & 1);
          AQ_IPROF(ipa[5] += clock64() - t1;)
          const float L2 = lb[qs * TILE + row] * 1.44269504088896340736f;
          mbar_arrive(&bars[C::B_L_EMPTY + qs]);
          const float thr = p_skip_thr(L2 + p.p_lshift, sl2);  // blocks of P * p_r below 2^-11
          for (int jj = 0; jj < nt; ++jj) {
            AQ_IPROF(long long t0 = clock64();)
            mbar_wait(&bars[C::B_SB_FULL], su & 1);
            AQ_IPROF(ipa[4] += clock64() - t0; ipa[9] += 1;)
            ++su;
            tc_fence_after();
  #pragma unroll
            for (int c0 = 0; c0 < CW; c0 += 32) tmem_ld32f(t_lane + C::T_SB + cbase + c0, x + c0);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&bars[C::B_SB_EMPTY]);
            const int64_t lim = kmax - (static_cast<int64_t>(jj) * TILE + cbase);
            // claim the P^F buffer first, so P = exp(S - L), its quantization and the
            // stores form one straight-line block per 32 keys that the scheduler can
            // interleave (MUFU work of one group overlaps ALU work of the previous)
            const int pb = pc % C::NP;
            AQ_IPROF(long long t2 = clock64();)
            if (pc >= C::NP) mbar_wait(&bars[C::B_P_EMPTY + pb], ((pc / C::NP) - 1) & 1);
            AQ_IPROF(ipa[6] += clock64() - t2;)
            ++pc;
            uint8_t* pcodes = smem + C::P0 + pb * C::P_BYTES;
            uint8_t* psf = pcodes + C::PB_SF;
            uint32_t scw[(CW + 63) / 64];
  #pragma unroll
            for (int s = 0; s < (CW + 63) / 64; ++s) scw[s] = 0;
            auto group32 = [&](int blk, bool masked) {
  #ifndef AQ_DBG_NOEXP2
              p_from_s<16>(x + blk * 16, cbase + blk * 16, sl2, L2);
  #endif
              if (masked) {
  #pragma unroll
                for (int c = 0; c < 32; ++c) x[blk * 16 + c] = (blk * 16 + c <= lim) ? x[blk * 16 + c] : 0.f;
              }
  #ifdef AQ_DBG_NOQ2
              PBlock qa, qb;
              qa.scale = __float_as_uint(x[blk * 16]) & 0xff; qa.codes[0] = __float_as_uint(x[blk * 16 + 1]); qa.codes[1] = __float_as_uint(x[blk * 16 + 2]);
              qb = qa;
  #else
              if constexpr (MX) {
                uint32_t cd[4], sc;
                quantize_p32_mx(x + blk * 16, cd, sc);
                *reinterpret_cast<uint4*>(pcodes + t8x32_off(row, cbase + blk * 16, TILE)) =
                    make_uint4(cd[0], cd[1], cd[2], cd[3]);
                scw[0] |= sc << (8 * (blk / 2));
                return;
              }
              const PBlock qa = quantize_p16_s(x + blk * 16, p_r);
              const PBlock qb = quantize_p16_s(x + blk * 16 + 16, p_r);
  #endif
              *reinterpret_cast<uint4*>(pcodes + t8x32_off(row, cbase + blk * 16, TILE)) =
                  make_uint4(qa.codes[0], qa.codes[1], qb.codes[0], qb.codes[1]);
              scw[blk / 4] |= (qa.scale << (8 * (blk & 3))) | (qb.scale << (8 * ((blk + 1) & 3)));
            };
            // exact early-out (pquant.cuh): 16-key blocks whose P is below 2^-11 in
            // every row of the warp get P^F = 0 with scale 0x01 without an exponential.
            // Checked with exponential back-off, so workloads where blocks rarely
            // qualify (short rows) pay for one check every ~16 tiles.
            uint32_t sk = 0;
            if constexpr (!MX) {
              if (early_out && chk_wait == 0) {  // warp-uniform; lanes with masked keys vote 0
                sk = __reduce_and_sync(0xffffffffu, lim >= CW - 1 ? p_skip_mask<CW / 16>(x, thr) : 0u);
                if (sk == 0) {
                  chk_pen = min(2 * chk_pen + 1, 15);
                  chk_wait = chk_pen;
                } else {
                  chk_pen = 0;
                }
              } else if (chk_wait > 0) {
                --chk_wait;
              }
            }
            if (sk != 0) {
  #pragma unroll
              for (int blk = 0; blk < CW / 16; blk += 2) {
                PBlock qa, qb;
                qa.scale = qb.scale = 1u;
                qa.codes[0] = qa.codes[1] = qb.codes[0] = qb.codes[1] = 0u;
                if (!((sk >> blk) & 1u)) {
                  p_from_s<8>(x + blk * 16, cbase + blk * 16, sl2, L2);
                  qa = quantize_p16_s(x + blk * 16, p_r);
                }
                if (!((sk >> (blk + 1)) & 1u)) {
                  p_from_s<8>(x + blk * 16 + 16, cbase + blk * 16 + 16, sl2, L2);
                  qb = quantize_p16_s(x + blk * 16 + 16, p_r);
                }
                *reinterpret_cast<uint4*>(pcodes + t8x32_off(row, cbase + blk * 16, TILE)) =
                    make_uint4(qa.codes[0], qa.codes[1], qb.codes[0], qb.codes[1]);
                scw[blk / 4] |= (qa.scale << (8 * (blk & 3))) | (qb.scale << (8 * ((blk + 1) & 3)));
              }
            } else if (lim >= CW - 1) {
  #pragma unroll
              for (int blk = 0; blk < CW / 16; blk += 2) group32(blk, false);
            } else {
  #pragma unroll
              for (int blk = 0; blk < CW / 16; blk += 2) group32(blk, true);
            }
            if constexpr (MX) {
              if constexpr (CW >= 64)
                *reinterpret_cast<uint16_t*>(psf + sf512_off(row, cbase / 32)) = static_cast<uint16_t>(scw[0]);
              else
                psf[sf512_off(row, cbase / 32)] = static_cast<uint8_t>(scw[0]);
            } else if constexpr (CW >= 64) {
  #pragma unroll
              for (int s = 0; s < CW / 64; ++s)
                *reinterpret_cast<uint32_t*>(psf + sf512_off(row, cbase / 16 + 4 * s)) = scw[s];
            } else {
              *reinterpret_cast<uint16_t*>(psf + sf512_off(row, cbase / 16)) = static_cast<uint16_t>(scw[0]);
            }
            if (p.pf_codes != nullptr && grow < p.n_q) {  // instrument: this row's P^F of the tile
              const int64_t n16 = ceil_div(p.n_k, 16);
              const int64_t c0 = static_cast<int64_t>(jj) * TILE + cbase;  // first key of this thread
              uint8_t* dc = p.pf_codes + (item.head * p.n_q + grow) * (n16 * 8);
              uint8_t* ds = p.pf_scales + (item.head * p.n_q + grow) * n16;
  #pragma unroll
              for (int b = 0; b < CW / 16; ++b) {
                const int64_t blk = c0 / 16 + b;
                if (blk < n16) {
                  *reinterpret_cast<uint2*>(dc + blk * 8) =
                      *reinterpret_cast<const uint2*>(pcodes + t8x32_off(row, cbase + 16 * b, TILE));
                  ds[blk] = psf[sf512_off(row, cbase / 16 + b)];
                }
              }
            }
            fence_async_smem();
            mbar_arrive(&bars[C::B_P_FULL + pb]);
          }
          // epilogue: O rows -> registers, release O, store
          AQ_IPROF(long long t3 = clock64();)
          mbar_wait(&bars[C::B_O_FULL], k & 1);
          AQ_IPROF(ipa[7] += clock64() - t3;)
          tc_fence_after();
          constexpr int DW = D / C::CSB;
          float o[DW];
          if constexpr (DW >= 32) {
  #pragma unroll
            for (int c = 0; c < DW; c += 32) tmem_ld32f(t_lane + C::T_O + half * DW + c, o + c);
          } else {
            uint32_t r16[16];
            tmem_ld16(t_lane + C::T_O + half * DW, r16);
  #pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __uint_as_float(r16[c]);
          }
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&bars[C::B_O_EMPTY]);
          if (p.o_mul != 1.f) {  // per-tensor scales t_v t_p (two-level NVFP4)
  #pragma unroll
            for (int c = 0; c < DW; ++c) o[c] *= p.o_mul;
          }
          if (grow < p.n_q && p.o != nullptr) {
            const int64_t base = (item.head * p.n_q + grow) * D + half * DW;
            if (p.o_dt == 0) {
              float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.o) + base);
  #pragma unroll
              for (int e = 0; e < DW; e += 4) d4[e / 4] = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
            } else {
              uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.o) + base);
  #pragma unroll
              for (int e = 0; e < DW; e += 8) {
                uint32_t h[4];
  #pragma unroll
                for (int q = 0; q < 4; ++q) {
                  if (p.o_dt == 1) {
                    const __nv_bfloat162 v = __floats2bfloat162_rn(o[e + 2 * q], o[e + 2 * q + 1]);
                    h[q] = *reinterpret_cast<const uint32_t*>(&v);
                  } else {
                    const __half2 v = __floats2half2_rn(o[e + 2 * q], o[e + 2 * q + 1]);
                    h[q] = *reinterpret_cast<const uint32_t*>(&v);
                  }
                }
                d4[e / 8] = make_uint4(h[0], h[1], h[2], h[3]);
              }
            }
          }
      }
      idump(false);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#ifndef AQ_FWDI_EARLY_NK
#define AQ_FWDI_EARLY_NK 24576
#endif
template <int D, bool MX = false>
cudaError_t launch(const FwdParams& p, cudaStream_t st) {
  using C = Cfg<D>;
  // The early-out pays where long rows push most P blocks below 2^-11 (C3
  // N = 32760: 75 % of warp blocks, 23.9 -> 20.0 ms; N = 32K causal 19.3 ->
  // 18.8 ms); for shorter rows its code costs more than it skips (C2 N = 8192
  // causal 2.63 -> 2.77 ms, N = 16K non-causal 19.0 -> 19.8 ms), so those run
  // the instance without it. Both give identical bits.
  auto kern = (!MX && p.n_k >= AQ_FWDI_EARLY_NK) ? attn_fwd_infer_kernel<D, MX, !MX> : attn_fwd_infer_kernel<D, MX, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::TOTAL);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = p.heads * ceil_div(p.n_q, TILE);
  const int grid = static_cast<int>(items < sms ? items : sms);
  kern<<<grid, C::NUM_THREADS, C::TOTAL, st>>>(p);
  return cudaGetLastError();
}

}  // namespace fwdi

extern "C" int aq_debug_fwdi_profile(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, fwdi::g_iprof, sizeof(fwdi::g_iprof)) != cudaSuccess) return 5;
  if (reset) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(fwdi::g_iprof, z, sizeof(z)) != cudaSuccess) return 5;
  }
  return 0;
}

cudaError_t launch_attn_fwd_infer(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return fwdi::launch<64>(p, st);
  if (p.d == 128) return fwdi::launch<128>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_attn_fwd_infer_mx(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return fwdi::launch<64, true>(p, st);
  if (p.d == 128) return fwdi::launch<128, true>(p, st);
  return cudaErrorInvalidValue;
}

}  // namespace aq
