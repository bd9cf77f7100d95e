// K4 / K5: fused two-pass NVFP4 attention forward on tcgen05 (sm_100a).
//
// Follows flash_forward_training / flash_forward_inference
// (attnqat/flash.py:176-246, :249-314): for each 128-row query tile
//   pass 1  S = Q^F K^F^T (FP4 block-scaled MMA, TMEM) -> online (m, l)
//           -> L = m + log l                               (flash.py:145-173, 217)
//   pass 2  S again -> P = exp(S - L) -> P^F = NVFP4(P) over 16-key blocks
//           aligned to global key index            (flash.py:222-236, 67-71)
//           O  += P^F V^F    (FP4 block-scaled MMA)
//           O' += P   V^F    (training only; kind::f16 with fp16 P^ = exp(S-m)
//                             and 1/l applied in the epilogue)
// O needs no rescaling: L is final before pass 2.
//
// Persistent kernel: one CTA per SM walks a static list of (head, query tile)
// work items (longest causal rows first). Roles:
//  * softmax warps (4*CS): warp w owns TMEM lanes 32*(w%4).. (one query row
//    per thread) and key columns [(w/4)*128/CS, ...) of every S tile; pass-1
//    (m, l) partials of a row are merged once per item, P^F blocks of 16 keys
//    never straddle a column split;
//  * one producer warp: 1-D bulk copies of pre-tiled Q / K / V operands
//    (layouts.cuh), running ahead across item boundaries;
//  * one MMA warp: the whole warp runs the schedule in warp-uniform registers,
//    an elected lane issues tcgen05.cp / mma / commit.
// K/V stream through an NS-stage ring, S through NB1 (pass 1) / NB2 (pass 2)
// TMEM buffers, P^F through NP SMEM buffers; every ring counts phases across
// items.
// Further instances (template flags, see the comments above attn_fwd_kernel):
// SAGE (sage3.py smoothing terms, two-level P with TRAIN), PLAIN
// (quantized=False: 16-bit S and P^V on kind::f16) and MX (MXFP4 operands on
// kind::mxf4 block32, 32-key UE8M0 P blocks).
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "pquant.cuh"
#include "ptx.cuh"
#include "rowstore.cuh"

namespace aq {

namespace fwd {

// float <-> unsigned with the same order (atomicMax on floats); 0 is below
// every encoded value, so a zeroed buffer is the identity
__device__ __forceinline__ unsigned f2ord(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// Tuning aid, compiled in with -DAQ_FWD_PROFILE and enabled at run time by
// AQ_FWD_DEBUG bit 32: cycle sums per softmax segment, accumulated from lane
// 0 of every softmax warp.
__device__ unsigned long long g_prof[16];
#ifdef AQ_FWD_PROFILE
#define AQ_PROF(...) __VA_ARGS__
#else
#define AQ_PROF(...)
#endif

template <int D, bool TRAIN, int CS, bool SAGE = false, bool PLAIN = false, bool MX = false>
struct Cfg {
  static_assert(!MX || (!SAGE && !PLAIN), "MXFP4 runs the plain NVFP4 layouts");
  static_assert(!PLAIN || (TRAIN && !SAGE), "plain attention runs on the training layout");
  static constexpr int NSW = 4 * CS;                 // softmax warps
  static constexpr int NUM_THREADS = 32 * (NSW + 3);
  static constexpr int PRODUCER = NSW, PRODUCER1 = NSW + 1, MMA = NSW + 2;
  static constexpr int NK1 = PLAIN ? 2 : 4;          // K ring (K codes + SF; 16-bit K for PLAIN), both passes
  static constexpr int CW = TILE / CS;               // key columns per softmax thread
  static constexpr int NS = TRAIN ? 2 : 5;           // V stages
  static constexpr int NB1 = 3;                      // S buffers in pass 1 (1 and 2 alias O / O')
  static constexpr int NB2 = TRAIN ? 1 : 2;          // S buffers in pass 2
  static constexpr int NP = TRAIN ? 2 : 3;           // P^F (and P^) buffers
  // TMEM columns: S buffer b at 128*b
  static constexpr uint32_t T_O = TRAIN ? 128 : 256, T_OP = 256;
  static constexpr uint32_t T_QSF = 384, T_PSF = T_QSF + 8, T_VSF = T_PSF + 8 * NP, T_KSF1 = T_VSF + 8 * NS;
  // shared memory
  static constexpr int Q_CODES = 0;                   // FP4 Q (16-bit Q tile for PLAIN)
  static constexpr int Q_SF = Q_CODES + (PLAIN ? TILE * D * 2 : TILE * D / 2);
  static constexpr int STAGE0 = Q_SF + (PLAIN ? 0 : (D / 64) * 512);
  // pass-2 stage: V^T codes + scale factors (+ V^F fp16); K tiles of both
  // passes come through the small K ring of producer 1
  static constexpr int ST_V = 0;
  static constexpr int ST_VSF = ST_V + (PLAIN ? 0 : TILE * D / 2);
  static constexpr int ST_VH = ST_VSF + (PLAIN ? 0 : 1024);
  static constexpr int STAGE_BYTES = ST_VH + (TRAIN ? TILE * D * 2 : 0);
  static constexpr int P0 = STAGE0 + NS * STAGE_BYTES;
  static constexpr int PB_CODES = 0, PB_SF = PLAIN ? 0 : TILE * TILE / 2, PB_H = PB_SF + (PLAIN ? 0 : 1024);
  static constexpr int P_BYTES = PB_H + (TRAIN ? TILE * TILE * 2 : 0);
  static constexpr int ML = P0 + NP * P_BYTES;       // pass-1 (m, l) partials
  // (m, l) partials (+ the exact row max and the two-level P exchange with SAGE)
  static constexpr int K1_0 = ML + (SAGE ? 3 : 2) * CS * TILE * 4;  // pass-1 K ring
  static constexpr int K1_BYTES = PLAIN ? TILE * D * 2 : TILE * D / 2 + (D / 64) * 512;
  // SAGE: per softmax warp, two 512-byte delta buffers (up to two q_bar rows x 64 keys)
  static constexpr int DL = K1_0 + NK1 * K1_BYTES;
  static constexpr int BARS = DL + (SAGE ? NSW * 1024 : 0);
  static constexpr int NUM_BARS = 48;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int NIQ = 4;                      // dynamic-schedule item ring (ItemQ)
  static constexpr int IQ = TMEM_SLOT + 16;
  static constexpr int USED = IQ + NIQ * 8;
  // one CTA per SM (the kernel owns all 512 TMEM columns)
  static constexpr int TOTAL = USED > 120 * 1024 ? USED : 120 * 1024;
  static constexpr int Q_BYTES = PLAIN ? TILE * D * 2 : TILE * D / 2 + (D / 64) * 512;
  static constexpr int K_BYTES = K1_BYTES;
  static constexpr int V_BYTES = PLAIN ? TILE * D * 2 : TILE * D / 2 + 1024 + (TRAIN ? TILE * D * 2 : 0);
  // barrier slots
  static constexpr int B_Q_FULL = 0, B_Q_EMPTY = 1, B_O_FULL = 2, B_O_EMPTY = 3, B_KV_FULL = 4,
                       B_KV_EMPTY = B_KV_FULL + NS, B_S_FULL = B_KV_EMPTY + NS, B_S_EMPTY = B_S_FULL + NB1,
                       B_P_FULL = B_S_EMPTY + NB1, B_P_EMPTY = B_P_FULL + NP, B_K1_FULL = B_P_EMPTY + NP,
                       B_K1_EMPTY = B_K1_FULL + NK1, B_IQ_FULL = B_K1_EMPTY + NK1, B_IQ_EMPTY = B_IQ_FULL + NIQ,
                       B_END = B_IQ_EMPTY + NIQ;
  static_assert(B_END <= NUM_BARS, "barrier slots");
  static_assert(USED <= 227 * 1024, "shared memory");
  static_assert(T_KSF1 + 8 * NK1 <= 512, "TMEM columns");
};

// Work item w -> (head, query tile, key tiles). Causal items are ordered by
// decreasing row length across all heads (longest-processing-time first), so
// the static round-robin over CTAs balances; K/V re-reads this causes stay
// far below the HBM roofline (ncu: ~1 TB/s on C2).
struct Item {
  int64_t head;
  int qt, nt;
};

#ifndef AQ_FWD_SNAKE_ROUNDS
#define AQ_FWD_SNAKE_ROUNDS 24
#endif
__device__ __forceinline__ Item work_item(const FwdParams& p, int64_t w, int q_tiles, int k_tiles) {
  Item it;
  if (p.causal && !p.item_ctr && p.heads * q_tiles < AQ_FWD_SNAKE_ROUNDS * static_cast<int64_t>(gridDim.x)) {
    // few rounds per CTA (e.g. a head shard on one of 8 GPUs): boustrophedon over
    // the CTAs as in K5, so the per-CTA sums of causal row lengths balance
    // (32 heads x 32 tiles: makespan / mean 1.14 -> 1.02); with many rounds the
    // plain order balances by itself and keeps consecutive heads together in L2
    const int64_t G = gridDim.x, r = w / G;
    if ((r & 1) && (r + 1) * G <= p.heads * q_tiles) w = r * G + (G - 1 - (w - r * G));
  }
  if (p.causal && p.head_group > 0) {
    // longest-first within groups of G heads, so the CTAs in flight share the
    // K / V tiles of a few heads in L2 (the 16-bit PLAIN operands are 4x the
    // FP4 bytes and would otherwise stream from HBM for every query tile)
    const int64_t gsz = static_cast<int64_t>(p.head_group) * q_tiles;
    const int64_t g = w / gsz, r = w % gsz;
    const int64_t G = min(static_cast<int64_t>(p.head_group), p.heads - g * p.head_group);
    it.qt = q_tiles - 1 - static_cast<int>(r / G);
    it.head = g * p.head_group + r % G;
    const int64_t last =
        static_cast<int64_t>(min(it.qt * TILE + TILE - 1, static_cast<int>(p.n_q) - 1)) + (p.n_k - p.n_q);
    it.nt = min(k_tiles, static_cast<int>(last / TILE) + 1);
  } else if (p.causal && p.item_ctr) {
    // dynamic schedule (see next_item): bands of item_band query tiles,
    // longest band first; inside a band head-major, longest row first. The
    // CTAs in flight then share each head's K / V / V^F tiles item_band ways in
    // L2, and the rows left for the queue's tail are at most item_band tiles
    const int64_t band = min(p.item_band, q_tiles), full = q_tiles / band;
    int64_t b, r, bs;
    if (w < full * band * p.heads) {
      b = w / (band * p.heads);
      r = w % (band * p.heads);
      bs = band;
    } else {
      b = full;
      r = w - full * band * p.heads;
      bs = q_tiles - full * band;
    }
    it.head = r / bs;
    it.qt = q_tiles - 1 - static_cast<int>(b * band + r % bs);
    const int64_t last =
        static_cast<int64_t>(min(it.qt * TILE + TILE - 1, static_cast<int>(p.n_q) - 1)) + (p.n_k - p.n_q);
    it.nt = min(k_tiles, static_cast<int>(last / TILE) + 1);
  } else if (p.causal) {
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

// running use counters of the NB1 S buffers (warp-uniform, no dynamic indexing)
struct SUses {
  int u0 = 0, u1 = 0, u2 = 0;
  __device__ __forceinline__ int take(int b) {
    const int u = b == 0 ? u0 : (b == 1 ? u1 : u2);
    if (b == 0) ++u0; else if (b == 1) ++u1; else ++u2;
    return u;
  }
};

// SAGE (sage3.py:113-194): the scores gain the high-precision smoothing terms
// S += delta[q tile][key] + bias[row] before the softmax (both passes); with
// TRAIN the kernel runs two-level P instead of O' -- P^F is quantized from
// P * r (r = 448*6 / max P over the row's key segment) and the f16 MMA
// accumulates dequant(P^F) * l / r, so the 1/r of every segment is applied
// before the accumulation (the FP4 PV MMA is skipped; O comes out of the O'
// epilogue).
// PLAIN (quantized=False, flash.py:195-200): S = Q K^T on 16-bit operands
// (kind::f16, fp16 or bf16 per p.plain_fmt), no P quantization, O = P^ V
// through the O' path with 1/l in the epilogue (written to p.o_hp).
// MX (MXFP4, codec.py:123-203 with flash.py:249-314): the same tiles and
// scale-factor images (one image per 128 K holds four UE8M0 scales), S and PV
// on kind::mxf4 block32 with scale-factor IDs 0 / 2 per K = 64 step, P
// quantized in 32-key blocks.
template <int D, bool TRAIN, int CS, bool SAGE = false, bool PLAIN = false, bool MX = false>
__global__ void __launch_bounds__(Cfg<D, TRAIN, CS, SAGE, PLAIN, MX>::NUM_THREADS, 1) attn_fwd_kernel(const FwdParams p) {
  using C = Cfg<D, TRAIN, CS, SAGE, PLAIN, MX>;
  static_assert(!SAGE || CS == 2, "the sage3 instances use 64 key columns per thread");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::TMEM_SLOT);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const int64_t n_items = p.heads * q_tiles;

  if (threadIdx.x == 0) {
    mbar_init(&bars[C::B_Q_FULL], 1);
    mbar_init(&bars[C::B_Q_EMPTY], 1);
    mbar_init(&bars[C::B_O_FULL], 1);
    mbar_init(&bars[C::B_O_EMPTY], 32 * C::NSW);
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&bars[C::B_KV_FULL + s], 1);
      mbar_init(&bars[C::B_KV_EMPTY + s], 1);
    }
    for (int b = 0; b < C::NB1; ++b) {
      mbar_init(&bars[C::B_S_FULL + b], 1);
      mbar_init(&bars[C::B_S_EMPTY + b], 32 * C::NSW);
    }
    for (int b = 0; b < C::NP; ++b) {
      mbar_init(&bars[C::B_P_FULL + b], 32 * C::NSW);
      mbar_init(&bars[C::B_P_EMPTY + b], 1);
    }
    for (int s = 0; s < C::NK1; ++s) {
      mbar_init(&bars[C::B_K1_FULL + s], 1);
      mbar_init(&bars[C::B_K1_EMPTY + s], 1);
    }
    for (int s = 0; s < C::NIQ; ++s) {
      mbar_init(&bars[C::B_IQ_FULL + s], 1);
      mbar_init(&bars[C::B_IQ_EMPTY + s], 2 + C::NSW);  // producer, MMA and softmax warps
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Work items. Static: the CTA's k-th item is blockIdx.x + k * gridDim.x.
  // Dynamic (p.item_ctr, causal rows; work_item's head-major order): producer
  // 1, the role that runs furthest ahead, claims items from a global counter
  // (zeroed before the launch; the first item is blockIdx.x, one claim in
  // flight ahead of use) and publishes them through an NIQ-slot ring; every
  // other warp reads the ring and releases its slot. -1 = no more items.
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

  if (warp == C::PRODUCER) {
    // ------------------------------------------------------------ producer
    int it = 0, k = 0;
    for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
      const Item item = work_item(p, w, q_tiles, k_tiles);
      const int64_t qtile_idx = item.head * q_tiles + item.qt;
      if (k > 0) mbar_wait(&bars[C::B_Q_EMPTY], (k - 1) & 1);
      if (elect_one()) {
        mbar_expect_tx(&bars[C::B_Q_FULL], C::Q_BYTES);
        if (PLAIN) {
          bulk_g2s(smem + C::Q_CODES, p.q_codes + qtile_idx * h_tile_bytes(D), TILE * D * 2, &bars[C::B_Q_FULL]);
        } else {
          bulk_g2s(smem + C::Q_CODES, p.q_codes + qtile_idx * fp4_tile_bytes(D), TILE * D / 2, &bars[C::B_Q_FULL]);
          bulk_g2s(smem + C::Q_SF, p.q_sf + qtile_idx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[C::B_Q_FULL]);
        }
      }
      __syncwarp();
      // pass-2 stages (V [+ V^F]); the K tiles of both passes come from producer 1's ring
      for (int j = 0; j < item.nt; ++j, ++it) {
        const int st = it % C::NS;
        if (it >= C::NS) mbar_wait(&bars[C::B_KV_EMPTY + st], ((it / C::NS) - 1) & 1);
        uint8_t* sb = smem + C::STAGE0 + st * C::STAGE_BYTES;
        const int64_t kt_idx = item.head * k_tiles + j;
        uint64_t* fb = &bars[C::B_KV_FULL + st];
        if (elect_one()) {
          mbar_expect_tx(fb, C::V_BYTES);
          if (!PLAIN) {
            bulk_g2s(sb + C::ST_V, p.v_codes + kt_idx * fp4_tile_bytes(D), TILE * D / 2, fb);
            bulk_g2s(sb + C::ST_VSF, p.v_sf + kt_idx * kSfTileBytesV, 1024, fb);
          }
          if (TRAIN) bulk_g2s(sb + C::ST_VH, p.v_h + kt_idx * h_tile_bytes(D), TILE * D * 2, fb);
        }
        __syncwarp();
      }
    }
  } else if (warp == C::PRODUCER1) {
    // ------------------------------------------------------------ producer 1: K ring
    // K codes + scale factors only (9 KB per tile), NK1 deep, for the S MMAs of
    // both passes, running ahead independently of the large pass-2 stages
    int i1 = 0;
    int claim = 0;  // lane 0: the next claimed item (dynamic)
    if (dyn && lane == 0) claim = static_cast<int>(gridDim.x) + atomicAdd(p.item_ctr, 1);
    for (int kk = 0;; ++kk) {
      int64_t w;
      if (!dyn) {
        w = blockIdx.x + static_cast<int64_t>(kk) * gridDim.x;
        if (w >= n_items) break;
      } else {
        w = kk == 0 ? static_cast<int64_t>(blockIdx.x) : static_cast<int64_t>(__shfl_sync(~0u, claim, 0));
        if (kk > 0 && lane == 0 && w < n_items) claim = static_cast<int>(gridDim.x) + atomicAdd(p.item_ctr, 1);
        const int s = kk % C::NIQ;
        if (kk >= C::NIQ) mbar_wait(&bars[C::B_IQ_EMPTY + s], ((kk / C::NIQ) - 1) & 1);
        if (lane == 0) {
          iq[s] = w < n_items ? w : -1;
          mbar_arrive(&bars[C::B_IQ_FULL + s]);
        }
        __syncwarp();
        if (w >= n_items) break;
      }
      const Item item = work_item(p, w, q_tiles, k_tiles);
      for (int jp = 0; jp < 2 * item.nt; ++jp, ++i1) {
        const int j = jp % item.nt;  // pass 1 then pass 2 re-read the same K tiles
        const int st = i1 % C::NK1;
        if (i1 >= C::NK1) mbar_wait(&bars[C::B_K1_EMPTY + st], ((i1 / C::NK1) - 1) & 1);
        uint8_t* sb = smem + C::K1_0 + st * C::K1_BYTES;
        const int64_t kt_idx = item.head * k_tiles + j;
        uint64_t* fb = &bars[C::B_K1_FULL + st];
        if (elect_one()) {
          mbar_expect_tx(fb, C::K_BYTES);
          if (PLAIN) {
            bulk_g2s(sb, p.k_codes + kt_idx * h_tile_bytes(D), TILE * D * 2, fb);
          } else {
            bulk_g2s(sb, p.k_codes + kt_idx * fp4_tile_bytes(D), TILE * D / 2, fb);
            bulk_g2s(sb + TILE * D / 2, p.k_sf + kt_idx * sf_tile_bytes_qk(D), (D / 64) * 512, fb);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == C::MMA) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_nvf4(128, 128);
    constexpr uint32_t id_pv = idesc_nvf4(128, D);
    const uint32_t id_op = idesc_f16(128, D, PLAIN ? static_cast<uint32_t>(p.plain_fmt) : 0u, /*a_mn*/ 0, /*b_mn*/ 1);
    const uint32_t id_s16 = idesc_f16(128, 128, static_cast<uint32_t>(p.plain_fmt), 0, 0);  // PLAIN S
    constexpr uint64_t t_k = desc_template(2048, 128);       // Q / K / P^F codes (K-major T8x32, 128 rows)
    constexpr uint64_t t_v = desc_template(D * 16, 128);     // V^T codes (K-major T8x32, D rows)
    constexpr uint64_t t_sf = desc_template(0, 128);         // SF512 images for tcgen05.cp
    constexpr uint64_t t_ph = desc_template(2048, 128);      // P^ fp16 (K-major T8x8)
    constexpr uint64_t t_vh = desc_template(128, 2048);      // V^F fp16 (MN-major T8x8)
    const uint32_t s0 = smem_u32(smem);
    const uint32_t q_base = s0 + C::Q_CODES;
    int it = 0, pc = 0, k = 0;
    SUses su;
    // S(i1) into buffer b, K from producer 1's ring (both passes, in order)
    int i1 = 0;
    auto issue_s1 = [&](int b) {
      const int u = su.take(b);
      const int st = i1 % C::NK1;
      mbar_wait(&bars[C::B_K1_FULL + st], (i1 / C::NK1) & 1);
      if (u > 0) mbar_wait(&bars[C::B_S_EMPTY + b], (u - 1) & 1);
      tc_fence_after();
      const uint32_t kb = s0 + C::K1_0 + st * C::K1_BYTES;
      if (elect_one()) {
        if constexpr (PLAIN) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks)
            mma_f16_ss(tmem + 128 * b, desc_at(t_ph, q_base + ks * 4096), desc_at(t_ph, kb + ks * 4096), id_s16,
                       ks > 0);
        } else if constexpr (MX) {
          tmem_cp_32x128_x4(tmem + C::T_KSF1 + 8 * st, desc_at(t_sf, kb + TILE * D / 2));
#pragma unroll
          for (int ks = 0; ks < D / 64; ++ks) {
            const uint32_t sid = 2u * ks;
            mma_mxf4_ss(tmem + 128 * b, desc_at(t_k, q_base + ks * 4096), desc_at(t_k, kb + ks * 4096),
                        idesc_mxf4(128, 128, sid), (tmem + C::T_QSF) | (sid << 30),
                        (tmem + C::T_KSF1 + 8 * st) | (sid << 30), ks > 0);
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < D / 64; ++ks)
            tmem_cp_32x128_x4(tmem + C::T_KSF1 + 8 * st + 4 * ks, desc_at(t_sf, kb + TILE * D / 2 + ks * 512));
#pragma unroll
          for (int ks = 0; ks < D / 64; ++ks)
            mma_nvf4_ss(tmem + 128 * b, desc_at(t_k, q_base + ks * 4096), desc_at(t_k, kb + ks * 4096), id_s,
                        tmem + C::T_QSF + 4 * ks, tmem + C::T_KSF1 + 8 * st + 4 * ks, ks > 0);
        }
        tc_commit(&bars[C::B_S_FULL + b]);
        tc_commit(&bars[C::B_K1_EMPTY + st]);
      }
      __syncwarp();
      ++i1;
    };
    for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
      const int nt = work_item(p, w, q_tiles, k_tiles).nt;
      mbar_wait(&bars[C::B_Q_FULL], k & 1);
      tc_fence_after();
      if (!PLAIN && elect_one()) {
        for (int ks = 0; ks < (MX ? 1 : D / 64); ++ks)
          tmem_cp_32x128_x4(tmem + C::T_QSF + 4 * ks, desc_at(t_sf, s0 + C::Q_SF + ks * 512));
      }
      __syncwarp();
      // pass 1: S tiles round-robin over NB1 buffers; buffers 1 and 2 alias
      // the O (/O') columns, so they wait for the previous item's epilogue
      for (int jj = 0; jj < nt; ++jj) {
        if (jj == 1 && k > 0) mbar_wait(&bars[C::B_O_EMPTY], (k - 1) & 1);
        issue_s1(jj % C::NB1);
      }
      if (nt == 1 && k > 0) mbar_wait(&bars[C::B_O_EMPTY], (k - 1) & 1);
      // pass 2: S tiles run up to NB2 ahead of the PV MMAs (S(ns) reuses the
      // buffer of S(ns - NB2), released as soon as the softmax warps loaded it)
      const int it2 = it;
      for (int ns = 0, np = 0; np < nt;) {
        if (ns < nt && ns <= np + C::NB2) {
          issue_s1(ns % C::NB2);
          if (ns == nt - 1 && elect_one()) tc_commit(&bars[C::B_Q_EMPTY]);  // last read of Q
          __syncwarp();
          ++ns;
          continue;
        }
        const int pj = np++;
        const int pb = pc % C::NP;
        const int st = (it2 + pj) % C::NS;
        mbar_wait(&bars[C::B_KV_FULL + st], ((it2 + pj) / C::NS) & 1);  // V^T (+ V^F) of this tile landed
        mbar_wait(&bars[C::B_P_FULL + pb], (pc / C::NP) & 1);
        ++pc;
        tc_fence_after();
        const uint32_t sb = s0 + C::STAGE0 + st * C::STAGE_BYTES;
        const uint32_t pbase = s0 + C::P0 + pb * C::P_BYTES;
        if (elect_one()) {
          if constexpr (MX) {
            tmem_cp_32x128_x4(tmem + C::T_PSF + 8 * pb, desc_at(t_sf, pbase + C::PB_SF));
            tmem_cp_32x128_x4(tmem + C::T_VSF + 8 * st, desc_at(t_sf, sb + C::ST_VSF));
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t sid = 2u * ks;
              mma_mxf4_ss(tmem + C::T_O, desc_at(t_k, pbase + C::PB_CODES + ks * 4096),
                          desc_at(t_v, sb + C::ST_V + ks * 2 * (D * 16)), idesc_mxf4(128, D, sid),
                          (tmem + C::T_PSF + 8 * pb) | (sid << 30), (tmem + C::T_VSF + 8 * st) | (sid << 30),
                          (pj > 0 || ks > 0));
            }
          } else if (!(SAGE && TRAIN) && !PLAIN) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              tmem_cp_32x128_x4(tmem + C::T_PSF + 8 * pb + 4 * ks, desc_at(t_sf, pbase + C::PB_SF + ks * 512));
              tmem_cp_32x128_x4(tmem + C::T_VSF + 8 * st + 4 * ks, desc_at(t_sf, sb + C::ST_VSF + ks * 512));
            }
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
              mma_nvf4_ss(tmem + C::T_O, desc_at(t_k, pbase + C::PB_CODES + ks * 4096),
                          desc_at(t_v, sb + C::ST_V + ks * 2 * (D * 16)), id_pv, tmem + C::T_PSF + 8 * pb + 4 * ks,
                          tmem + C::T_VSF + 8 * st + 4 * ks, (pj > 0 || ks > 0));
          }
          if (TRAIN) {
#pragma unroll
            for (int ks = 0; ks < TILE / 16; ++ks)
              mma_f16_ss(tmem + C::T_OP, desc_at(t_ph, pbase + C::PB_H + ks * 4096),
                         desc_at(t_vh, sb + C::ST_VH + ks * 256), id_op, (pj > 0 || ks > 0));
          }
          tc_commit(&bars[C::B_P_EMPTY + pb]);
          tc_commit(&bars[C::B_KV_EMPTY + st]);
        }
        __syncwarp();
      }
      it = it2 + nt;
      if (elect_one()) tc_commit(&bars[C::B_O_FULL]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    constexpr int CW = C::CW;
    const int row = 32 * (warp & 3) + lane;        // TMEM lane == query row in the tile
    const int half = warp >> 2;                    // which column split
    const int cbase = half * CW;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const float sl2 = p.scale_log2;  // log2(e) / sqrt(d)
    const bool prof = (p.debug & 32) != 0;
    float x[CW];
    SUses su;
    int pc = 0, k = 0;
    AQ_PROF(long long prof_wait = 0, prof_ld = 0, prof_p1 = 0, prof_p2m = 0, prof_pw = 0, prof_q = 0, prof_f = 0;)
    AQ_PROF(long long p1_wait = 0, p1_ld = 0, tiles = 0, prof_merge = 0, prof_ofull = 0, prof_epi = 0, prof_top = 0, prof_top2 = 0;)
    AQ_PROF(long long t_item = clock64();)
    AQ_PROF(const long long prof_start = clock64();)

#define AQ_ACQUIRE_S(b_)                                                      \
  do {                                                                        \
    const int b__ = (b_);                                                     \
    const int u__ = su.take(b__);                                             \
    AQ_PROF(const long long t0__ = clock64();)                                \
    mbar_wait(&bars[C::B_S_FULL + b__], u__ & 1);                             \
    tc_fence_after();                                                         \
    AQ_PROF(const long long t1__ = clock64();)                                \
    const uint32_t base__ = t_lane + 128 * b__ + cbase;                       \
    _Pragma("unroll") for (int c0 = 0; c0 < CW; c0 += 32) tmem_ld32f(base__ + c0, x + c0); \
    tmem_ld_wait();                                                           \
    tc_fence_before();                                                        \
    mbar_arrive(&bars[C::B_S_EMPTY + b__]);                                   \
    AQ_PROF(prof_wait += t1__ - t0__; prof_ld += clock64() - t1__;)           \
  } while (0)

    for (int64_t w = next_item(k); w >= 0; w = next_item(++k)) {
      AQ_PROF(prof_top += clock64() - t_item;)
      const Item item = work_item(p, w, q_tiles, k_tiles);
      const int nt = item.nt;
      const int64_t head = item.head;
      const int64_t grow = static_cast<int64_t>(item.qt) * TILE + row;
      int64_t kmax = p.n_k - 1;  // last visible key of this row (inclusive)
      if (p.causal) kmax = min(kmax, grow + (p.n_k - p.n_q));
      AQ_PROF(tiles += nt;)
      // sage3 score terms of this row: S = (main + delta[key]) + bias (sage3.py:158-172).
      // The delta row(s) of a warp's 32 rows (one, or two when b_q = 16) are
      // staged through a warp-private double buffer in shared memory, loaded
      // one S tile ahead (lane l: float4 l%16 of row l/16), so the global
      // load latency hides behind the S wait; b_q < 16 reads global memory.
      const float* dl_row = nullptr;
      float brow = 0.f;
      bool dl_fast = false, dl_lane = false;
      int dl_r = 0;
      const float* dl_src = nullptr;
      float* dl_s = reinterpret_cast<float*>(smem + C::DL) + warp * 256;
      float4 dl_next = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (SAGE) {
        const int64_t gr = grow < p.n_q ? grow : p.n_q - 1;
        const int64_t tq = p.n_q / p.sage_bq;
        if (p.sage_delta) {
          dl_row = p.sage_delta + (head * tq + gr / p.sage_bq) * p.sage_kpad + cbase;
          if (p.sage_bq >= 16) {
            dl_fast = true;
            int64_t w0 = static_cast<int64_t>(item.qt) * TILE + 32 * (warp & 3);
            w0 = (w0 < p.n_q ? w0 : p.n_q - 1) / p.sage_bq;
            dl_r = static_cast<int>(gr / p.sage_bq - w0);
            const int64_t src_row = w0 + (lane >> 4);
            dl_lane = src_row < tq && src_row * p.sage_bq < static_cast<int64_t>(item.qt) * TILE + 32 * (warp & 3) + 32;
            dl_src = p.sage_delta + (head * tq + (dl_lane ? src_row : w0)) * p.sage_kpad + cbase + (lane & 15) * 4;
          }
        }
        if (p.sage_bias) brow = p.sage_bias[head * p.n_q + gr];
      }
      auto dl_fetch = [&](int jj) {
        return dl_lane ? __ldg(reinterpret_cast<const float4*>(dl_src + static_cast<int64_t>(jj) * TILE))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      auto sage_pre = [&](int jj) {
        if constexpr (SAGE) {
          if (dl_fast) {
            if (jj == 0) {
              __syncwarp();
              reinterpret_cast<float4*>(dl_s)[lane] = dl_fetch(0);
              __syncwarp();
            }
            if (jj + 1 < nt) dl_next = dl_fetch(jj + 1);
          }
        }
      };
      auto sage_post = [&](int jj) {
        if constexpr (SAGE) {
          if (dl_fast && jj + 1 < nt) {
            reinterpret_cast<float4*>(dl_s + ((jj + 1) & 1) * 128)[lane] = dl_next;
            __syncwarp();
          }
        }
      };
      // The row-constant bias cancels in P = exp(S - L): the passes run on
      // main + delta and only the stored L gains bias / sqrt(d).
      auto sage_add = [&](int jj) {
        if constexpr (SAGE) {
          if (dl_row) {
            const float4* d4 = dl_fast ? reinterpret_cast<const float4*>(dl_s + (jj & 1) * 128 + dl_r * 64)
                                       : reinterpret_cast<const float4*>(dl_row + static_cast<int64_t>(jj) * TILE);
#pragma unroll
            for (int c = 0; c < CW; c += 4) {
              const float4 dv = d4[c / 4];
              const float2 a = __fadd2_rn(make_float2(x[c], x[c + 1]), make_float2(dv.x, dv.y));
              const float2 b = __fadd2_rn(make_float2(x[c + 2], x[c + 3]), make_float2(dv.z, dv.w));
              x[c] = a.x;
              x[c + 1] = a.y;
              x[c + 2] = b.x;
              x[c + 3] = b.y;
            }
          }
        }
      };
      float mtrue = -INFINITY;  // exact row max of S (two-level P over the whole row)

      // pass 1 -- online softmax statistics over this thread's columns (log2
      // domain). The exponentials use a reference max m that is only raised
      // when a tile's max exceeds it by more than 2^8 (terms stay <= 256), so
      // they do not wait for the tile's max reduction; a raise recomputes.
      float m = -INFINITY, l = 0.f;
      for (int jj = 0; jj < nt; ++jj) {
        sage_pre(jj);
        AQ_ACQUIRE_S(jj % C::NB1);
        AQ_PROF(const long long tp1 = clock64();)
        sage_add(jj);
        const int64_t lim = kmax - (static_cast<int64_t>(jj) * TILE + cbase);  // visible: c <= lim
        if (lim < CW - 1) {
#pragma unroll
          for (int c = 0; c < CW; ++c) x[c] = (c <= lim) ? x[c] : -INFINITY;
        }
        if constexpr (SAGE && TRAIN) {
          if (p.sage_seg == 0) {
#pragma unroll
            for (int c = 0; c < CW; ++c) mtrue = fmaxf(mtrue, x[c]);
          } else if (p.sage_seg < 0 && grow < p.n_q) {
            // segments of b_k keys that need not align with the 128-key tiles:
            // per 16-key block max, merged per segment, atomically into HBM
            const int64_t nseg = p.n_k / p.sage_bk;
            unsigned* sm_row = p.sage_segmax + (head * p.n_q + grow) * nseg;
            const int64_t k0 = static_cast<int64_t>(jj) * TILE + cbase;
            float run = -INFINITY;
            int64_t run_s = -1;
#pragma unroll
            for (int b = 0; b < CW / 16; ++b) {
              float v = x[16 * b];
#pragma unroll
              for (int e = 1; e < 16; ++e) v = fmaxf(v, x[16 * b + e]);
              const int64_t s = (k0 + 16 * b) / p.sage_bk;
              if (s != run_s) {
                if (run_s >= 0 && run_s < nseg && run > -INFINITY) atomicMax(sm_row + run_s, f2ord(run));
                run_s = s;
                run = v;
              } else {
                run = fmaxf(run, v);
              }
            }
            if (run_s >= 0 && run_s < nseg && run > -INFINITY) atomicMax(sm_row + run_s, f2ord(run));
          }
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
        // A rebase needs a term above 2^8, hence sum > 240 (or inf): only then (and
        // while no column is visible yet) is the tile max needed. Same m sequence,
        // hence the same bits, as taking the max of every tile.
        if (!(sum <= 240.0f) || m == -INFINITY) {
          // row max on the raw scores (the scale is positive)
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
        sage_post(jj);
        AQ_PROF(prof_p1 += clock64() - tp1;)
      }
      AQ_PROF(p1_wait = prof_wait; p1_ld = prof_ld; const long long t_m0 = clock64();)
      // merge the CS column-split partials of each row
      float* ml = reinterpret_cast<float*>(smem + C::ML);
      ml[(half * 2 + 0) * TILE + row] = m;
      ml[(half * 2 + 1) * TILE + row] = l;
      if constexpr (SAGE) ml[(2 * CS + half) * TILE + row] = mtrue;
      named_bar_sync(1, 32 * C::NSW);
      float mt = -INFINITY;
#pragma unroll
      for (int h = 0; h < CS; ++h) mt = fmaxf(mt, ml[(h * 2) * TILE + row]);
      float lt = 0.f;
#pragma unroll
      for (int h = 0; h < CS; ++h) lt += ml[(h * 2 + 1) * TILE + row] * ex2(ml[(h * 2) * TILE + row] - mt);
      if constexpr (SAGE) {
#pragma unroll
        for (int h = 0; h < CS; ++h) mtrue = fmaxf(mtrue, ml[(2 * CS + h) * TILE + row]);
      }
      named_bar_sync(1, 32 * C::NSW);  // the partials buffer is reused by the next item
      // natural-log L is what the reference stores (flash.py:217); pass 2 uses
      // L2 = L * log2(e) recomputed from the stored value so the backward, which
      // only sees L, rebuilds bit-identical P (and P^F).
      const float L_nat = (mt + __log2f(lt)) * 0.69314718055994530942f;
      if (half == 0 && grow < p.n_q)
        p.lse[head * p.n_q + grow] = SAGE ? L_nat + brow * (sl2 * 0.69314718055994530942f) : L_nat;
      const float L2 = L_nat * 1.44269504088896340736f;
      const float l_scale = lt;  // P^ = exp(S - m) = P * l

      AQ_PROF(prof_merge += clock64() - t_m0;)
      // pass 2 -- P, P^F (NVFP4 over 16-key blocks), P^ for O'
      for (int jj = 0; jj < nt; ++jj) {
        sage_pre(jj);
        AQ_ACQUIRE_S(jj % C::NB2);
        AQ_PROF(const long long tm0 = clock64();)
        sage_add(jj);
        const int64_t lim = kmax - (static_cast<int64_t>(jj) * TILE + cbase);
        p_from_s<CW / 2>(x, cbase, sl2, L2);
        if (lim < CW - 1) {
#pragma unroll
          for (int c = 0; c < CW; ++c) x[c] = (c <= lim) ? x[c] : 0.f;
        }
        // two-level P (sage3.py:98-110, 186-190): per 16-key block its max
        // bm, the factor r = 448*6 / (max of its segment) and l / r for the f16
        // accumulation of dequant(P^F) * l / r
        float bm[CW / 16], rr[CW / 16], fr[CW / 16];
        if constexpr (SAGE && TRAIN) {
#pragma unroll
          for (int b = 0; b < CW / 16; ++b) {
            float v0 = fmaxf(x[16 * b], x[16 * b + 1]), v1 = fmaxf(x[16 * b + 2], x[16 * b + 3]);
#pragma unroll
            for (int e = 4; e < 16; e += 2) {
              v0 = fmaxf(v0, x[16 * b + e]);
              v1 = fmaxf(v1, x[16 * b + e + 1]);
            }
            bm[b] = fmaxf(v0, v1);
          }
          float sm[CW / 16];
          const int seg = p.sage_seg;
#pragma unroll
          for (int b = 0; b < CW / 16; ++b) sm[b] = bm[b];
          if (seg == 0) {  // the whole row: max P = exp(max S - L)
            const float v = ex2(fmaf(mtrue, sl2, -L2));
#pragma unroll
            for (int b = 0; b < CW / 16; ++b) sm[b] = v;
          } else if (seg < 0) {  // segment maxima of S from pass 1 (ordered after the merge barrier)
            const int64_t nseg = p.n_k / p.sage_bk;
            const int64_t gr = grow < p.n_q ? grow : p.n_q - 1;
            const unsigned* sm_row = p.sage_segmax + (head * p.n_q + gr) * nseg;
            const int64_t k0 = static_cast<int64_t>(jj) * TILE + cbase;
#pragma unroll
            for (int b = 0; b < CW / 16; ++b) {
              const int64_t s = (k0 + 16 * b) / p.sage_bk;
              const unsigned u = s < nseg ? __ldcg(sm_row + s) : 0u;
              sm[b] = u ? ex2(fmaf(ord2f(u), sl2, -L2)) : 0.f;
            }
          } else if (seg == 32) {
            sm[0] = sm[1] = fmaxf(bm[0], bm[1]);
            sm[2] = sm[3] = fmaxf(bm[2], bm[3]);
          } else if (seg >= 64) {
            float v = fmaxf(fmaxf(bm[0], bm[1]), fmaxf(bm[2], bm[3]));
            if (seg == 128) {  // the other column split holds the other 64 keys
              float* pm = reinterpret_cast<float*>(smem + C::ML) + (jj & 1) * (CS * TILE);
              pm[half * TILE + row] = v;
              named_bar_sync(2, 32 * C::NSW);
              v = fmaxf(pm[row], pm[TILE + row]);
            }
#pragma unroll
            for (int b = 0; b < CW / 16; ++b) sm[b] = v;
          }
#pragma unroll
          for (int b = 0; b < CW / 16; ++b) {
            const bool pos = sm[b] > 0.f;
            rr[b] = pos ? 2688.0f * rcp_approx(sm[b]) : 1.0f;
            fr[b] = pos ? l_scale * sm[b] * (1.0f / 2688.0f) : l_scale;
          }
        }
        const int pb = pc % C::NP;
        AQ_PROF(const long long tm1 = clock64();)
        if (pc >= C::NP) mbar_wait(&bars[C::B_P_EMPTY + pb], ((pc / C::NP) - 1) & 1);
        ++pc;
        AQ_PROF(const long long tm2 = clock64();)
        uint8_t* pcodes = smem + C::P0 + pb * C::P_BYTES + C::PB_CODES;
        uint8_t* psf = smem + C::P0 + pb * C::P_BYTES + C::PB_SF;
        uint32_t scw[(CW + 63) / 64];
#pragma unroll
        for (int s = 0; s < (CW + 63) / 64; ++s) scw[s] = 0;
        if constexpr (MX) {  // 32-key UE8M0 blocks: codes + one scale byte each
          uint32_t scs = 0;
#pragma unroll
          for (int b = 0; b < CW / 32; ++b) {
            uint32_t cd[4], sc;
            quantize_p32_mx(x + 32 * b, cd, sc);
            *reinterpret_cast<uint4*>(pcodes + t8x32_off(row, cbase + 32 * b, TILE)) = make_uint4(cd[0], cd[1], cd[2], cd[3]);
            scs |= sc << (8 * b);
          }
          *reinterpret_cast<uint16_t*>(psf + sf512_off(row, cbase / 32)) = static_cast<uint16_t>(scs);
        }
#pragma unroll
        for (int blk = 0; blk < ((PLAIN || MX) ? 0 : CW / 16); blk += 2) {
          const PBlock qa = (SAGE && TRAIN) ? quantize_p16_r(x + blk * 16, bm[blk], rr[blk])
                                            : quantize_p16_s(x + blk * 16, p.p_r);
          const PBlock qb = (SAGE && TRAIN) ? quantize_p16_r(x + blk * 16 + 16, bm[blk + 1], rr[blk + 1])
                                            : quantize_p16_s(x + blk * 16 + 16, p.p_r);
          *reinterpret_cast<uint4*>(pcodes + t8x32_off(row, cbase + blk * 16, TILE)) =
              make_uint4(qa.codes[0], qa.codes[1], qb.codes[0], qb.codes[1]);
          scw[blk / 4] |= (qa.scale << (8 * (blk & 3))) | (qb.scale << (8 * ((blk + 1) & 3)));
          if constexpr (SAGE && TRAIN) {  // f16 dequant(P^F) * l / r for the accumulating MMA
            uint8_t* ph = smem + C::P0 + pb * C::P_BYTES + C::PB_H;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const PBlock& q = t ? qb : qa;
              const __half2 f2 = __float2half2_rn(q.sv * fr[blk + t]);
#pragma unroll
              for (int h8 = 0; h8 < 2; ++h8) {
                __half2 hh[4];
                e2m1x8_to_h2(q.codes[h8], hh);
                uint32_t h[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const __half2 o2 = __hmul2(hh[e], f2);
                  h[e] = *reinterpret_cast<const uint32_t*>(&o2);
                }
                *reinterpret_cast<uint4*>(ph + t8x8_off(row, cbase + blk * 16 + 16 * t + 8 * h8)) =
                    make_uint4(h[0], h[1], h[2], h[3]);
              }
            }
          }
        }
        if (PLAIN || MX) {
        } else if (CW >= 64) {
#pragma unroll
          for (int s = 0; s < CW / 64; ++s)
            *reinterpret_cast<uint32_t*>(psf + sf512_off(row, cbase / 16 + 4 * s)) = scw[s];
        } else {
          *reinterpret_cast<uint16_t*>(psf + sf512_off(row, cbase / 16)) = static_cast<uint16_t>(scw[0]);
        }
        if (TRAIN && !SAGE) {
          const bool bf = PLAIN && p.plain_fmt == 1;  // PLAIN with bf16 operands: P^ in bf16
          uint8_t* ph = smem + C::P0 + pb * C::P_BYTES + C::PB_H;
#pragma unroll
          for (int c8 = 0; c8 < CW / 8; ++c8) {
            uint32_t h[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 ph2 = __fmul2_rn(make_float2(x[c8 * 8 + 2 * e], x[c8 * 8 + 2 * e + 1]),
                                            make_float2(l_scale, l_scale));
              if (bf) {
                const __nv_bfloat162 v = __floats2bfloat162_rn(ph2.x, ph2.y);
                h[e] = *reinterpret_cast<const uint32_t*>(&v);
              } else {
                const __half2 v = __floats2half2_rn(ph2.x, ph2.y);
                h[e] = *reinterpret_cast<const uint32_t*>(&v);
              }
            }
            *reinterpret_cast<uint4*>(ph + t8x8_off(row, cbase + c8 * 8)) = make_uint4(h[0], h[1], h[2], h[3]);
          }
        }
        if (!PLAIN && !MX && p.pf_codes != nullptr && grow < p.n_q) {  // instrument: this row's P^F of the tile
          const int64_t n16 = ceil_div(p.n_k, 16);
          const int64_t c0 = static_cast<int64_t>(jj) * TILE + cbase;
          uint8_t* dc = p.pf_codes + (head * p.n_q + grow) * (n16 * 8);
          uint8_t* dsc = p.pf_scales + (head * p.n_q + grow) * n16;
#pragma unroll
          for (int b = 0; b < CW / 16; ++b) {
            const int64_t blk = c0 / 16 + b;
            if (blk < n16) {
              *reinterpret_cast<uint2*>(dc + blk * 8) =
                  *reinterpret_cast<const uint2*>(pcodes + t8x32_off(row, cbase + 16 * b, TILE));
              dsc[blk] = psf[sf512_off(row, cbase / 16 + b)];
            }
          }
        }
        AQ_PROF(const long long tm3 = clock64();)
        fence_async_smem();
        mbar_arrive(&bars[C::B_P_FULL + pb]);
        sage_post(jj);
        AQ_PROF(const long long tm4 = clock64(); prof_p2m += tm1 - tm0; prof_pw += tm2 - tm1;)
        AQ_PROF(prof_q += tm3 - tm2; prof_f += tm4 - tm3;)
      }

      // epilogue: this thread's D/CS columns of O (and O' * 1/l) -> registers,
      // release the O columns, then store
      AQ_PROF(const long long t_e0 = clock64();)
      mbar_wait(&bars[C::B_O_FULL], k & 1);
      tc_fence_after();
      AQ_PROF(const long long t_e1 = clock64(); prof_ofull += t_e1 - t_e0;)
      const float inv_l = 1.f / l_scale;
      constexpr int DW = D / CS;             // output columns of this thread
      float o[TRAIN ? 2 : 1][DW];
#pragma unroll
      for (int out = 0; out < (TRAIN ? 2 : 1); ++out) {
#pragma unroll
        for (int c = 0; c < DW; c += (DW < 32 ? DW : 32)) {
          if (DW >= 32) {
            tmem_ld32f(t_lane + (out ? C::T_OP : C::T_O) + half * DW + c, o[out] + c);
          } else {
            uint32_t r[16];
            tmem_ld16(t_lane + (out ? C::T_OP : C::T_O) + half * DW + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[out][c + e] = __uint_as_float(r[e]);
          }
        }
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars[C::B_O_EMPTY]);
      AQ_PROF(const long long t_e2 = clock64(); prof_top2 += t_e2 - t_e1;)
      // stores (rowstore.cuh): in training the P buffers are idle here
      // (O_FULL: every PV MMA has read them; the next writes are the next
      // item's pass 2 by these same warps, after the next merge barrier), so
      // each warp stages its 32 rows there and writes whole row segments
      constexpr bool STAGE_OUT = TRAIN && C::NSW * 32 * DW * 4 <= C::NP * C::P_BYTES;
      const int64_t row0 = static_cast<int64_t>(item.qt) * TILE + 32 * (warp & 3);
#pragma unroll
      for (int out = 0; out < (TRAIN ? 2 : 1); ++out) {
        void* dst = out ? p.o_hp : p.o;
        if (dst == nullptr) continue;
        const int dt = out ? p.o_hp_dt : p.o_dt;
        const float mul = out ? inv_l * p.ohp_mul : p.o_mul;  // per-tensor scales (1 = reference)
        const int es = dt == 0 ? 4 : 2;
        if constexpr (STAGE_OUT) {
          warp_store_rows<DW>(smem + C::P0 + warp * 32 * DW * 4, lane, o[out], mul, dt,
                              reinterpret_cast<uint8_t*>(dst) + ((head * p.n_q + row0) * D + half * DW) * es,
                              static_cast<int64_t>(D) * es, static_cast<int>(p.n_q - row0 < 32 ? p.n_q - row0 : 32));
        } else if (grow < p.n_q) {
          store_row<DW>(reinterpret_cast<uint8_t*>(dst) + ((head * p.n_q + grow) * D + half * DW) * es, o[out], mul, dt);
        }
      }
      AQ_PROF(prof_epi += clock64() - t_e1; t_item = clock64();)
    }
#undef AQ_ACQUIRE_S
#ifdef AQ_FWD_PROFILE
    if (prof && lane == 0) {
      atomicAdd(&g_prof[0], static_cast<unsigned long long>(p1_wait));
      atomicAdd(&g_prof[1], static_cast<unsigned long long>(p1_ld));
      atomicAdd(&g_prof[2], static_cast<unsigned long long>(prof_p1));
      atomicAdd(&g_prof[4], static_cast<unsigned long long>(prof_ld - p1_ld));
      atomicAdd(&g_prof[5], static_cast<unsigned long long>(prof_p2m));
      atomicAdd(&g_prof[6], static_cast<unsigned long long>(prof_pw));
      atomicAdd(&g_prof[7], static_cast<unsigned long long>(prof_q));
      atomicAdd(&g_prof[8], static_cast<unsigned long long>(prof_f));
      atomicAdd(&g_prof[9], static_cast<unsigned long long>(clock64() - prof_start));
      atomicAdd(&g_prof[10], static_cast<unsigned long long>(tiles));
      atomicAdd(&g_prof[11], 1ull);
      atomicAdd(&g_prof[12], static_cast<unsigned long long>(prof_merge));
      atomicAdd(&g_prof[13], static_cast<unsigned long long>(prof_ofull));
      atomicAdd(&g_prof[14], static_cast<unsigned long long>(prof_epi));
      atomicAdd(&g_prof[15], static_cast<unsigned long long>(prof_top));
      atomicAdd(&g_prof[3], static_cast<unsigned long long>(prof_top2));
    }
#else
    (void)prof;
#endif
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool TRAIN, int CS, bool SAGE = false, bool PLAIN = false, bool MX = false>
cudaError_t launch(const FwdParams& p, cudaStream_t st) {
  using C = Cfg<D, TRAIN, CS, SAGE, PLAIN, MX>;
  auto kern = attn_fwd_kernel<D, TRAIN, CS, SAGE, PLAIN, MX>;
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

}  // namespace fwd

// Tuning-aid environment switches (read once): AQ_FWD_CS = 2 | 4 column
// splits of the training forward (default 2: 8 softmax warps, 64 key columns
// per thread);
// AQ_FWD_DEBUG bit 32 = per-segment cycle counters (aq_debug_fwd_profile),
// bit 64 = no exact pass-2 early-out in the inference kernel (A/B timing).
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
static int fwd_debug() {
  static const int d = env_int("AQ_FWD_DEBUG", 0);
  return d;
}
static int fwd_cs() {
  // default 2: the same column split (and (m, l) merge order) as the
  // inference kernel, so training and inference forwards agree bit for bit
  static const int cs = env_int("AQ_FWD_CS", 2) == 4 ? 4 : 2;
  return cs;
}

extern "C" int aq_debug_fwd_profile(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, fwd::g_prof, sizeof(fwd::g_prof)) != cudaSuccess) return 5;
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(fwd::g_prof, z, sizeof(z)) != cudaSuccess) return 5;
  }
  return 0;
}

cudaError_t launch_attn_fwd_mx(const FwdParams& p, cudaStream_t st) {
  // inference: the split-pass kernel; AQ_FWD_INFER=0 keeps it on K4 (comparisons)
  if (!p.train && env_int("AQ_FWD_INFER", 1)) return launch_attn_fwd_infer_mx(p, st);
  // training: the split-pass kernel K11's MX instance (AQ_FWD_QAT=0 keeps K4's),
  // on the same item order as the NVFP4 training forward
  if (p.train && env_int("AQ_FWD_QAT", 1)) {
    FwdParams q = p;
    if (!q.causal || !env_int("AQ_FWD_DYN", 1) || ceil_div(q.n_q, TILE) < env_int("AQ_FWDQ_DYN_MIN_QT", 8))
      q.item_ctr = nullptr;
    q.item_band = std::max(1, env_int("AQ_FWD_BAND", 8));
    return launch_attn_fwd_qat_mx(q, st);
  }
  FwdParams q = p;
  q.item_ctr = nullptr;  // K4's MX instance keeps its static order
  if (q.d == 64) return q.train ? fwd::launch<64, true, 2, false, false, true>(q, st)
                                : fwd::launch<64, false, 2, false, false, true>(q, st);
  if (q.d == 128) return q.train ? fwd::launch<128, true, 2, false, false, true>(q, st)
                                 : fwd::launch<128, false, 2, false, false, true>(q, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_attn_fwd_plain(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return fwd::launch<64, true, 2, false, true>(p, st);
  if (p.d == 128) return fwd::launch<128, true, 2, false, true>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_attn_fwd_sage(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return p.train ? fwd::launch<64, true, 2, true>(p, st) : fwd::launch<64, false, 2, true>(p, st);
  if (p.d == 128) return p.train ? fwd::launch<128, true, 2, true>(p, st) : fwd::launch<128, false, 2, true>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_attn_fwd(const FwdParams& p_in, cudaStream_t st) {
  FwdParams p = p_in;
  p.debug = fwd_debug();
  p.item_band = std::max(1, env_int("AQ_FWD_BAND", 8));
  const int64_t q_tiles = ceil_div(p.n_q, TILE);
  // inference: the split-pass kernel (attn_fwd_infer.cu); AQ_FWD_INFER=0 keeps
  // it on this kernel (tuning comparisons)
  if (!p.train && env_int("AQ_FWD_INFER", 1)) {
    // K5 keeps its static snake order: it reads no V^F and is not L2-bound; a
    // dynamic queue cost it 1 % at C2 and 4 % at C3 (ring reads, registers)
    // for 4 % at 32 K causal
    p.item_ctr = nullptr;
    return launch_attn_fwd_infer(p, st);
  }
  // training: the split-pass kernel K11 (attn_fwd_qat.cu; AQ_FWD_QAT=0 keeps
  // K4), on the dynamic banded item order for causal rows from 8 query tiles
  // (C4: 2.07 -> 1.78 ms against its static order, 1 K keys 1.43 -> 1.37, 2 K
  // 2.32 -> 2.07; K4 on its best order: 2.11 / 1.51 / 2.39 ms)
  if (p.train && fwd_cs() == 2 && env_int("AQ_FWD_QAT", 1)) {
    if (!p.causal || !env_int("AQ_FWD_DYN", 1) || q_tiles < env_int("AQ_FWDQ_DYN_MIN_QT", 8)) p.item_ctr = nullptr;
    return launch_attn_fwd_qat(p, st);
  }
  // the dynamic item queue serves long causal rows of the training kernel, where
  // the banded head-major order keeps K / V / V^F in L2 (8 K keys: 4.45 -> 3.89
  // ms, 16 K: 16.7 -> 14.7 ms at 64 K tokens x 32 heads); below 32 query tiles
  // the static longest-first order is as fast or faster (1 K keys: -6 % dynamic).
  // AQ_FWD_DYN=0: static order always; AQ_FWD_BAND: query tiles per band
  if (!p.causal || !p.train || !env_int("AQ_FWD_DYN", 1) || q_tiles < env_int("AQ_FWD_DYN_MIN_QT", 32))
    p.item_ctr = nullptr;
  if (fwd_cs() == 2) {
    if (p.d == 64) return p.train ? fwd::launch<64, true, 2>(p, st) : fwd::launch<64, false, 2>(p, st);
    if (p.d == 128) return p.train ? fwd::launch<128, true, 2>(p, st) : fwd::launch<128, false, 2>(p, st);
    return cudaErrorInvalidValue;
  }
  if (p.d == 64) return p.train ? fwd::launch<64, true, 4>(p, st) : fwd::launch<64, false, 4>(p, st);
  if (p.d == 128) return p.train ? fwd::launch<128, true, 4>(p, st) : fwd::launch<128, false, 4>(p, st);
  return cudaErrorInvalidValue;
}

}  // namespace aq
