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
// CTA = one (head, 128-query tile). Warps 0-3: softmax / quantize / epilogue,
// one thread per query row (TMEM lane). Warp 4: bulk-copy producer. Warp 5:
// single-thread tcgen05 MMA issuer. K/V tiles stream through an NS-stage
// mbarrier ring; operands arrive pre-laid-out by the quantizers (layouts.cuh).
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "pquant.cuh"
#include "ptx.cuh"

namespace aq {

namespace fwd {

constexpr int NS = 2;            // K/V pipeline stages
constexpr int NUM_THREADS = 192; // 4 softmax warps + producer + MMA

template <int D, bool TRAIN>
struct Smem {
  static constexpr int Q_CODES = 0;
  static constexpr int Q_SF = Q_CODES + TILE * D / 2;
  static constexpr int STAGE0 = Q_SF + (D / 64) * 512;
  // stage: K codes | K sf | V^T codes | V^T sf | V fp16 (train)
  static constexpr int ST_K = 0;
  static constexpr int ST_KSF = ST_K + TILE * D / 2;
  static constexpr int ST_V = ST_KSF + (D / 64) * 512;
  static constexpr int ST_VSF = ST_V + TILE * D / 2;
  static constexpr int ST_VH = ST_VSF + 1024;
  static constexpr int STAGE_BYTES = ST_VH + (TRAIN ? TILE * D * 2 : 0);
  static constexpr int P_CODES = STAGE0 + NS * STAGE_BYTES;
  static constexpr int P_SF = P_CODES + TILE * TILE / 2;
  static constexpr int P_H = P_SF + 1024;
  static constexpr int BARS = P_H + (TRAIN ? TILE * TILE * 2 : 0);
  static constexpr int NUM_BARS = 16;
  static constexpr int TMEM_SLOT = BARS + NUM_BARS * 8;
  static constexpr int USED = TMEM_SLOT + 16;
  // Force one CTA per SM: the kernel allocates all 512 TMEM columns.
  static constexpr int TOTAL = USED > 120 * 1024 ? USED : 120 * 1024;
  static constexpr int K_BYTES = TILE * D / 2 + (D / 64) * 512;
  static constexpr int V_BYTES = TILE * D / 2 + 1024 + (TRAIN ? TILE * D * 2 : 0);
};

// TMEM columns
constexpr uint32_t T_S0 = 0, T_S1 = 128, T_O = 128, T_OP = 256;
constexpr uint32_t T_QSF = 384, T_KSF = 392, T_PSF = 408, T_VSF = 416;

enum Bar { B_Q = 0, B_KV_FULL = 1, B_KV_EMPTY = 1 + NS, B_S_FULL = 1 + 2 * NS, B_S_EMPTY = 3 + 2 * NS,
           B_P_FULL = 5 + 2 * NS, B_P_EMPTY = 6 + 2 * NS, B_O_FULL = 7 + 2 * NS };

struct TileRange {
  int j_begin, j_end;  // key tiles [j_begin, j_end)
};

__device__ __forceinline__ TileRange key_tiles(const FwdParams& p, int q0) {
  const int last_row = min(q0 + TILE - 1, static_cast<int>(p.n_q) - 1);
  int j_end = static_cast<int>(ceil_div(p.n_k, TILE));
  if (p.causal) {
    const int64_t lim = static_cast<int64_t>(last_row) + (p.n_k - p.n_q);  // flash.py:127-128
    j_end = min(j_end, static_cast<int>(lim / TILE) + 1);
  }
  return {0, j_end};
}

template <int D, bool TRAIN>
__global__ void __launch_bounds__(NUM_THREADS, 1) attn_fwd_kernel(const FwdParams p) {
  using L = Smem<D, TRAIN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BARS);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::TMEM_SLOT);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int qt = blockIdx.x;
  const int64_t head = blockIdx.y;
  const int q0 = qt * TILE;
  const int q_tiles = static_cast<int>(ceil_div(p.n_q, TILE));
  const int k_tiles = static_cast<int>(ceil_div(p.n_k, TILE));
  const TileRange tr = key_tiles(p, q0);
  const int nt = tr.j_end - tr.j_begin;

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_Q], 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[B_KV_FULL + s], 1);
      mbar_init(&bars[B_KV_EMPTY + s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[B_S_FULL + b], 1);
      mbar_init(&bars[B_S_EMPTY + b], 128);
    }
    mbar_init(&bars[B_P_FULL], 128);
    mbar_init(&bars[B_P_EMPTY], 1);
    mbar_init(&bars[B_O_FULL], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const int64_t qtile_idx = head * q_tiles + qt;
      mbar_expect_tx(&bars[B_Q], TILE * D / 2 + (D / 64) * 512);
      bulk_g2s(smem + L::Q_CODES, p.q_codes + qtile_idx * fp4_tile_bytes(D), TILE * D / 2, &bars[B_Q]);
      bulk_g2s(smem + L::Q_SF, p.q_sf + qtile_idx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[B_Q]);
      int it = 0;
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = tr.j_begin; j < tr.j_end; ++j, ++it) {
          const int st = it % NS;
          if (it >= NS) mbar_wait(&bars[B_KV_EMPTY + st], ((it / NS) - 1) & 1);
          uint8_t* sb = smem + L::STAGE0 + st * L::STAGE_BYTES;
          const int64_t kt_idx = head * k_tiles + j;
          const uint32_t bytes = L::K_BYTES + (pass ? L::V_BYTES : 0);
          mbar_expect_tx(&bars[B_KV_FULL + st], bytes);
          bulk_g2s(sb + L::ST_K, p.k_codes + kt_idx * fp4_tile_bytes(D), TILE * D / 2, &bars[B_KV_FULL + st]);
          bulk_g2s(sb + L::ST_KSF, p.k_sf + kt_idx * sf_tile_bytes_qk(D), (D / 64) * 512, &bars[B_KV_FULL + st]);
          if (pass) {
            bulk_g2s(sb + L::ST_V, p.v_codes + kt_idx * fp4_tile_bytes(D), TILE * D / 2, &bars[B_KV_FULL + st]);
            bulk_g2s(sb + L::ST_VSF, p.v_sf + kt_idx * kSfTileBytesV, 1024, &bars[B_KV_FULL + st]);
            if (TRAIN)
              bulk_g2s(sb + L::ST_VH, p.v_h + kt_idx * h_tile_bytes(D), TILE * D * 2, &bars[B_KV_FULL + st]);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_s = idesc_nvf4(128, 128);
      const uint32_t id_pv = idesc_nvf4(128, D);
      const uint32_t id_op = idesc_f16(128, D, /*f16*/ 0, /*a_mn*/ 0, /*b_mn*/ 1);
      const uint32_t q_base = smem_u32(smem + L::Q_CODES);
      mbar_wait(&bars[B_Q], 0);
      tc_fence_after();
      for (int ks = 0; ks < D / 64; ++ks)
        tmem_cp_32x128_x4(tmem + T_QSF + 4 * ks, smem_desc(smem_u32(smem + L::Q_SF + ks * 512), 0, 128));
      int it = 0;
      int s_use0 = 0, s_use1 = 0;
      auto issue_s = [&](int st, uint32_t s_col) {
        const uint32_t kb = smem_u32(smem + L::STAGE0 + st * L::STAGE_BYTES + L::ST_K);
        const uint32_t ksf = smem_u32(smem + L::STAGE0 + st * L::STAGE_BYTES + L::ST_KSF);
        for (int ks = 0; ks < D / 64; ++ks)
          tmem_cp_32x128_x4(tmem + T_KSF + 8 * st + 4 * ks, smem_desc(ksf + ks * 512, 0, 128));
        for (int ks = 0; ks < D / 64; ++ks) {
          const uint64_t da = smem_desc(q_base + ks * 2 * 2048, 2048, 128);
          const uint64_t db = smem_desc(kb + ks * 2 * 2048, 2048, 128);
          mma_nvf4_ss(tmem + s_col, da, db, id_s, tmem + T_QSF + 4 * ks, tmem + T_KSF + 8 * st + 4 * ks, ks > 0);
        }
      };
      // pass 1: S tiles into alternating buffers
      for (int jj = 0; jj < nt; ++jj, ++it) {
        const int st = it % NS;
        const int b = jj & 1;
        mbar_wait(&bars[B_KV_FULL + st], (it / NS) & 1);
        const int use = b ? s_use1 : s_use0;
        if (use > 0) mbar_wait(&bars[B_S_EMPTY + b], (use - 1) & 1);
        tc_fence_after();
        issue_s(st, b ? T_S1 : T_S0);
        tc_commit(&bars[B_S_FULL + b]);
        tc_commit(&bars[B_KV_EMPTY + st]);
        if (b) ++s_use1; else ++s_use0;
      }
      // pass 2: S(jj) is issued ahead of PV(jj-1)
      const int it2 = it;
      for (int jj = 0; jj <= nt; ++jj) {
        if (jj < nt) {
          const int st = (it2 + jj) % NS;
          mbar_wait(&bars[B_KV_FULL + st], ((it2 + jj) / NS) & 1);
          if (s_use0 > 0) mbar_wait(&bars[B_S_EMPTY + 0], (s_use0 - 1) & 1);
          tc_fence_after();
          issue_s(st, T_S0);
          tc_commit(&bars[B_S_FULL + 0]);
          ++s_use0;
        }
        if (jj > 0) {
          const int pj = jj - 1;
          const int st = (it2 + pj) % NS;
          mbar_wait(&bars[B_P_FULL], pj & 1);
          tc_fence_after();
          const uint32_t sb = smem_u32(smem + L::STAGE0 + st * L::STAGE_BYTES);
          for (int ks = 0; ks < 2; ++ks) {
            tmem_cp_32x128_x4(tmem + T_PSF + 4 * ks, smem_desc(smem_u32(smem + L::P_SF + ks * 512), 0, 128));
            tmem_cp_32x128_x4(tmem + T_VSF + 8 * st + 4 * ks, smem_desc(sb + L::ST_VSF + ks * 512, 0, 128));
          }
          const uint32_t pa = smem_u32(smem + L::P_CODES);
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t da = smem_desc(pa + ks * 2 * 2048, 2048, 128);
            const uint64_t db = smem_desc(sb + L::ST_V + ks * 2 * (D * 16), D * 16, 128);
            mma_nvf4_ss(tmem + T_O, da, db, id_pv, tmem + T_PSF + 4 * ks, tmem + T_VSF + 8 * st + 4 * ks,
                        (pj > 0 || ks > 0));
          }
          if (TRAIN) {
            const uint32_t ph = smem_u32(smem + L::P_H);
            for (int ks = 0; ks < TILE / 16; ++ks) {
              const uint64_t da = smem_desc(ph + ks * 2 * 2048, 2048, 128);
              const uint64_t db = smem_desc(sb + L::ST_VH + ks * 2 * 128, 128, 2048);
              mma_f16_ss(tmem + T_OP, da, db, id_op, (pj > 0 || ks > 0));
            }
          }
          tc_commit(&bars[B_P_EMPTY]);
          tc_commit(&bars[B_KV_EMPTY + st]);
        }
      }
      tc_commit(&bars[B_O_FULL]);
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int row = threadIdx.x;  // 0..127 == TMEM lane
    const int64_t grow = q0 + row;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = p.scale_log2;  // log2(e) / sqrt(d)
    const int64_t offset = p.n_k - p.n_q;
    // last valid key for this row (inclusive), global index
    int64_t kmax = p.n_k - 1;
    if (p.causal) kmax = min(kmax, grow + offset);
    float m = -INFINITY, l = 0.f;
    int s_use0 = 0, s_use1 = 0;
    uint32_t s[TILE];

#define AQ_LOAD_S(col)                                              \
  do {                                                              \
    _Pragma("unroll") for (int c0 = 0; c0 < TILE; c0 += 32) {       \
      uint32_t r_[32];                                              \
      tmem_ld32(t_lane + (col) + c0, r_);                           \
      _Pragma("unroll") for (int e_ = 0; e_ < 32; ++e_) s[c0 + e_] = r_[e_]; \
    }                                                               \
    tmem_ld_wait();                                                 \
  } while (0)

    // pass 1 -- online softmax statistics (flash.py:145-173), log2 domain
    for (int jj = 0; jj < nt; ++jj) {
      const int b = jj & 1;
      mbar_wait(&bars[B_S_FULL + b], (b ? s_use1 : s_use0) & 1);
      tc_fence_after();
      AQ_LOAD_S(b ? T_S1 : T_S0);
      tc_fence_before();
      mbar_arrive(&bars[B_S_EMPTY + b]);
      if (b) ++s_use1; else ++s_use0;
      const int64_t k0 = static_cast<int64_t>(tr.j_begin + jj) * TILE;
      const int64_t lim = kmax - k0;  // keys c <= lim are visible
      float mloc = -INFINITY;
#pragma unroll
      for (int c = 0; c < TILE; ++c) {
        const float t = (c <= lim) ? __uint_as_float(s[c]) * sl2 : -INFINITY;
        s[c] = __float_as_uint(t);
        mloc = fmaxf(mloc, t);
      }
      const float m_new = fmaxf(m, mloc);
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < TILE; ++c) acc += ex2(__uint_as_float(s[c]) - m_new);
      l = l * ex2(m - m_new) + acc;
      m = m_new;
    }
    // natural-log L is what the reference stores (flash.py:217); pass 2 uses
    // L2 = L * log2(e) recomputed from the stored value so the backward, which
    // only sees L, rebuilds bit-identical P (and P^F).
    const float L_nat = (m + __log2f(l)) * 0.69314718055994530942f;
    if (grow < p.n_q) p.lse[head * p.n_q + grow] = L_nat;
    const float L2 = L_nat * 1.44269504088896340736f;
    const float l_scale = l;           // P^ = exp(S - m) = P * l

    // pass 2 -- P, P^F (NVFP4 over 16-key blocks), P^ for O'
    for (int jj = 0; jj < nt; ++jj) {
      mbar_wait(&bars[B_S_FULL + 0], s_use0 & 1);
      tc_fence_after();
      AQ_LOAD_S(T_S0);
      tc_fence_before();
      mbar_arrive(&bars[B_S_EMPTY + 0]);
      ++s_use0;
      const int64_t k0 = static_cast<int64_t>(tr.j_begin + jj) * TILE;
      const int64_t lim = kmax - k0;
#pragma unroll
      for (int c = 0; c < TILE; ++c) {
        const float t = (c <= lim) ? __uint_as_float(s[c]) * sl2 - L2 : -INFINITY;
        s[c] = __float_as_uint(ex2(t));
      }
      if (jj > 0) mbar_wait(&bars[B_P_EMPTY], (jj - 1) & 1);
      uint8_t* pc = smem + L::P_CODES;
      uint8_t* psf = smem + L::P_SF;
#pragma unroll
      for (int blk = 0; blk < TILE / 16; ++blk) {
        float pv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pv[e] = __uint_as_float(s[blk * 16 + e]);
        const PBlock q = quantize_p16(pv);
        *reinterpret_cast<uint2*>(pc + t8x32_off(row, blk * 16, TILE)) = make_uint2(q.codes[0], q.codes[1]);
        psf[sf512_off(row, blk)] = static_cast<uint8_t>(q.scale);
      }
      if (TRAIN) {
        uint8_t* ph = smem + L::P_H;
#pragma unroll
        for (int c8 = 0; c8 < TILE / 8; ++c8) {
          uint32_t h[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __half2 v = __floats2half2_rn(__uint_as_float(s[c8 * 8 + 2 * e]) * l_scale,
                                                __uint_as_float(s[c8 * 8 + 2 * e + 1]) * l_scale);
            h[e] = *reinterpret_cast<const uint32_t*>(&v);
          }
          *reinterpret_cast<uint4*>(ph + t8x8_off(row, c8 * 8)) = make_uint4(h[0], h[1], h[2], h[3]);
        }
      }
      fence_async_smem();
      mbar_arrive(&bars[B_P_FULL]);
    }

    // epilogue: O (and O' * 1/l) rows -> global
    mbar_wait(&bars[B_O_FULL], 0);
    tc_fence_after();
    const float inv_l = 1.f / l_scale;
    for (int out = 0; out < (TRAIN ? 2 : 1); ++out) {
      void* dst = out ? p.o_hp : p.o;
      const int dt = out ? p.o_hp_dt : p.o_dt;
      const float mul = out ? inv_l : 1.f;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t r[32];
        tmem_ld32(t_lane + (out ? T_OP : T_O) + c, r);
        tmem_ld_wait();
        if (dst != nullptr && grow < p.n_q) {
          const int64_t base = (head * p.n_q + grow) * D + c;
          if (dt == 0) {
            float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + base);
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              d4[e / 4] = make_float4(__uint_as_float(r[e]) * mul, __uint_as_float(r[e + 1]) * mul,
                                      __uint_as_float(r[e + 2]) * mul, __uint_as_float(r[e + 3]) * mul);
          } else {
            uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(dst) + base);
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint32_t h[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float a = __uint_as_float(r[e + 2 * k]) * mul, bb = __uint_as_float(r[e + 2 * k + 1]) * mul;
                if (dt == 1) {
                  const __nv_bfloat162 v = __floats2bfloat162_rn(a, bb);
                  h[k] = *reinterpret_cast<const uint32_t*>(&v);
                } else {
                  const __half2 v = __floats2half2_rn(a, bb);
                  h[k] = *reinterpret_cast<const uint32_t*>(&v);
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

template <int D, bool TRAIN>
cudaError_t launch(const FwdParams& p, cudaStream_t st) {
  using L = Smem<D, TRAIN>;
  auto kern = attn_fwd_kernel<D, TRAIN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(ceil_div(p.n_q, TILE)), static_cast<unsigned>(p.heads));
  kern<<<grid, NUM_THREADS, L::TOTAL, st>>>(p);
  return cudaGetLastError();
}

}  // namespace fwd

cudaError_t launch_attn_fwd(const FwdParams& p, cudaStream_t st) {
  if (p.d == 64) return p.train ? fwd::launch<64, true>(p, st) : fwd::launch<64, false>(p, st);
  if (p.d == 128) return p.train ? fwd::launch<128, true>(p, st) : fwd::launch<128, false>(p, st);
  return cudaErrorInvalidValue;
}

}  // namespace aq
