// K1 / K2 / K3: bit-exact NVFP4 block quantizers and the dequantizer.
//
// Semantics follow the reference codec (attnqat/codec.py):
//   scale code  = E4M3_RNE_sat448(amax / 6), bumped 0 -> 1 (2^-9) when the
//                 block is non-zero (codec.py:169-177)
//   element     = E2M1_RNE_sat6(x / decoded_scale) (codec.py:191-203),
//                 all-zero blocks store zero codes, an exact +-0.0 input
//                 stores nibble 0x0 while a small negative that rounds to
//                 zero keeps the sign nibble 0x8 (codec.py:84-87)
//   packing     = two codes per byte, lower index in the low nibble
//                 (codec.py:206-213)
// Bit-exactness needs IEEE division (div.rn.f32) for amax/6 and x/s, the
// hardware cvt.rn.satfinite.{e4m3x2,e2m1x2}.f32 converts, and no FTZ (this
// file is compiled without --use_fast_math).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"
#include "ptx.cuh"

namespace aq {

enum DType : int { kF32 = 0, kBF16 = 1, kF16 = 2 };

__device__ __forceinline__ float load_elem(const void* p, int64_t i, int dt) {
  if (dt == kBF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  if (dt == kF16) return __half2float(reinterpret_cast<const __half*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
}

// load 16 consecutive elements (16-byte aligned rows are the common case)
__device__ __forceinline__ void load16(const void* p, int64_t i0, int dt, float (&v)[16]) {
  const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(p) + i0;
  if (dt == kBF16 && ((reinterpret_cast<uintptr_t>(pb) & 15) == 0)) {
    const uint4* q = reinterpret_cast<const uint4*>(pb);
    uint4 a = q[0], b = q[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[2 * j] = __uint_as_float(w[j] << 16);
      v[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = load_elem(p, i0 + j, dt);
}

__device__ __forceinline__ void store_elem(void* p, int64_t i, int dt, float x) {
  if (dt == kBF16)
    reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(x);
  else if (dt == kF16)
    reinterpret_cast<__half*>(p)[i] = __float2half_rn(x);
  else
    reinterpret_cast<float*>(p)[i] = x;
}

__device__ __forceinline__ uint32_t h16_bits(float x, int dt) {
  return dt == kF16 ? static_cast<uint32_t>(__half_as_ushort(__float2half_rn(x)))
                    : static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(x)));
}

// Quantize one 16-element block: scale code, 16 packed codes, and (when
// WANT_FQ) the exact dequantized values as f16x2 (exact in fp16 and bf16).
struct Block16 {
  uint32_t scale;
  uint32_t packed[2];
  __half2 fq[8];
  bool finite;
};

template <bool WANT_FQ, bool CHECK_FINITE = true>
__device__ __forceinline__ void quantize_block16(const float (&v)[16], Block16& out) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = fmaxf(fabsf(v[2 * j]), fabsf(v[2 * j + 1]));
  const float amax = fmaxf(fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3])), fmaxf(fmaxf(a[4], a[5]), fmaxf(a[6], a[7])));
  // fmaxf drops NaN, so test finiteness separately: x * 0 is NaN for NaN / inf
  if (CHECK_FINITE) {
    float2 z = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 16; j += 2) z = __ffma2_rn(make_float2(v[j], v[j + 1]), make_float2(0.f, 0.f), z);
    out.finite = (z.x + z.y == 0.f);
  } else {
    out.finite = true;
  }
  const float raw = div_rn(amax, 6.0f, 0.16666667163372039795f);  // = fl(amax / 6)
  uint32_t sc = cvt_e4m3(raw);
  if (sc == 0 && amax > 0.f) sc = 1;  // tiny non-zero block keeps 2^-9 (codec.py:175-176)
  out.scale = sc;
  const float s = e4m3_to_f32(sc);
  const float r = s > 0.f ? __frcp_rn(s) : 0.f;
  // x / s correctly rounded (Markstein step, packed fp32x2); adding +0 maps
  // an exact -0.0 input (and every element of an all-zero block, r = 0) to
  // +0, which encodes as nibble 0x0 (codec.py:84, 199-201)
  const float2 r2 = make_float2(r, r), s2n = make_float2(-s, -s), zero2 = make_float2(0.f, 0.f);
  float q[16];
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 x = make_float2(v[j], v[j + 1]);
    const float2 q0 = __fmul2_rn(x, r2);
    const float2 rem = __ffma2_rn(q0, s2n, x);
    const float2 qq = __fadd2_rn(__ffma2_rn(rem, r2, q0), zero2);
    q[j] = qq.x;
    q[j + 1] = qq.y;
  }
  out.packed[0] = cvt_e2m1x8(q);
  out.packed[1] = cvt_e2m1x8(q + 8);
  if (WANT_FQ) {
    const __half sh = __float2half_rn(s);  // exact: E4M3 values are fp16 values
    const __half2 s2 = __halves2half2(sh, sh);
    __half2 c[4];
    e2m1x8_to_h2(out.packed[0], c);
#pragma unroll
    for (int i = 0; i < 4; ++i) out.fq[i] = __hmul2(c[i], s2);
    e2m1x8_to_h2(out.packed[1], c);
#pragma unroll
    for (int i = 0; i < 4; ++i) out.fq[4 + i] = __hmul2(c[i], s2);
  }
}

// Per-tensor FP32 scale t (two-level NVFP4): the block quantizer sees x / t,
// applied as x * (1 / t). t = 1 multiplies by 1.0 (exact), so the reference's
// bits are unchanged; the branch keeps that case free.
__device__ __forceinline__ void scale16(float (&v)[16], float inv_ts) {
  if (inv_ts != 1.f) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const float2 t = __fmul2_rn(make_float2(v[j], v[j + 1]), make_float2(inv_ts, inv_ts));
      v[j] = t.x;
      v[j + 1] = t.y;
    }
  }
}

__device__ __forceinline__ uint32_t h2_to(const __half2 h, int dt) {
  // f16 pair -> the same pair in dt (16-bit dtypes only); exact for fq values
  if (dt == kF16) return *reinterpret_cast<const uint32_t*>(&h);
  const float2 f = __half22float2(h);
  const __nv_bfloat162 b = __floats2bfloat162_rn(f.x, f.y);
  return *reinterpret_cast<const uint32_t*>(&b);
}

__device__ __forceinline__ void store_fq16(void* p, int64_t i0, int dt, const __half2 (&fq)[8], float ts = 1.f) {
  if (ts != 1.f) {  // two-level NVFP4: dequantized value = t * scale * code
    const __half* fh = reinterpret_cast<const __half*>(fq);
#pragma unroll
    for (int j = 0; j < 16; ++j) store_elem(p, i0 + j, dt, __half2float(fh[j]) * ts);
    return;
  }
  if (dt == kF32) {
    float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + i0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = __half22float2(fq[2 * i]), b = __half22float2(fq[2 * i + 1]);
      d[i] = make_float4(a.x, a.y, b.x, b.y);
    }
  } else {
    uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p) + i0);
    d[0] = make_uint4(h2_to(fq[0], dt), h2_to(fq[1], dt), h2_to(fq[2], dt), h2_to(fq[3], dt));
    d[1] = make_uint4(h2_to(fq[4], dt), h2_to(fq[5], dt), h2_to(fq[6], dt), h2_to(fq[7], dt));
  }
}

// ---------------------------------------------------------------------------
// K1: blocks along the contiguous (column) axis. x is [heads][n][cols] with
// row stride `ld` elements and head stride `hs` elements. One thread per 32
// columns (two blocks; cols % 32 == 16 leaves a final single block).
// Optional outputs (nullptr to skip):
//   codes_ref [heads*n][cols/2], scales_ref [heads*n][cols/16]  (reference layout)
//   fq        [heads*n][cols] dense dequantized values (dtype fq_dt)
//   codes_t   T8x32 tiles per head (n padded to 128; pad rows written as 0)
//   sf_t      SF512 images per tile
//   fqh_t     T8x8 16-bit tiles of the dequantized values (dtype fqh_dt)
// ---------------------------------------------------------------------------
// NPAIR > 0: compile-time block pairs per row (d = 64 / 128), so the per-thread
// index math is shifts and masks; 0 = runtime (any cols). Rows are contiguous
// across heads in the common case (n % 128 == 0, hs == n * ld): then no
// division by n is needed at all (64-bit division dominated the instruction
// count of the first version).
template <bool WANT_FQ, int NPAIR>
__global__ void __launch_bounds__(256) quantize_rows_kernel(RowsArgs a) {
  const int64_t nb = a.cols / 16;
  const int64_t npair = NPAIR > 0 ? NPAIR : (nb + 1) / 2;
  const int64_t n_pad = (a.codes_t || a.sf_t || a.fqh_t) ? ceil_div(a.n, TILE) * TILE : a.n;
  const int64_t total = a.heads * n_pad * npair;
  const int D = static_cast<int>(a.cols);
  const bool flat = n_pad == a.n && a.hs == a.n * a.ld;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bp = NPAIR > 0 ? (t & (NPAIR - 1)) : t % npair;
    const int64_t rowp = NPAIR > 0 ? (t / NPAIR) : t / npair;
    int64_t h, r;
    if (flat) {
      h = 0;
      r = rowp;          // row index over all heads; source offset rowp * ld
    } else {
      h = rowp / n_pad;
      r = rowp % n_pad;
    }
    const bool real = flat || r < a.n;
    const int64_t row = flat ? rowp : h * a.n + r;
    // n_pad is a multiple of TILE in tiled mode, so tiles of consecutive heads are consecutive
    const int64_t tile = rowp / TILE;
    const int rr = static_cast<int>(rowp % TILE);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t b = bp * 2 + half;
      if (b >= nb) break;
      float v[16];
      if (real) {
        load16(a.x, (flat ? rowp * a.ld : h * a.hs + r * a.ld) + b * 16, a.x_dt, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
      Block16 q;
      scale16(v, a.inv_ts);
      quantize_block16<WANT_FQ>(v, q);
      if (real) {
        if (!q.finite && a.nonfinite) atomicOr(a.nonfinite, 1);
        if (a.codes_ref)
          *reinterpret_cast<uint2*>(a.codes_ref + row * (a.cols / 2) + b * 8) = make_uint2(q.packed[0], q.packed[1]);
        if (a.scales_ref) a.scales_ref[row * nb + b] = static_cast<uint8_t>(q.scale);
        if (WANT_FQ && a.fq) store_fq16(a.fq, row * a.cols + b * 16, a.fq_dt, q.fq, a.ts);
      }
      if (a.codes_t)
        *reinterpret_cast<uint2*>(a.codes_t + tile * fp4_tile_bytes(D) + t8x32_off(rr, static_cast<int>(b) * 16, TILE)) =
            make_uint2(q.packed[0], q.packed[1]);
      if (a.sf_t)
        a.sf_t[tile * sf_tile_bytes_qk(D) + sf512_off(rr, static_cast<int>(b))] = static_cast<uint8_t>(q.scale);
      if (WANT_FQ && a.fqh_t) {
        uint8_t* base = reinterpret_cast<uint8_t*>(a.fqh_t) + tile * h_tile_bytes(D);
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8)
          *reinterpret_cast<uint4*>(base + t8x8_off(rr, static_cast<int>(b) * 16 + h8 * 8)) =
              make_uint4(h2_to(q.fq[4 * h8], a.fqh_dt), h2_to(q.fq[4 * h8 + 1], a.fqh_dt),
                         h2_to(q.fq[4 * h8 + 2], a.fqh_dt), h2_to(q.fq[4 * h8 + 3], a.fqh_dt));
      }
    }
  }
}

// K1 fast path: the attention staging case only -- bf16 rows, whole 128-row
// tiles (n % 128 == 0, contiguous heads), MMA tile outputs only. No per-block
// output-pointer branches, no reference-layout or fake-quant stores: one
// thread = 32 columns (two blocks) of one row, one 16-byte code store and one
// 2-byte scale store.
// n = rows per head; a ragged last tile (n % 128 != 0, e.g. C3's N = 32760) is
// zero-padded exactly as the general kernel pads it (zero blocks through the
// same quantizer, no non-finite check).
template <int D, bool FQH, bool F32 = false>
__global__ void __launch_bounds__(256) quantize_rows_tiled_kernel(const void* __restrict__ xv, int64_t heads,
                                                                  int64_t n, uint8_t* __restrict__ codes_t,
                                                                  uint8_t* __restrict__ sf_t,
                                                                  uint8_t* __restrict__ fqh_t, int fqh_dt,
                                                                  float inv_ts, int* __restrict__ nonfinite) {
  constexpr int NPAIR = D / 32;
  const int64_t n_pad = ceil_div(n, TILE) * TILE;
  const int64_t total = heads * n_pad * NPAIR;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int bp = static_cast<int>(t & (NPAIR - 1));
    const int64_t rowp = t / NPAIR;  // padded row over all heads (tiles of consecutive heads are consecutive)
    const int64_t tile = rowp / TILE;
    const int rr = static_cast<int>(rowp % TILE);
    int64_t row = rowp;              // source row
    bool real = true;
    if (n_pad != n) {
      const int64_t h = rowp / n_pad, r = rowp % n_pad;
      real = r < n;
      row = h * n + r;
    }
    Block16 q[2];
    if (!real) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
      quantize_block16<FQH, true>(v, q[0]);
      q[1] = q[0];
    } else if constexpr (F32) {  // fp32 input (the sage3 centred operands)
      const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(xv) + row * D + bp * 32);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 f = src[4 * h + j];
          v[4 * j] = f.x;
          v[4 * j + 1] = f.y;
          v[4 * j + 2] = f.z;
          v[4 * j + 3] = f.w;
        }
        scale16(v, inv_ts);
        quantize_block16<FQH, true>(v, q[h]);
      }
    } else {
      const uint4* src =
          reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(xv) + row * D + bp * 32);
      const uint4 w[4] = {src[0], src[1], src[2], src[3]};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t ww[8] = {w[2 * h].x, w[2 * h].y, w[2 * h].z, w[2 * h].w,
                                w[2 * h + 1].x, w[2 * h + 1].y, w[2 * h + 1].z, w[2 * h + 1].w};
        float v[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[2 * j] = __uint_as_float(ww[j] << 16);
          v[2 * j + 1] = __uint_as_float(ww[j] & 0xFFFF0000u);
        }
        scale16(v, inv_ts);
        quantize_block16<FQH, true>(v, q[h]);
      }
    }
    // NaN / Inf input (codec.py:313-314): flag it for the host to raise InvalidValue
    if (real && nonfinite != nullptr && !(q[0].finite && q[1].finite)) atomicOr(nonfinite, 1);
    if (FQH) {
      // the 16-bit fake-quantized operand tile the backward reuses (T8x8)
      uint8_t* base = fqh_t + tile * h_tile_bytes(D);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8)
          *reinterpret_cast<uint4*>(base + t8x8_off(rr, bp * 32 + h * 16 + h8 * 8)) =
              make_uint4(h2_to(q[h].fq[4 * h8], fqh_dt), h2_to(q[h].fq[4 * h8 + 1], fqh_dt),
                         h2_to(q[h].fq[4 * h8 + 2], fqh_dt), h2_to(q[h].fq[4 * h8 + 3], fqh_dt));
    }
    *reinterpret_cast<uint4*>(codes_t + tile * fp4_tile_bytes(D) + t8x32_off(rr, bp * 32, TILE)) =
        make_uint4(q[0].packed[0], q[0].packed[1], q[1].packed[0], q[1].packed[1]);
    *reinterpret_cast<uint16_t*>(sf_t + tile * sf_tile_bytes_qk(D) + sf512_off(rr, 2 * bp)) =
        static_cast<uint16_t>(q[0].scale | (q[1].scale << 8));
  }
}

// ---------------------------------------------------------------------------
// K2: blocks along the token axis (the V operand, quantized as V^T with the
// token tail zero-padded to a multiple of 16; codec.py:359-381). x is
// [heads][n][cols]. One CTA per (head, 32-token slab): the slab is staged in
// shared memory with coalesced loads, then thread c quantizes column c's two
// 16-token blocks and writes 16 contiguous code bytes.
// Optional outputs:
//   codes_ref [heads][cols][n16/2], scales_ref [heads][cols][n16/16]  (n16 = ceil16(n))
//   fq        [heads][n][cols] dense (fake_quantize_cols)
//   codes_t   T8x32 V^T tiles: per (head, 128-token tile) a cols x 128 tile
//   sf_t      SF512 images (2 K-steps per tile)
//   fqh_t     T8x8 16-bit tiles [128 tokens][cols] of the dequantized V
// ---------------------------------------------------------------------------
constexpr int kColsSlab = 64;   // tokens per CTA step (4 blocks of 16)
constexpr int kColsMax = 128;   // columns staged per pass

// K2 fast path: the attention staging case only -- bf16 V, whole 128-token
// tiles, contiguous heads, MMA tile outputs (V^T codes + scales) only. A CTA
// stages 64 tokens x D columns as bf16 in shared memory (16-byte loads); a
// thread then owns a column pair x 32 tokens: 32 four-byte shared loads give
// both columns' 32 values, four blocks are quantized, and each column's 32
// codes leave as one 16-byte store (plus one 2-byte scale store).
template <int D, bool FQH>
__global__ void __launch_bounds__(128) quantize_cols_tiled_kernel(const __nv_bfloat16* __restrict__ x, int64_t heads,
                                                                  int64_t n, uint8_t* __restrict__ codes_t,
                                                                  uint8_t* __restrict__ sf_t, uint8_t* __restrict__ fqh_t,
                                                                  int fqh_dt, uint8_t* __restrict__ fqh2_t,
                                                                  int fqh2_dt, float inv_ts, int* __restrict__ nonfinite) {
  constexpr int SLAB = 64, PITCH = D + 8;  // tokens per CTA step; padded row (16-bit elements)
  // the slab (64 contiguous token rows, 16 KB at D = 128) arrives by one 1-D bulk
  // copy, double-buffered so the next slab's load overlaps this slab's work (the
  // column-pair reads below touch one row per instruction: no padding needed)
  // (dynamic shared memory: with the f16 stage it exceeds the 48 KB static limit)
  extern __shared__ __align__(128) uint8_t qc_smem[];
  auto slab = reinterpret_cast<__nv_bfloat16(*)[SLAB][D]>(qc_smem);                        // [2][SLAB][D]
  auto bar = reinterpret_cast<uint64_t*>(qc_smem + 2 * SLAB * D * 2);                       // [2]
  // training: the dequantized values, as f16 pairs, for the T8x8 operand tiles
  auto slab_h = reinterpret_cast<__half(*)[PITCH]>(qc_smem + 2 * SLAB * D * 2 + 16);        // [SLAB][PITCH]
  constexpr uint32_t SLAB_BYTES = SLAB * D * 2;
  constexpr int CV = D / 8;  // 16-byte vectors per token row
  const int64_t tiles = n / TILE;
  const int64_t nslabs = heads * tiles * (TILE / SLAB);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    if (blockIdx.x < nslabs) {
      mbar_expect_tx(&bar[0], SLAB_BYTES);
      bulk_g2s(&slab[0][0][0], x + static_cast<int64_t>(blockIdx.x) * SLAB * D, SLAB_BYTES, &bar[0]);
    }
  }
  int it = 0;
  for (int64_t sidx = blockIdx.x; sidx < nslabs; sidx += gridDim.x, ++it) {
    const int64_t tok0 = sidx * SLAB;  // flat token index over all heads (tiles never straddle heads)
    const int buf = it & 1;
    __syncthreads();  // every thread is done with slab[buf ^ 1] (previous slab) and slab_h
    if (threadIdx.x == 0 && sidx + gridDim.x < nslabs) {
      fence_async_smem();
      mbar_expect_tx(&bar[buf ^ 1], SLAB_BYTES);
      bulk_g2s(&slab[buf ^ 1][0][0], x + (sidx + gridDim.x) * SLAB * D, SLAB_BYTES, &bar[buf ^ 1]);
    }
    mbar_wait(&bar[buf], (it >> 1) & 1);
    const int64_t tile = tok0 / TILE;
    const int kt0 = static_cast<int>(tok0 % TILE);
    for (int wi = threadIdx.x; wi < (D / 2) * (SLAB / 32); wi += blockDim.x) {
      const int cp = wi % (D / 2);     // column pair
      const int g32 = wi / (D / 2);    // 32-token group
      float v0[32], v1[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(&slab[buf][g32 * 32 + j][2 * cp]);
        v0[j] = __uint_as_float(w << 16);
        v1[j] = __uint_as_float(w & 0xFFFF0000u);
      }
      const int kt = kt0 + g32 * 32;
      Block16 q[2][2];  // [column][16-token block]
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        float* v = cc ? v1 : v0;
        scale16(*reinterpret_cast<float(*)[16]>(v), inv_ts);
        scale16(*reinterpret_cast<float(*)[16]>(v + 16), inv_ts);
        quantize_block16<FQH, true>(*reinterpret_cast<const float(*)[16]>(v), q[cc][0]);
        quantize_block16<FQH, true>(*reinterpret_cast<const float(*)[16]>(v + 16), q[cc][1]);
        if (nonfinite != nullptr && !(q[cc][0].finite && q[cc][1].finite)) atomicOr(nonfinite, 1);
        const int col = 2 * cp + cc;
        *reinterpret_cast<uint4*>(codes_t + tile * fp4_tile_bytes(D) + t8x32_off(col, kt, D)) =
            make_uint4(q[cc][0].packed[0], q[cc][0].packed[1], q[cc][1].packed[0], q[cc][1].packed[1]);
        *reinterpret_cast<uint16_t*>(sf_t + tile * kSfTileBytesV + sf512_off(col, kt / 16)) =
            static_cast<uint16_t>(q[cc][0].scale | (q[cc][1].scale << 8));
      }
      if (FQH) {
        // token-major f16 pairs (column 2cp, 2cp+1) of the dequantized values
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t a0 = *reinterpret_cast<const uint32_t*>(&q[0][b].fq[j]);
            const uint32_t a1 = *reinterpret_cast<const uint32_t*>(&q[1][b].fq[j]);
            const int tt = g32 * 32 + b * 16 + 2 * j;
            *reinterpret_cast<uint32_t*>(&slab_h[tt][2 * cp]) = __byte_perm(a0, a1, 0x5410);
            *reinterpret_cast<uint32_t*>(&slab_h[tt + 1][2 * cp]) = __byte_perm(a0, a1, 0x7632);
          }
      }
    }
    if (FQH) {
      __syncthreads();
      for (int i = threadIdx.x; i < SLAB * CV; i += blockDim.x) {
        const int tt = i % SLAB, c8 = (i / SLAB) * 8;
        const uint4 w = *reinterpret_cast<const uint4*>(&slab_h[tt][c8]);
        const __half2 h[4] = {*reinterpret_cast<const __half2*>(&w.x), *reinterpret_cast<const __half2*>(&w.y),
                              *reinterpret_cast<const __half2*>(&w.z), *reinterpret_cast<const __half2*>(&w.w)};
        const uint32_t off = static_cast<uint32_t>(tile * h_tile_bytes(D)) + t8x8_off(kt0 + tt, c8);
        if (fqh_t)
          *reinterpret_cast<uint4*>(fqh_t + off) =
              make_uint4(h2_to(h[0], fqh_dt), h2_to(h[1], fqh_dt), h2_to(h[2], fqh_dt), h2_to(h[3], fqh_dt));
        if (fqh2_t)
          *reinterpret_cast<uint4*>(fqh2_t + off) =
              make_uint4(h2_to(h[0], fqh2_dt), h2_to(h[1], fqh2_dt), h2_to(h[2], fqh2_dt), h2_to(h[3], fqh2_dt));
      }
    }
  }
}

template <bool WANT_FQ>
__global__ void __launch_bounds__(128) quantize_cols_kernel(RowsArgs a) {
  __shared__ float slab[kColsSlab][kColsMax + 1];
  const int64_t n16 = ceil_div(a.n, 16);
  const bool tiled = a.codes_t || a.sf_t || a.fqh_t || a.fqh2_t;
  const int64_t nslabs = tiled ? ceil_div(a.n, TILE) * (TILE / kColsSlab) : ceil_div(a.n, kColsSlab);
  const int D = static_cast<int>(a.cols);
  for (int64_t sidx = blockIdx.x; sidx < a.heads * nslabs; sidx += gridDim.x) {
    const int64_t h = sidx / nslabs;
    const int64_t tok0 = (sidx % nslabs) * kColsSlab;
    for (int c0 = 0; c0 < D; c0 += kColsMax) {
      const int cw = min(kColsMax, D - c0);
      __syncthreads();
      const bool vec = a.x_dt == kBF16 && (cw % 8) == 0 && (a.ld % 8) == 0 && (a.hs % 8) == 0 &&
                       (c0 % 8) == 0 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
      if (vec) {
        // all 16-byte loads of the slab in flight at once (up to 8 per thread), then unpack
        const int cv = cw / 8;
        const int nvec = kColsSlab * cv;
        constexpr int PER = kColsSlab * (kColsMax / 8) / 128;
        uint4 w[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = threadIdx.x + k * 128;
          const int tt = i / cv, c = (i % cv) * 8;
          const int64_t tok = tok0 + tt;
          w[k] = (i < nvec && tok < a.n)
                     ? *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.x) + h * a.hs +
                                                       tok * a.ld + c0 + c)
                     : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int i = threadIdx.x + k * 128;
          if (i >= nvec) break;
          const int tt = i / cv, c = (i % cv) * 8;
          const uint32_t ww[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            slab[tt][c + 2 * j] = __uint_as_float(ww[j] << 16);
            slab[tt][c + 2 * j + 1] = __uint_as_float(ww[j] & 0xFFFF0000u);
          }
        }
      } else {
        for (int i = threadIdx.x; i < kColsSlab * cw; i += blockDim.x) {
          const int tt = i / cw, c = i % cw;
          const int64_t tok = tok0 + tt;
          slab[tt][c] = tok < a.n ? load_elem(a.x, h * a.hs + tok * a.ld + c0 + c, a.x_dt) : 0.f;
        }
      }
      __syncthreads();
      // one work item = (column, 32-token group): every thread busy for narrow d too
      for (int wi = threadIdx.x; wi < cw * (kColsSlab / 32); wi += blockDim.x) {
        const int c = wi % cw;
        const int g32 = wi / cw;
        const int64_t col = c0 + c;
        {
          uint32_t codes[4];
          uint32_t scales = 0;
#pragma unroll
          for (int hb = 0; hb < 2; ++hb) {
            const int tb = g32 * 32 + hb * 16;  // first slab row of this block
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = slab[tb + j][c];
            Block16 q;
            scale16(v, a.inv_ts);
            quantize_block16<WANT_FQ>(v, q);
            codes[2 * hb] = q.packed[0];
            codes[2 * hb + 1] = q.packed[1];
            scales |= q.scale << (8 * hb);
            const int64_t b0 = tok0 + tb;
            const int64_t blk = b0 / 16;
            if (blk < n16) {
              if (!q.finite && a.nonfinite) atomicOr(a.nonfinite, 1);
              if (a.codes_ref)
                *reinterpret_cast<uint2*>(a.codes_ref + (h * a.cols + col) * (n16 * 8) + blk * 8) =
                    make_uint2(q.packed[0], q.packed[1]);
              if (a.scales_ref) a.scales_ref[(h * a.cols + col) * n16 + blk] = static_cast<uint8_t>(q.scale);
              if (WANT_FQ && a.fq) {
                const __half* fh = reinterpret_cast<const __half*>(q.fq);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (b0 + j < a.n) store_elem(a.fq, (h * a.n + b0 + j) * a.cols + col, a.fq_dt, __half2float(fh[j]) * a.ts);
              }
            }
            if (WANT_FQ && (a.fqh_t || a.fqh2_t)) {
              // overwrite this column of the slab with its dequantized values; the
              // T8x8 tile is written cooperatively below with 16-byte stores
              const __half* fh = reinterpret_cast<const __half*>(q.fq);
#pragma unroll
              for (int j = 0; j < 16; ++j) slab[tb + j][c] = __half2float(fh[j]);
            }
          }
          if (tiled) {
            const int64_t tstart = tok0 + g32 * 32;
            const int64_t tile = h * ceil_div(a.n, TILE) + tstart / TILE;
            const int kt = static_cast<int>(tstart % TILE);
            if (a.codes_t)
              *reinterpret_cast<uint4*>(a.codes_t + tile * fp4_tile_bytes(D) + t8x32_off(static_cast<int>(col), kt, D)) =
                  make_uint4(codes[0], codes[1], codes[2], codes[3]);
            if (a.sf_t)
              *reinterpret_cast<uint16_t*>(a.sf_t + tile * kSfTileBytesV + sf512_off(static_cast<int>(col), kt / 16)) =
                  static_cast<uint16_t>(scales);
          }
        }
      }
      if (WANT_FQ && (a.fqh_t || a.fqh2_t)) {
        __syncthreads();
        const int64_t tile = h * ceil_div(a.n, TILE) + tok0 / TILE;
        const int kt = static_cast<int>(tok0 % TILE);
        const int cv = cw / 8;
        for (int copy = 0; copy < 2; ++copy) {
          void* dstp = copy ? a.fqh2_t : a.fqh_t;
          const int dt = copy ? a.fqh2_dt : a.fqh_dt;
          if (dstp == nullptr) continue;
          uint8_t* base = reinterpret_cast<uint8_t*>(dstp) + tile * h_tile_bytes(D);
          for (int i = threadIdx.x; i < kColsSlab * cv; i += blockDim.x) {
            const int tt = i % kColsSlab, c8 = (i / kColsSlab) * 8;
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float x0 = slab[tt][c8 + 2 * e], x1 = slab[tt][c8 + 2 * e + 1];
              if (dt == kF16) {
                const __half2 hv = __floats2half2_rn(x0, x1);
                w[e] = *reinterpret_cast<const uint32_t*>(&hv);
              } else {
                const __nv_bfloat162 bv = __floats2bfloat162_rn(x0, x1);
                w[e] = *reinterpret_cast<const uint32_t*>(&bv);
              }
            }
            *reinterpret_cast<uint4*>(base + t8x8_off(kt + tt, c0 + c8)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
  }
}

// K3: reference-layout codes + scales -> dense values. rows x cols.
__global__ void __launch_bounds__(256) dequantize_kernel(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                                                         int64_t cols, void* out, int out_dt, float ts) {
  const int64_t nb = cols / 16;
  const int64_t total = rows * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / nb, b = t % nb;
    const float s = e4m3_to_f32(scales[t]);
    const uint2 w = *reinterpret_cast<const uint2*>(codes + r * (cols / 2) + b * 8);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t word = j < 8 ? w.x : w.y;
      const uint32_t code = (word >> (4 * (j & 7))) & 0xF;
      store_elem(out, r * cols + b * 16 + j, out_dt, e2m1_to_f32(code) * s * ts);  // ts = 1: exact
    }
  }
}

static int grid_for(int64_t work) {
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// Plain (unquantized) attention operands: [heads][n][d] -> 16-bit T8x8 tiles,
// padding rows zero. One thread = 8 consecutive columns of one row.
template <int D>
__global__ void __launch_bounds__(256) tile16_kernel(const void* __restrict__ x, int x_dt, int64_t heads, int64_t n,
                                                     int fmt, uint8_t* __restrict__ out) {
  const int64_t n_pad = ceil_div(n, TILE) * TILE;
  const int64_t total = heads * n_pad * (D / 8);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(t % (D / 8));
    const int64_t rp = t / (D / 8);  // padded row over all heads
    const int64_t h = rp / n_pad, r = rp % n_pad;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = r < n ? load_elem(x, (h * n + r) * D + c8 * 8 + e, x_dt) : 0.f;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (fmt == 1) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        w[e] = *reinterpret_cast<const uint32_t*>(&b);
      } else {
        const __half2 b = __floats2half2_rn(v[2 * e], v[2 * e + 1]);
        w[e] = *reinterpret_cast<const uint32_t*>(&b);
      }
    }
    *reinterpret_cast<uint4*>(out + (h * (n_pad / TILE) + r / TILE) * h_tile_bytes(D) +
                              t8x8_off(static_cast<int>(r % TILE), c8 * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

cudaError_t launch_tile16(const void* x, int x_dt, int64_t heads, int64_t n, int d, int fmt, uint8_t* out,
                          cudaStream_t st) {
  const int g = grid_for(heads * ceil_div(n, TILE) * TILE * (d / 8));
  if (d == 64) tile16_kernel<64><<<g, 256, 0, st>>>(x, x_dt, heads, n, fmt, out);
  else if (d == 128) tile16_kernel<128><<<g, 256, 0, st>>>(x, x_dt, heads, n, fmt, out);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_quantize_rows(const RowsArgs& a, cudaStream_t st) {
  const int64_t n_pad = (a.codes_t || a.sf_t || a.fqh_t) ? ceil_div(a.n, TILE) * TILE : a.n;
  const bool fast = (a.x_dt == kBF16 || a.x_dt == kF32) && a.codes_t && a.sf_t && !a.fq && !a.codes_ref &&
                    !a.scales_ref && a.ld == a.cols && a.hs == a.n * a.cols &&
                    (a.cols == 64 || a.cols == 128) && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
  if (fast && a.x_dt == kF32 && !a.fqh_t) {
    const int g = grid_for(a.heads * n_pad * (a.cols / 32));
    if (a.cols == 128) quantize_rows_tiled_kernel<128, false, true><<<g, 256, 0, st>>>(a.x, a.heads, a.n, a.codes_t, a.sf_t, nullptr, 0, a.inv_ts, a.nonfinite);
    else quantize_rows_tiled_kernel<64, false, true><<<g, 256, 0, st>>>(a.x, a.heads, a.n, a.codes_t, a.sf_t, nullptr, 0, a.inv_ts, a.nonfinite);
    return cudaGetLastError();
  }
  if (fast && a.x_dt == kBF16) {
    const int g = grid_for(a.heads * n_pad * (a.cols / 32));
    const auto* x = a.x;
    uint8_t* fqh = static_cast<uint8_t*>(a.fqh_t);
    if (a.cols == 128) {
      if (fqh) quantize_rows_tiled_kernel<128, true><<<g, 256, 0, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, fqh, a.fqh_dt, a.inv_ts, a.nonfinite);
      else quantize_rows_tiled_kernel<128, false><<<g, 256, 0, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, nullptr, 0, a.inv_ts, a.nonfinite);
    } else {
      if (fqh) quantize_rows_tiled_kernel<64, true><<<g, 256, 0, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, fqh, a.fqh_dt, a.inv_ts, a.nonfinite);
      else quantize_rows_tiled_kernel<64, false><<<g, 256, 0, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, nullptr, 0, a.inv_ts, a.nonfinite);
    }
    return cudaGetLastError();
  }
  const int g = grid_for(a.heads * n_pad * ((a.cols / 16 + 1) / 2));
  const bool fq = a.fq || a.fqh_t;
  if (a.cols == 128) {
    if (fq) quantize_rows_kernel<true, 4><<<g, 256, 0, st>>>(a);
    else quantize_rows_kernel<false, 4><<<g, 256, 0, st>>>(a);
  } else if (a.cols == 64) {
    if (fq) quantize_rows_kernel<true, 2><<<g, 256, 0, st>>>(a);
    else quantize_rows_kernel<false, 2><<<g, 256, 0, st>>>(a);
  } else {
    if (fq) quantize_rows_kernel<true, 0><<<g, 256, 0, st>>>(a);
    else quantize_rows_kernel<false, 0><<<g, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

// K2 inference fast path (bf16, no 16-bit tiles): one CTA of D threads per
// 32-token slab staged through shared memory with 16-byte loads; thread c
// quantizes column c's two 16-token blocks and writes 16 code bytes + 2 scales.
template <int D>
__global__ void __launch_bounds__(D) quantize_cols_slab_kernel(const __nv_bfloat16* __restrict__ x, int64_t heads,
                                                               int64_t n, uint8_t* __restrict__ codes_t,
                                                               uint8_t* __restrict__ sf_t, float inv_ts,
                                                               int* __restrict__ nonfinite) {
  // 32 contiguous token rows per slab, double-buffered 1-D bulk copies (the
  // column reads touch one row per instruction: no padding needed). A ragged
  // head (n % 128 != 0, e.g. C3's N = 32760) is zero-padded to whole tiles, as
  // quantize_padded pads V^T (codec.py:359-381): the slab's rows past n are
  // zeroed in shared memory and quantized like the general kernel does.
  __shared__ __align__(128) __nv_bfloat16 slab[2][32][D];
  __shared__ __align__(8) uint64_t bar[2];
  const int64_t n_pad = ceil_div(n, TILE) * TILE;
  const int64_t spp = n_pad / 32;  // slabs per head
  const int64_t nslabs = heads * spp;
  const int c = threadIdx.x;
  auto valid_rows = [&](int64_t sidx) {
    const int64_t left = n - (sidx % spp) * 32;
    return static_cast<int>(left < 0 ? 0 : (left < 32 ? left : 32));
  };
  auto issue = [&](int64_t sidx, int b) {  // thread 0
    const int valid = valid_rows(sidx);
    if (valid > 0) {
      mbar_expect_tx(&bar[b], static_cast<uint32_t>(valid) * D * 2);
      bulk_g2s(&slab[b][0][0], x + ((sidx / spp) * n + (sidx % spp) * 32) * D, static_cast<uint32_t>(valid) * D * 2,
               &bar[b]);
    } else {
      mbar_arrive(&bar[b]);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    if (blockIdx.x < nslabs) issue(blockIdx.x, 0);
  }
  int it = 0;
  for (int64_t sidx = blockIdx.x; sidx < nslabs; sidx += gridDim.x, ++it) {
    const int64_t tok0 = sidx * 32;  // flat padded token index (n_pad % 128 == 0: slabs never straddle heads)
    const int buf = it & 1;
    __syncthreads();  // every thread is done with slab[buf ^ 1]
    if (threadIdx.x == 0 && sidx + gridDim.x < nslabs) {
      fence_async_smem();
      issue(sidx + gridDim.x, buf ^ 1);
    }
    mbar_wait(&bar[buf], (it >> 1) & 1);
    const int valid = valid_rows(sidx);  // uniform over the CTA
    if (valid < 32) {
      for (int r = valid; r < 32; ++r) slab[buf][r][c] = __float2bfloat16_rn(0.f);
      __syncthreads();
    }
    Block16 q[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __bfloat162float(slab[buf][16 * b + j][c]);
      scale16(v, inv_ts);
      quantize_block16<false, true>(v, q[b]);
    }
    if (nonfinite != nullptr && !(q[0].finite && q[1].finite)) atomicOr(nonfinite, 1);
    const int64_t tile = tok0 / TILE;
    const int kt = static_cast<int>(tok0 % TILE);
    *reinterpret_cast<uint4*>(codes_t + tile * fp4_tile_bytes(D) + t8x32_off(c, kt, D)) =
        make_uint4(q[0].packed[0], q[0].packed[1], q[1].packed[0], q[1].packed[1]);
    *reinterpret_cast<uint16_t*>(sf_t + tile * kSfTileBytesV + sf512_off(c, kt / 16)) =
        static_cast<uint16_t>(q[0].scale | (q[1].scale << 8));
  }
}

cudaError_t launch_quantize_cols(const RowsArgs& a, cudaStream_t st) {
  // fast paths: bf16, contiguous heads, MMA tile outputs only; the inference
  // (slab) kernel also takes a ragged last tile, the training kernel whole tiles
  const bool fast = a.x_dt == kBF16 && a.codes_t && a.sf_t && !a.fq && !a.codes_ref && !a.scales_ref &&
                    a.ld == a.cols && a.hs == a.n * a.cols &&
                    (a.cols == 64 || a.cols == 128) && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
  const bool fqh = a.fqh_t || a.fqh2_t;
  if (fast && (!fqh || a.n % TILE == 0)) {
    int64_t g = a.heads * (a.n / 64);
    if (g > 148 * 64) g = 148 * 64;
    const auto* x = static_cast<const __nv_bfloat16*>(a.x);
    auto* h1 = static_cast<uint8_t*>(a.fqh_t);
    auto* h2 = static_cast<uint8_t*>(a.fqh2_t);
    const int gg = static_cast<int>(g);
    if (!fqh) {
      int64_t gs = a.heads * (ceil_div(a.n, TILE) * TILE / 32);
      if (gs > 148 * 16) gs = 148 * 16;
      if (a.cols == 128)
        quantize_cols_slab_kernel<128><<<static_cast<int>(gs), 128, 0, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, a.inv_ts, a.nonfinite);
      else
        quantize_cols_slab_kernel<64><<<static_cast<int>(gs), 64, 0, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, a.inv_ts, a.nonfinite);
      return cudaGetLastError();
    }
    // dynamic smem: two bf16 slabs, the barriers, the f16 stage (training)
    const int sm = static_cast<int>(2 * 64 * a.cols * 2 + 16 + (fqh ? 64 * (a.cols + 8) * 2 : 0));
    if (a.cols == 128) {
      if (fqh) {
        cudaFuncSetAttribute(quantize_cols_tiled_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        quantize_cols_tiled_kernel<128, true><<<gg, 128, sm, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, h1, a.fqh_dt, h2, a.fqh2_dt, a.inv_ts, a.nonfinite);
      } else {
        quantize_cols_tiled_kernel<128, false><<<gg, 128, sm, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, nullptr, 0, nullptr, 0, a.inv_ts, a.nonfinite);
      }
    } else {
      if (fqh) quantize_cols_tiled_kernel<64, true><<<gg, 128, sm, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, h1, a.fqh_dt, h2, a.fqh2_dt, a.inv_ts, a.nonfinite);
      else quantize_cols_tiled_kernel<64, false><<<gg, 128, sm, st>>>(x, a.heads, a.n, a.codes_t, a.sf_t, nullptr, 0, nullptr, 0, a.inv_ts, a.nonfinite);
    }
    return cudaGetLastError();
  }
  const bool tiled = a.codes_t || a.sf_t || a.fqh_t || a.fqh2_t;
  const int64_t nslabs = tiled ? ceil_div(a.n, TILE) * (TILE / kColsSlab) : ceil_div(a.n, kColsSlab);
  int64_t g = a.heads * nslabs;
  if (g > 148 * 64) g = 148 * 64;
  if (a.fq || a.fqh_t || a.fqh2_t)
    quantize_cols_kernel<true><<<static_cast<int>(g), 128, 0, st>>>(a);
  else
    quantize_cols_kernel<false><<<static_cast<int>(g), 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                              int out_dt, cudaStream_t st, float ts) {
  dequantize_kernel<<<grid_for(rows * (cols / 16)), 256, 0, st>>>(codes, scales, rows, cols, out, out_dt, ts);
  return cudaGetLastError();
}



// ---------------------------------------------------------------------------
// Element-wise code rounding (codec.py:63-112): round_to_fp4 / round_to_e4m3.
// Exact in the input precision (fp32 or fp64): the code is the number of
// rounding midpoints below |x|, a tie (|x| exactly on a midpoint) goes to the
// even code. Every midpoint of both formats is exact in fp32, so comparing in
// the input's own precision reproduces the reference's float64 rounding with
// no double rounding. fp4: |x| saturates at 6, a negative non-zero value keeps
// the sign nibble (codec.py:84-87). e4m3: 0 <= x, saturates at 448 (0x7E).
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ double e4m3_code_value(int c) {
  return c < 8 ? c * 0.001953125 : (1.0 + (c & 7) * 0.125) * ldexp(1.0, (c >> 3) - 7);
}

template <typename T, int FMT>
__global__ void __launch_bounds__(256) round_codes_kernel(const T* __restrict__ x, int64_t n,
                                                          uint8_t* __restrict__ codes, int* invalid) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T v = x[i];
    const bool finite = isfinite(static_cast<double>(v));
    if (!finite || (FMT == 1 && v < T(0))) {
      if (invalid) atomicOr(invalid, 1);
      codes[i] = 0;
      continue;
    }
    const T mag = fabs(v);
    int lo = 0, hi = 0;
    if (FMT == 0) {
      const T m = mag < T(6) ? mag : T(6);
      const T mids[7] = {T(0.25), T(0.75), T(1.25), T(1.75), T(2.5), T(3.5), T(5)};
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        lo += mids[k] < m;
        hi += mids[k] <= m;
      }
    } else {
      const T m = mag < T(448) ? mag : T(448);
      // binary search over the 126 midpoints mid(c) = (val(c) + val(c+1)) / 2, c = 0..125
      int a = 0, b = 126;  // lo = #mids < m
      while (a < b) {
        const int c = (a + b) >> 1;
        if (static_cast<T>(0.5 * (e4m3_code_value(c) + e4m3_code_value(c + 1))) < m) a = c + 1;
        else b = c;
      }
      lo = a;
      hi = (lo < 126 && static_cast<T>(0.5 * (e4m3_code_value(lo) + e4m3_code_value(lo + 1))) == m) ? lo + 1 : lo;
    }
    int code = lo != hi ? lo + (lo & 1) : lo;
    if (FMT == 0 && signbit(static_cast<double>(v)) && v != T(0)) code |= 0x8;
    codes[i] = static_cast<uint8_t>(code);
  }
}

}  // namespace

cudaError_t launch_round_codes(const void* x, int x_is_f64, int64_t n, int format, uint8_t* codes, int* invalid,
                               cudaStream_t st) {
  int64_t g = ceil_div(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  const int grid = static_cast<int>(g < 1 ? 1 : g);
  if (x_is_f64) {
    if (format == 0) round_codes_kernel<double, 0><<<grid, 256, 0, st>>>(static_cast<const double*>(x), n, codes, invalid);
    else round_codes_kernel<double, 1><<<grid, 256, 0, st>>>(static_cast<const double*>(x), n, codes, invalid);
  } else {
    if (format == 0) round_codes_kernel<float, 0><<<grid, 256, 0, st>>>(static_cast<const float*>(x), n, codes, invalid);
    else round_codes_kernel<float, 1><<<grid, 256, 0, st>>>(static_cast<const float*>(x), n, codes, invalid);
  }
  return cudaGetLastError();
}



// ---------------------------------------------------------------------------
// MXFP4 (32-element blocks, E8M0 power-of-two scales; codec.py:123-142,
// 169-203): scale code = round-to-nearest power of two of amax / 6 with ties
// up (0 for an all-zero block), elements = E2M1_RNE(x / 2^(code-127)). The
// division by a power of two is exact, so x * 2^(127-code) feeds the hardware
// E2M1 convert directly; amax / 6 is IEEE-rounded (its E8M0 rounding cannot
// straddle the 1.5 * 2^e midpoint for fp32-representable inputs).
// ---------------------------------------------------------------------------
namespace {

template <typename T>
__device__ __forceinline__ uint32_t e8m0_code(T raw) {  // raw > 0, finite (codec.py:123-136)
  int e;
  const T m = frexp(raw, &e);                  // raw = m 2^e, m in [0.5, 1)
  const int ex = (T(2) * m < T(1.5)) ? e - 1 : e;
  const int c = ex + 127;
  return static_cast<uint32_t>(c < 0 ? 0 : (c > 254 ? 254 : c));
}

__device__ __forceinline__ float e8m0_value(uint32_t code) { return ldexpf(1.0f, static_cast<int>(code) - 127); }
// the same value from the exponent bits; code 0 is 2^-127 (an fp32 subnormal),
// as in the reference (codec.py:123-136), not the 0.0 that code << 23 would give
__device__ __forceinline__ float e8m0_bits(uint32_t code) {
  return code ? __int_as_float(static_cast<int>(code << 23)) : __int_as_float(0x00400000);
}

__global__ void __launch_bounds__(256) quantize_mx_kernel(const void* x, int x_dt, int64_t rows, int64_t cols,
                                                          uint8_t* codes, uint8_t* scales, void* fq, int fq_dt,
                                                          int* nonfinite) {
  const int64_t nb = cols / 32;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * nb;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / nb, b = t % nb;
    const int64_t i0 = r * cols + b * 32;
    float v[32];
    float amax = 0.f;
    bool finite = true;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = load_elem(x, i0 + j, x_dt);
      finite = finite && isfinite(v[j]);
      amax = fmaxf(amax, fabsf(v[j]));
    }
    if (!finite && nonfinite) atomicOr(nonfinite, 1);
    const float raw = div_rn(amax, 6.0f, 0.16666667163372039795f);
    const uint32_t sc = raw > 0.f ? e8m0_code(raw) : 0u;
    const float rs = __int_as_float(static_cast<int>((254u - sc) << 23));  // 2^(127 - code), exact
    const float s = e8m0_value(sc);
    float q[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) q[j] = v[j] * rs + 0.0f;  // + 0 maps -0.0 to +0 (codec.py:84)
    uint32_t packed[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) packed[k] = cvt_e2m1x8(q + 8 * k);
    if (codes)
      *reinterpret_cast<uint4*>(codes + r * (cols / 2) + b * 16) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    if (scales) scales[t] = static_cast<uint8_t>(sc);
    if (fq) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        store_elem(fq, i0 + j, fq_dt, e2m1_to_f32((packed[j >> 3] >> (4 * (j & 7))) & 0xF) * s);
    }
  }
}

__global__ void __launch_bounds__(256) dequantize_mx_kernel(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                                                            int64_t cols, void* out, int out_dt) {
  const int64_t nb = cols / 32;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * nb;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / nb, b = t % nb;
    const float s = e8m0_value(scales[t]);
    const uint4 w = *reinterpret_cast<const uint4*>(codes + r * (cols / 2) + b * 16);
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 32; ++j)
      store_elem(out, r * cols + b * 32 + j, out_dt, e2m1_to_f32((ww[j >> 3] >> (4 * (j & 7))) & 0xF) * s);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) e8m0_codes_kernel(const T* __restrict__ x, int64_t n, uint8_t* codes,
                                                         int* invalid) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T v = x[i];
    if (!isfinite(static_cast<double>(v)) || !(v > T(0))) {
      if (invalid) atomicOr(invalid, 1);
      codes[i] = 0;
      continue;
    }
    codes[i] = static_cast<uint8_t>(e8m0_code(v));
  }
}

}  // namespace

// MXFP4 attention operands straight into the MMA tiles (codec.py:123-203 per
// block, layouts.cuh images): Q / K rows blocked along d (one SF512 image per
// tile holds the 4 blocks of 32 of a 128-wide row), V^T blocked along tokens
// (per column, 4 blocks of 32 tokens per tile). Padding rows / tokens are zero.
__device__ __forceinline__ void mx_block(const float* v, uint32_t (&packed)[4], uint32_t& sc) {
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) amax = fmaxf(amax, fabsf(v[j]));
  const float raw = div_rn(amax, 6.0f, 0.16666667163372039795f);
  sc = raw > 0.f ? e8m0_code(raw) : 0u;
  const float rs = __int_as_float(static_cast<int>((254u - sc) << 23));
  float q[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) q[j] = v[j] * rs + 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) packed[k] = cvt_e2m1x8(q + 8 * k);
}

template <int D>
__global__ void __launch_bounds__(256) mx_rows_tiled_kernel(const void* x, int x_dt, int64_t heads, int64_t n,
                                                            uint8_t* codes_t, uint8_t* sf_t, uint8_t* fqh_t = nullptr) {
  const int64_t n_pad = ceil_div(n, TILE) * TILE;
  const int64_t total = heads * n_pad * (D / 32);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(t % (D / 32));
    const int64_t rp = t / (D / 32);
    const int64_t h = rp / n_pad, r = rp % n_pad;
    float v[32];
    if (x_dt == kBF16 && r < n && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {  // 4 x 16-byte loads
      const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + (h * n + r) * D + b * 32);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const uint4 w = src[q4];
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[8 * q4 + 2 * e] = __uint_as_float(ww[e] << 16);
          v[8 * q4 + 2 * e + 1] = __uint_as_float(ww[e] & 0xFFFF0000u);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = r < n ? load_elem(x, (h * n + r) * D + b * 32 + j, x_dt) : 0.f;
    }
    uint32_t packed[4], sc;
    mx_block(v, packed, sc);
    const int64_t tile = h * (n_pad / TILE) + r / TILE;
    const int rr = static_cast<int>(r % TILE);
    *reinterpret_cast<uint4*>(codes_t + tile * fp4_tile_bytes(D) + t8x32_off(rr, 32 * b, TILE)) =
        make_uint4(packed[0], packed[1], packed[2], packed[3]);
    sf_t[tile * sf_tile_bytes_qk(D) + sf512_off(rr, b)] = static_cast<uint8_t>(sc);
    if (fqh_t) {  // the bf16 fake-quantized operand tile of the backward (T8x8):
      // byte-permute lookups of the E2M1 magnitudes' bf16 bytes, the sign bit
      // from the code, then one exact bf16x2 multiply by the power-of-two scale
      const __nv_bfloat16 sb = __float2bfloat16_rn(e8m0_bits(sc));
      const __nv_bfloat162 s2 = __halves2bfloat162(sb, sb);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint32_t w[4];
#pragma unroll
        for (int q4 = 0; q4 < 2; ++q4) {
          const uint32_t cw = (packed[g] >> (16 * q4)) & 0xFFFFu;   // 4 codes
          const uint32_t sel = cw & 0x7777u;                          // magnitudes
          const uint32_t lo = __byte_perm(0xC0800000u, 0xC0804000u, sel);
          const uint32_t hi = __byte_perm(0x3F3F3F00u, 0x40404040u, sel);
          uint32_t v01 = __byte_perm(lo, hi, 0x5140), v23 = __byte_perm(lo, hi, 0x7362);
          // signs: code bit 3 of each nibble -> bit 15 of each bf16 half
          v01 |= ((cw & 0x8u) << 12) | ((cw & 0x80u) << 24);
          v23 |= ((cw & 0x800u) << 4) | ((cw & 0x8000u) << 16);
          const __nv_bfloat162 p01 = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v01), s2);
          const __nv_bfloat162 p23 = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&v23), s2);
          w[2 * q4] = *reinterpret_cast<const uint32_t*>(&p01);
          w[2 * q4 + 1] = *reinterpret_cast<const uint32_t*>(&p23);
        }
        *reinterpret_cast<uint4*>(fqh_t + tile * h_tile_bytes(D) + t8x8_off(rr, 32 * b + 8 * g)) =
            make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256) mx_cols_tiled_kernel(const void* x, int x_dt, int64_t heads, int64_t n,
                                                            uint8_t* codes_t, uint8_t* sf_t, uint8_t* fqh_t,
                                                            int fqh_bf16 = 0) {
  const int64_t n_pad = ceil_div(n, TILE) * TILE;
  const int64_t total = heads * (n_pad / 32) * D;  // (head, 32-token block, column)
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % D);
    const int64_t bb = t / D;                 // 32-token block over all heads
    const int64_t h = bb / (n_pad / 32), tok0 = (bb % (n_pad / 32)) * 32;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = tok0 + j < n ? load_elem(x, (h * n + tok0 + j) * D + c, x_dt) : 0.f;
    uint32_t packed[4], sc;
    mx_block(v, packed, sc);
    const int64_t tile = h * (n_pad / TILE) + tok0 / TILE;
    const int kt = static_cast<int>(tok0 % TILE);
    *reinterpret_cast<uint4*>(codes_t + tile * fp4_tile_bytes(D) + t8x32_off(c, kt, D)) =
        make_uint4(packed[0], packed[1], packed[2], packed[3]);
    sf_t[tile * kSfTileBytesV + sf512_off(c, kt / 32)] = static_cast<uint8_t>(sc);
    if (fqh_t) {  // training: V^F as fp16 T8x8 tiles for the O' MMA (exact: E2M1 x power of two)
      const float s = e8m0_bits(sc);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float fv = e2m1_to_f32((packed[j >> 3] >> (4 * (j & 7))) & 0xF) * s;
        if (fqh_bf16)
          *reinterpret_cast<__nv_bfloat16*>(fqh_t + tile * h_tile_bytes(D) + t8x8_off(kt + j, c)) =
              __float2bfloat16_rn(fv);
        else
          *reinterpret_cast<__half*>(fqh_t + tile * h_tile_bytes(D) + t8x8_off(kt + j, c)) = __float2half_rn(fv);
      }
    }
  }
}

// bf16 fast path of mx_cols_tiled_kernel: one CTA (D threads) per 32-token slab,
// staged through shared memory with 16-byte coalesced loads; thread c
// quantizes column c.
template <int D>
__global__ void __launch_bounds__(D) mx_cols_slab_kernel(const __nv_bfloat16* __restrict__ x, int64_t heads, int64_t n,
                                                         uint8_t* codes_t, uint8_t* sf_t, uint8_t* fqh_t, int fqh_bf16,
                                                         uint8_t* fqh2_t = nullptr) {
  constexpr int PITCH = D + 8;
  __shared__ __align__(16) __nv_bfloat16 slab[32][PITCH];
  const int64_t n_pad = ceil_div(n, TILE) * TILE;
  const int64_t nslabs = heads * (n_pad / 32);
  const int c = threadIdx.x;
  for (int64_t sidx = blockIdx.x; sidx < nslabs; sidx += gridDim.x) {
    const int64_t h = sidx / (n_pad / 32), tok0 = (sidx % (n_pad / 32)) * 32;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32 * D / 8 / D; ++k) {
      const int i = threadIdx.x + k * D;
      const int tt = i / (D / 8), cc = (i % (D / 8)) * 8;
      uint4 w = make_uint4(0u, 0u, 0u, 0u);
      if (tok0 + tt < n) w = *reinterpret_cast<const uint4*>(x + (h * n + tok0 + tt) * D + cc);
      *reinterpret_cast<uint4*>(&slab[tt][cc]) = w;
    }
    __syncthreads();
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __bfloat162float(slab[j][c]);
    uint32_t packed[4], sc;
    mx_block(v, packed, sc);
    const int64_t tile = h * (n_pad / TILE) + tok0 / TILE;
    const int kt = static_cast<int>(tok0 % TILE);
    *reinterpret_cast<uint4*>(codes_t + tile * fp4_tile_bytes(D) + t8x32_off(c, kt, D)) =
        make_uint4(packed[0], packed[1], packed[2], packed[3]);
    sf_t[tile * kSfTileBytesV + sf512_off(c, kt / 32)] = static_cast<uint8_t>(sc);
    // dequantized values back into the slab (16-bit, same element width),
    // then 16-byte T8x8 stores of 8 columns per token; fqh2_t gets the fp16
    // copy when fqh_t takes bf16 (training + backward in one pass)
    for (int pass = 0; pass < 2; ++pass) {
      uint8_t* dst = pass == 0 ? fqh_t : fqh2_t;
      if (!dst) continue;
      const bool bf = pass == 0 && fqh_bf16;
      const float s = e8m0_bits(sc);
      __syncthreads();  // every column has read its tokens / the previous copy is stored
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float fv = e2m1_to_f32((packed[j >> 3] >> (4 * (j & 7))) & 0xF) * s;
        if (bf) slab[j][c] = __float2bfloat16_rn(fv);
        else *reinterpret_cast<__half*>(&slab[j][c]) = __float2half_rn(fv);
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 32 * D / 8 / D; ++k) {
        const int i = threadIdx.x + k * D;
        const int tt = i % 32, c8 = (i / 32) * 8;
        *reinterpret_cast<uint4*>(dst + tile * h_tile_bytes(D) + t8x8_off(kt + tt, c8)) =
            *reinterpret_cast<const uint4*>(&slab[tt][c8]);
      }
    }
  }
}

template <int D>
static void mx_cols(const void* v, int x_dt, int64_t heads, int64_t n_k, uint8_t* codes, uint8_t* sf, uint8_t* fqh,
                    int fqh_bf16, cudaStream_t st, uint8_t* fqh2_f16 = nullptr) {
  if (x_dt == kBF16 && (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
    int64_t g = heads * (ceil_div(n_k, TILE) * TILE / 32);
    if (g > 148 * 16) g = 148 * 16;
    mx_cols_slab_kernel<D><<<static_cast<int>(g), D, 0, st>>>(static_cast<const __nv_bfloat16*>(v), heads, n_k, codes,
                                                              sf, fqh, fqh_bf16, fqh2_f16);
  } else {
    const int gv = grid_for(heads * ceil_div(n_k, TILE) * 4 * D);
    mx_cols_tiled_kernel<D><<<gv, 256, 0, st>>>(v, x_dt, heads, n_k, codes, sf, fqh, fqh_bf16);
    if (fqh2_f16) mx_cols_tiled_kernel<D><<<gv, 256, 0, st>>>(v, x_dt, heads, n_k, codes, sf, fqh2_f16, 0);
  }
}

cudaError_t launch_mx_bwd_operands(const void* q, const void* k, const void* v, int x_dt, int64_t heads,
                                   int64_t n_q, int64_t n_k, int d, uint8_t* q_codes, uint8_t* q_sf, uint8_t* q_h,
                                   uint8_t* k_codes, uint8_t* k_sf, uint8_t* k_h, uint8_t* v_codes, uint8_t* v_sf,
                                   uint8_t* v_h, cudaStream_t st, uint8_t* v_h16) {
  const int gq = grid_for(heads * ceil_div(n_q, TILE) * TILE * (d / 32));
  const int gk = grid_for(heads * ceil_div(n_k, TILE) * TILE * (d / 32));
  const int gv = grid_for(heads * ceil_div(n_k, TILE) * 4 * d);
  // (the V^T codes / scales are a by-product here: the backward reads V^F only)
  if (d == 128) {
    mx_cols<128>(v, x_dt, heads, n_k, v_codes, v_sf, v_h, 1, st, v_h16);
    mx_rows_tiled_kernel<128><<<gq, 256, 0, st>>>(q, x_dt, heads, n_q, q_codes, q_sf, q_h);
    mx_rows_tiled_kernel<128><<<gk, 256, 0, st>>>(k, x_dt, heads, n_k, k_codes, k_sf, k_h);
  } else if (d == 64) {
    mx_cols<64>(v, x_dt, heads, n_k, v_codes, v_sf, v_h, 1, st, v_h16);
    mx_rows_tiled_kernel<64><<<gq, 256, 0, st>>>(q, x_dt, heads, n_q, q_codes, q_sf, q_h);
    mx_rows_tiled_kernel<64><<<gk, 256, 0, st>>>(k, x_dt, heads, n_k, k_codes, k_sf, k_h);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_mx_attn_operands(const void* q, const void* k, const void* v, int x_dt, int64_t heads,
                                    int64_t n_q, int64_t n_k, int d, uint8_t* q_codes, uint8_t* q_sf,
                                    uint8_t* k_codes, uint8_t* k_sf, uint8_t* v_codes, uint8_t* v_sf,
                                    uint8_t* v_h16, cudaStream_t st) {
  const int gq = grid_for(heads * ceil_div(n_q, TILE) * TILE * (d / 32));
  const int gk = grid_for(heads * ceil_div(n_k, TILE) * TILE * (d / 32));
  const int gv = grid_for(heads * ceil_div(n_k, TILE) * 4 * d);
  if (d == 128) {
    mx_rows_tiled_kernel<128><<<gq, 256, 0, st>>>(q, x_dt, heads, n_q, q_codes, q_sf);
    mx_rows_tiled_kernel<128><<<gk, 256, 0, st>>>(k, x_dt, heads, n_k, k_codes, k_sf);
    mx_cols<128>(v, x_dt, heads, n_k, v_codes, v_sf, v_h16, 0, st);
  } else if (d == 64) {
    mx_rows_tiled_kernel<64><<<gq, 256, 0, st>>>(q, x_dt, heads, n_q, q_codes, q_sf);
    mx_rows_tiled_kernel<64><<<gk, 256, 0, st>>>(k, x_dt, heads, n_k, k_codes, k_sf);
    mx_cols<64>(v, x_dt, heads, n_k, v_codes, v_sf, v_h16, 0, st);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_quantize_mx(const void* x, int x_dt, int64_t rows, int64_t cols, uint8_t* codes, uint8_t* scales,
                               void* fq, int fq_dt, int* nonfinite, cudaStream_t st) {
  quantize_mx_kernel<<<grid_for(rows * (cols / 32)), 256, 0, st>>>(x, x_dt, rows, cols, codes, scales, fq, fq_dt,
                                                                    nonfinite);
  return cudaGetLastError();
}

cudaError_t launch_dequantize_mx(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                                 int out_dt, cudaStream_t st) {
  dequantize_mx_kernel<<<grid_for(rows * (cols / 32)), 256, 0, st>>>(codes, scales, rows, cols, out, out_dt);
  return cudaGetLastError();
}

cudaError_t launch_e8m0_codes(const void* x, int x_is_f64, int64_t n, uint8_t* codes, int* invalid, cudaStream_t st) {
  if (x_is_f64)
    e8m0_codes_kernel<double><<<grid_for(n), 256, 0, st>>>(static_cast<const double*>(x), n, codes, invalid);
  else
    e8m0_codes_kernel<float><<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(x), n, codes, invalid);
  return cudaGetLastError();
}

}  // namespace aq
