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

// Quantize one 16-element block. Returns the scale code; fills packed codes
// (8 bytes as two u32) and the decoded (exact) fake-quantized values.
struct Block16 {
  uint32_t scale;
  uint32_t packed[2];
  float fq[16];
  bool finite;
};

__device__ __forceinline__ void quantize_block16(const float (&v)[16], Block16& out) {
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) amax = fmaxf(amax, fabsf(v[j]));
  // NaN propagates as "not <= max" ; inf fails too
  bool finite = true;
#pragma unroll
  for (int j = 0; j < 16; ++j) finite &= (fabsf(v[j]) <= 3.402823466e38f);
  out.finite = finite;
  const float raw = __fdiv_rn(amax, 6.0f);
  uint32_t sc = cvt_e4m3(raw);
  if (sc == 0 && amax > 0.f) sc = 1;  // tiny non-zero block keeps 2^-9
  out.scale = sc;
  const float s = e4m3_to_f32(sc);
  uint32_t w0 = 0, w1 = 0;
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    float q0 = 0.f, q1 = 0.f;
    if (s > 0.f) {
      q0 = (v[j] == 0.f) ? 0.f : __fdiv_rn(v[j], s);
      q1 = (v[j + 1] == 0.f) ? 0.f : __fdiv_rn(v[j + 1], s);
    }
    const uint32_t byte = cvt_e2m1x2(q0, q1);
    out.fq[j] = e2m1_to_f32(byte & 0xF) * s;
    out.fq[j + 1] = e2m1_to_f32(byte >> 4) * s;
    if (j < 8)
      w0 |= byte << (4 * j);
    else
      w1 |= byte << (4 * (j - 8));
  }
  out.packed[0] = w0;
  out.packed[1] = w1;
}

// ---------------------------------------------------------------------------
// K1: blocks along the contiguous (column) axis. x is [heads][n][cols] with
// row stride `ld` elements and head stride `hs` elements. One thread per block.
// Optional outputs (nullptr to skip):
//   codes_ref [heads*n][cols/2], scales_ref [heads*n][cols/16]  (reference layout)
//   fq        [heads*n][cols] dense dequantized values (dtype fq_dt)
//   codes_t   T8x32 tiles per head (n padded to 128; pad rows written as 0)
//   sf_t      SF512 images per tile
//   fqh_t     T8x8 16-bit tiles of the dequantized values (dtype fqh_dt)
// ---------------------------------------------------------------------------


__global__ void __launch_bounds__(256) quantize_rows_kernel(RowsArgs a) {
  const int64_t nb = a.cols / 16;
  const int64_t n_pad = (a.codes_t || a.sf_t || a.fqh_t) ? ceil_div(a.n, TILE) * TILE : a.n;
  const int64_t total = a.heads * n_pad * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = t % nb;
    const int64_t rowp = t / nb;
    const int64_t h = rowp / n_pad;
    const int64_t r = rowp % n_pad;
    const bool real = r < a.n;
    float v[16];
    if (real) {
      load16(a.x, h * a.hs + r * a.ld + b * 16, a.x_dt, v);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
    }
    Block16 q;
    quantize_block16(v, q);
    if (real) {
      const int64_t row = h * a.n + r;
      if (!q.finite && a.nonfinite) atomicOr(a.nonfinite, 1);
      if (a.codes_ref) {
        uint2* dst = reinterpret_cast<uint2*>(a.codes_ref + row * (a.cols / 2) + b * 8);
        *dst = make_uint2(q.packed[0], q.packed[1]);
      }
      if (a.scales_ref) a.scales_ref[row * nb + b] = static_cast<uint8_t>(q.scale);
      if (a.fq) {
#pragma unroll
        for (int j = 0; j < 16; ++j) store_elem(a.fq, row * a.cols + b * 16 + j, a.fq_dt, q.fq[j]);
      }
    }
    const int64_t tile = h * (n_pad / TILE) + r / TILE;
    const int rr = static_cast<int>(r % TILE);
    const int D = static_cast<int>(a.cols);
    if (a.codes_t) {
      uint2* dst = reinterpret_cast<uint2*>(a.codes_t + tile * fp4_tile_bytes(D) + t8x32_off(rr, b * 16, TILE));
      *dst = make_uint2(q.packed[0], q.packed[1]);
    }
    if (a.sf_t) a.sf_t[tile * sf_tile_bytes_qk(D) + sf512_off(rr, static_cast<int>(b))] = static_cast<uint8_t>(q.scale);
    if (a.fqh_t) {
      uint8_t* base = reinterpret_cast<uint8_t*>(a.fqh_t) + tile * h_tile_bytes(D);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int col0 = static_cast<int>(b) * 16 + half * 8;
        uint4 w;
        w.x = h16_bits(q.fq[half * 8 + 0], a.fqh_dt) | (h16_bits(q.fq[half * 8 + 1], a.fqh_dt) << 16);
        w.y = h16_bits(q.fq[half * 8 + 2], a.fqh_dt) | (h16_bits(q.fq[half * 8 + 3], a.fqh_dt) << 16);
        w.z = h16_bits(q.fq[half * 8 + 4], a.fqh_dt) | (h16_bits(q.fq[half * 8 + 5], a.fqh_dt) << 16);
        w.w = h16_bits(q.fq[half * 8 + 6], a.fqh_dt) | (h16_bits(q.fq[half * 8 + 7], a.fqh_dt) << 16);
        *reinterpret_cast<uint4*>(base + t8x8_off(rr, col0)) = w;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2: blocks along the token axis (the V operand, quantized as V^T with the
// token tail zero-padded to a multiple of 16; codec.py:359-381). x is
// [heads][n][cols]. One thread per (column, 32-token group) = two blocks.
// Optional outputs:
//   codes_ref [heads][cols][n16/2], scales_ref [heads][cols][n16/16]  (n16 = ceil16(n))
//   fq        [heads][n][cols] dense (fake_quantize_cols)
//   codes_t   T8x32 V^T tiles: per (head, 128-token tile) a cols x 128 tile
//   sf_t      SF512 images (2 K-steps per tile)
//   fqh_t     T8x8 16-bit tiles [128 tokens][cols] of the dequantized V
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) quantize_cols_kernel(RowsArgs a) {
  const int64_t n16 = ceil_div(a.n, 16);
  const bool tiled = a.codes_t || a.sf_t || a.fqh_t;
  const int64_t ngroups = tiled ? ceil_div(a.n, TILE) * (TILE / 32) : ceil_div(a.n, 32);
  const int64_t total = a.heads * ngroups * a.cols;
  const int D = static_cast<int>(a.cols);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = t % a.cols;
    const int64_t g = (t / a.cols) % ngroups;
    const int64_t h = t / (a.cols * ngroups);
    const int64_t tok0 = g * 32;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t b0 = tok0 + half * 16;  // first token of this block
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t tok = b0 + j;
        v[j] = tok < a.n ? load_elem(a.x, h * a.hs + tok * a.ld + c, a.x_dt) : 0.f;
      }
      Block16 q;
      quantize_block16(v, q);
      const int64_t blk = b0 / 16;
      if (blk < n16) {
        if (!q.finite && a.nonfinite) atomicOr(a.nonfinite, 1);
        if (a.codes_ref) {
          uint2* dst = reinterpret_cast<uint2*>(a.codes_ref + (h * a.cols + c) * (n16 * 8) + blk * 8);
          *dst = make_uint2(q.packed[0], q.packed[1]);
        }
        if (a.scales_ref) a.scales_ref[(h * a.cols + c) * n16 + blk] = static_cast<uint8_t>(q.scale);
        if (a.fq) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (b0 + j < a.n) store_elem(a.fq, (h * a.n + b0 + j) * a.cols + c, a.fq_dt, q.fq[j]);
        }
      }
      if (tiled) {
        const int64_t n_tiles = ceil_div(a.n, TILE);
        const int64_t tile = h * n_tiles + b0 / TILE;
        const int kt = static_cast<int>(b0 % TILE);  // token index inside the tile
        if (a.codes_t) {
          uint2* dst =
              reinterpret_cast<uint2*>(a.codes_t + tile * fp4_tile_bytes(D) + t8x32_off(static_cast<int>(c), kt, D));
          *dst = make_uint2(q.packed[0], q.packed[1]);
        }
        if (a.sf_t) a.sf_t[tile * kSfTileBytesV + sf512_off(static_cast<int>(c), kt / 16)] = static_cast<uint8_t>(q.scale);
        if (a.fqh_t) {
          uint8_t* base = reinterpret_cast<uint8_t*>(a.fqh_t) + tile * h_tile_bytes(D);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            *reinterpret_cast<uint16_t*>(base + t8x8_off(kt + j, static_cast<int>(c))) =
                static_cast<uint16_t>(h16_bits(q.fq[j], a.fqh_dt));
        }
      }
    }
  }
}

// K3: reference-layout codes + scales -> dense values. rows x cols.
__global__ void __launch_bounds__(256) dequantize_kernel(const uint8_t* codes, const uint8_t* scales, int64_t rows,
                                                         int64_t cols, void* out, int out_dt) {
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
      store_elem(out, r * cols + b * 16 + j, out_dt, e2m1_to_f32(code) * s);
    }
  }
}

static int grid_for(int64_t work) {
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

cudaError_t launch_quantize_rows(const RowsArgs& a, cudaStream_t st) {
  const int64_t n_pad = (a.codes_t || a.sf_t || a.fqh_t) ? ceil_div(a.n, TILE) * TILE : a.n;
  quantize_rows_kernel<<<grid_for(a.heads * n_pad * (a.cols / 16)), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_quantize_cols(const RowsArgs& a, cudaStream_t st) {
  const bool tiled = a.codes_t || a.sf_t || a.fqh_t;
  const int64_t ngroups = tiled ? ceil_div(a.n, TILE) * (TILE / 32) : ceil_div(a.n, 32);
  quantize_cols_kernel<<<grid_for(a.heads * ngroups * a.cols), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                              int out_dt, cudaStream_t st) {
  dequantize_kernel<<<grid_for(rows * (cols / 16)), 256, 0, st>>>(codes, scales, rows, cols, out, out_dt);
  return cudaGetLastError();
}

}  // namespace aq
