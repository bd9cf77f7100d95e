// Epilogue row stores through shared memory (sm_100a).
//
// The attention kernels hold their outputs one row per thread (TMEM lane ==
// row): lane l of a warp has N consecutive columns of row r0 + l. Stored
// directly, every warp instruction touches 32 rows (32 separate lines); at
// 128 x 128 outputs per item that kept the LSU busy for thousands of cycles
// per item (K4 at 1 K keys: ~1000 cycles per warp-tile, a fifth of the
// kernel). Here a warp stages its 32 row segments in a private shared-memory
// buffer -- 16-byte chunks XOR-swizzled by row, conflict-free for the writes
// (8 rows per phase, distinct chunks) and for the reads (one row per phase)
// -- and writes them back 32 / nch rows per instruction with contiguous,
// full-line row segments. K4 (persistent: its next item waits on these
// stores): 2.16 -> 2.11 ms at C4, 1.61 -> 1.52 ms at 1 K keys. K7's
// non-persistent CTAs retire while direct stores drain, and staging its
// dK / dV / dQ there made the backward 7 % slower, so K7 keeps store_row's
// direct form.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace aq {

// v: this lane's N values (row r0 + lane), written as dt (0 fp32, 1 bf16,
// 2 fp16) times mul. stg: the warp's buffer, 32 * N * 4 bytes, 16-byte
// aligned, not touched by anyone else until this returns. dst0: byte address
// of row r0's segment; stride: bytes between consecutive rows; rows: how many
// of the 32 rows exist (ragged tails). N * element size must be a multiple of 16.
template <int N>
__device__ __forceinline__ void warp_store_rows(uint8_t* stg, int lane, const float* v, float mul, int dt,
                                                uint8_t* dst0, int64_t stride, int rows) {
  const int nch = dt == 0 ? N / 4 : N / 8;  // 16-byte chunks per row segment
  const int rb = nch * 16;
  const int sw = (nch < 8 ? nch : 8) - 1;   // swizzle within the row's chunks
  uint8_t* mine = stg + lane * rb;
  if (dt == 0) {
#pragma unroll
    for (int c = 0; c < N / 4; ++c)
      *reinterpret_cast<uint4*>(mine + ((c ^ (lane & sw)) * 16)) =
          make_uint4(__float_as_uint(v[4 * c] * mul), __float_as_uint(v[4 * c + 1] * mul),
                     __float_as_uint(v[4 * c + 2] * mul), __float_as_uint(v[4 * c + 3] * mul));
  } else {
#pragma unroll
    for (int c = 0; c < N / 8; ++c) {
      uint32_t h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = v[8 * c + 2 * q] * mul, b = v[8 * c + 2 * q + 1] * mul;
        if (dt == 1) {
          const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
          h[q] = *reinterpret_cast<const uint32_t*>(&t);
        } else {
          const __half2 t = __floats2half2_rn(a, b);
          h[q] = *reinterpret_cast<const uint32_t*>(&t);
        }
      }
      *reinterpret_cast<uint4*>(mine + ((c ^ (lane & sw)) * 16)) = make_uint4(h[0], h[1], h[2], h[3]);
    }
  }
  __syncwarp();
  const int rpi = 32 / nch;  // rows per warp instruction
  const int rsub = lane / nch, cc = lane % nch;
  for (int r0 = 0; r0 < 32; r0 += rpi) {
    const int rr = r0 + rsub;
    const uint4 t = *reinterpret_cast<const uint4*>(stg + rr * rb + ((cc ^ (rr & sw)) * 16));
    if (rr < rows) *reinterpret_cast<uint4*>(dst0 + rr * stride + cc * 16) = t;
  }
  __syncwarp();
}

// The direct form (one lane, one row segment), for kernels without idle
// shared memory at the epilogue.
template <int N>
__device__ __forceinline__ void store_row(uint8_t* dst, const float* v, float mul, int dt) {
  if (dt == 0) {
#pragma unroll
    for (int c = 0; c < N / 4; ++c)
      reinterpret_cast<float4*>(dst)[c] = make_float4(v[4 * c] * mul, v[4 * c + 1] * mul, v[4 * c + 2] * mul, v[4 * c + 3] * mul);
  } else {
#pragma unroll
    for (int c = 0; c < N / 8; ++c) {
      uint32_t h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = v[8 * c + 2 * q] * mul, b = v[8 * c + 2 * q + 1] * mul;
        if (dt == 1) {
          const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
          h[q] = *reinterpret_cast<const uint32_t*>(&t);
        } else {
          const __half2 t = __floats2half2_rn(a, b);
          h[q] = *reinterpret_cast<const uint32_t*>(&t);
        }
      }
      reinterpret_cast<uint4*>(dst)[c] = make_uint4(h[0], h[1], h[2], h[3]);
    }
  }
}

}  // namespace aq
