// HBM layouts shared by the quantizers (producers) and the attention kernels
// (consumers). The attention kernels move whole 128-token tiles with single
// 1-D bulk copies, so every per-tile operand is stored in HBM already in the
// exact shared-memory image the tcgen05 descriptors expect:
//
//  * FP4 operand tile ("T8x32"): rows x K packed e2m1, no swizzle. 8-row x
//    16-byte core matrices (8 rows x 32 codes). Core (row/8, k/32) lives at
//    (k/32)*KCHUNK + (row/8)*128, row r%8 at +16*(r%8). KCHUNK = rows*16.
//    Used for Q and K (rows = tokens, K = d) and V^T (rows = d, K = tokens).
//  * Scale-factor tile ("SF512"): per 64-wide K step, a 512-byte image for
//    tcgen05.cp.32x128b.warpx4: byte (r%32)*16 + (r/32)*4 + (k/16)%4.
//  * 16-bit operand tile ("T8x8"): [tokens][d] 128 x D elements, core
//    (tok/8, col/8) at (col/8)*2048 + (tok/8)*128, within core (tok%8)*16 +
//    (col%8)*2. Usable as a K-major operand (K = col) or an MN-major operand
//    (MN = col) by choosing LBO/SBO in the descriptor.
#pragma once
#include <cstdint>

namespace aq {

constexpr int TILE = 128;  // tokens per attention tile (M of every MMA)

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// bytes of one FP4 token tile with D columns (Q/K) or one V^T tile (D rows x 128 tokens)
__host__ __device__ __forceinline__ int64_t fp4_tile_bytes(int D) { return static_cast<int64_t>(TILE) * D / 2; }
// bytes of the SF images of one Q/K tile (D/64 K-steps) or one V^T tile (2 K-steps)
__host__ __device__ __forceinline__ int64_t sf_tile_bytes_qk(int D) { return (D / 64) * 512; }
constexpr int64_t kSfTileBytesV = 2 * 512;
// bytes of one 16-bit T8x8 tile
__host__ __device__ __forceinline__ int64_t h_tile_bytes(int D) { return static_cast<int64_t>(TILE) * D * 2; }

// byte offset of the 8 codes (16 consecutive K) of row `r` starting at K index `k` (k % 16 == 0)
// inside a T8x32 tile with `rows` rows.
__host__ __device__ __forceinline__ uint32_t t8x32_off(int r, int k, int rows) {
  return static_cast<uint32_t>((k >> 5) * (rows * 16) + (r >> 3) * 128 + (r & 7) * 16 + ((k & 31) >> 1));
}
// byte offset of the scale of row r, K-block kb (16 elements) inside an SF512 sequence.
__host__ __device__ __forceinline__ uint32_t sf512_off(int r, int kb) {
  return static_cast<uint32_t>((kb >> 2) * 512 + (r & 31) * 16 + (r >> 5) * 4 + (kb & 3));
}
// byte offset of element (tok, col) inside a T8x8 16-bit tile.
__host__ __device__ __forceinline__ uint32_t t8x8_off(int tok, int col) {
  return static_cast<uint32_t>((col >> 3) * 2048 + (tok >> 3) * 128 + (tok & 7) * 16 + (col & 7) * 2);
}

}  // namespace aq
