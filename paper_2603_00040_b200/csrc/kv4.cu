// FP4 KV cache: K and V^T already quantized in the reference's QuantTensor
// layout (codec.py:260-299; the ATQ4 payload of tensors.py:173-188) are
// re-laid into the attention kernels' tile images (layouts.cuh) without
// touching a single value, so attention over a stored 4-bit KV cache gives
// the same bits as attention over the K / V it was quantized from.
//
//   K   : codes [heads][n][d/2], scales [heads][n][d/16]      (quantize(K))
//   V^T : codes [heads][d][n16/2], scales [heads][d][n16/16]  (quantize_padded(V.T))
//
// Pure byte movement (HBM-bound): one thread per 16-element block moves its 8
// code bytes and 1 scale byte; tile padding (rows / tokens past n) is zero,
// exactly what the quantizers write for zero-padded operands.
#include <cstdint>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"

namespace aq {
namespace {

__global__ void __launch_bounds__(256) pack_k_tiles(const uint8_t* __restrict__ codes,
                                                     const uint8_t* __restrict__ scales, int64_t heads, int64_t n,
                                                     int d, uint8_t* __restrict__ codes_t, uint8_t* __restrict__ sf_t) {
  const int nb = d / 16;
  const int64_t tiles = ceil_div(n, TILE);
  const int64_t total = heads * tiles * TILE * nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(t % nb);
    const int64_t rp = t / nb;                     // padded row over all heads
    const int64_t h = rp / (tiles * TILE);
    const int64_t r = rp % (tiles * TILE);
    const int64_t tile = h * tiles + r / TILE;
    const int rr = static_cast<int>(r % TILE);
    uint2 c = make_uint2(0u, 0u);
    uint8_t s = 0;
    if (r < n) {
      const int64_t row = h * n + r;
      c = *reinterpret_cast<const uint2*>(codes + row * (d / 2) + b * 8);
      s = scales[row * nb + b];
    }
    *reinterpret_cast<uint2*>(codes_t + tile * fp4_tile_bytes(d) + t8x32_off(rr, b * 16, TILE)) = c;
    sf_t[tile * sf_tile_bytes_qk(d) + sf512_off(rr, b)] = s;
  }
}

__global__ void __launch_bounds__(256) pack_vt_tiles(const uint8_t* __restrict__ codes,
                                                      const uint8_t* __restrict__ scales, int64_t heads, int64_t n,
                                                      int d, uint8_t* __restrict__ codes_t, uint8_t* __restrict__ sf_t) {
  const int64_t n16 = ceil_div(n, 16) * 16;
  const int64_t tiles = ceil_div(n, TILE);
  constexpr int kBlocks = TILE / 16;               // token blocks per tile
  const int64_t total = heads * tiles * d * kBlocks;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(t % kBlocks);
    const int64_t rest = t / kBlocks;
    const int c = static_cast<int>(rest % d);      // V^T row = head-dim column
    const int64_t ht = rest / d;                   // (head, tile)
    const int64_t h = ht / tiles;
    const int64_t kt = ht % tiles;
    const int64_t tok = kt * TILE + b * 16;
    uint2 v = make_uint2(0u, 0u);
    uint8_t s = 0;
    if (tok < n16) {
      const int64_t row = h * d + c;
      v = *reinterpret_cast<const uint2*>(codes + row * (n16 / 2) + tok / 2);
      s = scales[row * (n16 / 16) + tok / 16];
    }
    *reinterpret_cast<uint2*>(codes_t + ht * fp4_tile_bytes(d) + t8x32_off(c, b * 16, d)) = v;
    sf_t[ht * kSfTileBytesV + sf512_off(c, b)] = s;
  }
}

int grid_for(int64_t work) {
  int64_t g = ceil_div(work, 256);
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_pack_kv4(const uint8_t* k_codes, const uint8_t* k_scales, const uint8_t* vt_codes,
                            const uint8_t* vt_scales, int64_t heads, int64_t n, int d, uint8_t* k_codes_t,
                            uint8_t* k_sf_t, uint8_t* v_codes_t, uint8_t* v_sf_t, cudaStream_t st) {
  const int64_t tiles = ceil_div(n, TILE);
  pack_k_tiles<<<grid_for(heads * tiles * TILE * (d / 16)), 256, 0, st>>>(k_codes, k_scales, heads, n, d, k_codes_t,
                                                                          k_sf_t);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pack_vt_tiles<<<grid_for(heads * tiles * d * (TILE / 16)), 256, 0, st>>>(vt_codes, vt_scales, heads, n, d,
                                                                            v_codes_t, v_sf_t);
  return cudaGetLastError();
}

}  // namespace aq
