// NVFP4 quantization of one 16-key block of softmax probabilities, shared by
// the forward (P^F codes feed the FP4 PV MMA) and the backward (P^F values
// feed the bf16 dV MMA) so both sides see bit-identical P^F -- the property
// test_flash.py:230-244 pins for the reference.
//   scale = E4M3_RNE(amax / 6), bumped to 2^-9 for tiny non-zero blocks
//           (codec.py:169-177); codes = E2M1_RNE(p / scale) (codec.py:196-202).
// P >= 0, so no sign / negative-zero handling is needed. p / scale uses the
// reciprocal of the (exactly representable) scale: P itself carries ~1e-7
// relative error from the exp, so this costs no parity.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace aq {

struct PBlock {
  uint32_t scale;     // E4M3 code
  uint32_t codes[2];  // 16 packed e2m1 codes, low nibble = lower key
  float sv;           // decoded scale
};

__device__ __forceinline__ PBlock quantize_p16(const float* p) {
  float amax = 0.f;
#pragma unroll
  for (int e = 0; e < 16; ++e) amax = fmaxf(amax, p[e]);
  uint32_t sc = cvt_e4m3(__fdiv_rn(amax, 6.0f));
  if (sc == 0 && amax > 0.f) sc = 1;
  PBlock b;
  b.scale = sc;
  b.sv = e4m3_to_f32(sc);
  const float rs = b.sv > 0.f ? __frcp_rn(b.sv) : 0.f;
  b.codes[0] = b.codes[1] = 0;
#pragma unroll
  for (int e = 0; e < 16; e += 2) b.codes[e >> 3] |= cvt_e2m1x2(p[e] * rs, p[e + 1] * rs) << (4 * (e & 7));
  return b;
}

// decoded value of code e (0..15) of a quantized block
__device__ __forceinline__ float pblock_value(const PBlock& b, int e) {
  return e2m1_to_f32((b.codes[e >> 3] >> (4 * (e & 7))) & 0xF) * b.sv;
}

}  // namespace aq
