// NVFP4 quantization of one 16-key block of softmax probabilities, shared by
// the forward (P^F codes feed the FP4 PV MMA) and the backward (P^F values
// feed the bf16 dV MMA) so both sides see bit-identical P^F -- the property
// test_flash.py:230-244 pins for the reference.
//   scale = E4M3_RNE(amax / 6), bumped to 2^-9 for tiny non-zero blocks
//           (codec.py:169-177); codes = E2M1_RNE(p / scale) (codec.py:196-202).
// P >= 0, so no sign / negative-zero handling is needed. amax / 6 and
// p / scale use multiplications by (approximate) reciprocals: P itself
// carries ~1e-7 relative error from the exp, so a 1-ulp difference only
// matters for values within an ulp of a rounding midpoint (rare, and the
// forward and backward still agree exactly because both run this code).
#pragma once
#include <cstdint>

#include "fastexp.cuh"
#include "ptx.cuh"

namespace aq {

struct PBlock {
  uint32_t scale;     // E4M3 code
  uint32_t codes[2];  // 16 packed e2m1 codes, low nibble = lower key
  float sv;           // decoded scale
};

__device__ __forceinline__ PBlock quantize_p16(const float* p) {
  float m0 = fmaxf(p[0], p[1]), m1 = fmaxf(p[2], p[3]), m2 = fmaxf(p[4], p[5]), m3 = fmaxf(p[6], p[7]);
  float m4 = fmaxf(p[8], p[9]), m5 = fmaxf(p[10], p[11]), m6 = fmaxf(p[12], p[13]), m7 = fmaxf(p[14], p[15]);
  const float amax = fmaxf(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)), fmaxf(fmaxf(m4, m5), fmaxf(m6, m7)));
  uint32_t sc = cvt_e4m3(amax * (1.0f / 6.0f));
  if (sc == 0 && amax > 0.f) sc = 1;
  PBlock b;
  b.scale = sc;
  b.sv = e4m3_to_f32_cvt(sc);
  const float rs = b.sv > 0.f ? rcp_approx(b.sv) : 0.f;
  float q[16];
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    const float2 v = __fmul2_rn(make_float2(p[e], p[e + 1]), make_float2(rs, rs));
    q[e] = v.x;
    q[e + 1] = v.y;
  }
  b.codes[0] = cvt_e2m1x8(q);
  b.codes[1] = cvt_e2m1x8(q + 8);
  return b;
}

// Two-level P (sage3.py:98-110): the block of P * r quantized without
// materializing P * r -- amax and 1/scale absorb the factor r (the clamp to
// 448*6 is implicit: both conversions saturate). amax = max of the block of P.
__device__ __forceinline__ PBlock quantize_p16_r(const float* p, float amax, float r) {
  const float am = amax * r;
  uint32_t sc = cvt_e4m3(am * (1.0f / 6.0f));
  if (sc == 0 && am > 0.f) sc = 1;
  PBlock b;
  b.scale = sc;
  b.sv = e4m3_to_f32_cvt(sc);
  const float rs = b.sv > 0.f ? rcp_approx(b.sv) * r : 0.f;
  float q[16];
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    const float2 v = __fmul2_rn(make_float2(p[e], p[e + 1]), make_float2(rs, rs));
    q[e] = v.x;
    q[e + 1] = v.y;
  }
  b.codes[0] = cvt_e2m1x8(q);
  b.codes[1] = cvt_e2m1x8(q + 8);
  return b;
}

// NVFP4 P block under a per-tensor P scale t_p (r = 1 / t_p): the block of
// P * r is quantized (two-level NVFP4: P^F = t_p * scale * code). r = 1 is the
// reference's semantics and gives exactly quantize_p16's bits (amax * 1 and
// rcp * 1 are exact), so the parity path is unchanged.
__device__ __forceinline__ PBlock quantize_p16_s(const float* p, float r) {
  float m0 = fmaxf(p[0], p[1]), m1 = fmaxf(p[2], p[3]), m2 = fmaxf(p[4], p[5]), m3 = fmaxf(p[6], p[7]);
  float m4 = fmaxf(p[8], p[9]), m5 = fmaxf(p[10], p[11]), m6 = fmaxf(p[12], p[13]), m7 = fmaxf(p[14], p[15]);
  const float amax = fmaxf(fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)), fmaxf(fmaxf(m4, m5), fmaxf(m6, m7)));
  return quantize_p16_r(p, amax, r);
}

// MXFP4 P block (32 keys, codec.py:123-203): UE8M0 scale = nearest power of
// two of amax / 6 with ties up (0 for a zero block), codes = E2M1_RNE(p / scale)
// with the exact power-of-two reciprocal. P >= 0.
__device__ __forceinline__ void quantize_p32_mx(const float* p, uint32_t (&codes)[4], uint32_t& sc) {
  float m0 = p[0], m1 = p[1];
#pragma unroll
  for (int e = 2; e < 32; e += 2) {
    m0 = fmaxf(m0, p[e]);
    m1 = fmaxf(m1, p[e + 1]);
  }
  const float amax = fmaxf(m0, m1);
  const float raw = div_rn(amax, 6.0f, 0.16666667163372039795f);
  sc = 0u;
  if (raw > 0.f) {
    const uint32_t bits = __float_as_uint(raw);
    const uint32_t be = bits >> 23;  // raw <= 1/6 < 2^127: no overflow, no clamp at 254
    if (be != 0) {
      sc = be + ((bits & 0x7FFFFFu) >= 0x400000u ? 1u : 0u);  // nearest power of two, ties up
    } else {  // subnormal raw (codec.py:123-136 through frexp)
      int e;
      const float m = frexpf(raw, &e);
      const int c = ((2.0f * m < 1.5f) ? e - 1 : e) + 127;
      sc = static_cast<uint32_t>(c < 0 ? 0 : c);
    }
  }
  const float rs = __int_as_float(static_cast<int>((254u - sc) << 23));
  float q[32];
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    const float2 v = __fmul2_rn(make_float2(p[e], p[e + 1]), make_float2(rs, rs));
    q[e] = v.x;
    q[e + 1] = v.y;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) codes[k] = cvt_e2m1x8(q + 8 * k);
}

// P = exp(S - L) for 2*NP consecutive in-tile key columns starting at column
// c0 (c0 % 16 == 0): t = S_raw * log2(e)/sqrt(d) - L2 (one FFMA2 per pair),
// exp2 split between MUFU and the FMA-pipe polynomial by in-tile pair index.
// Shared by forward pass 2 and the backward so both rebuild identical P.
template <int NP>
__device__ __forceinline__ void p_from_s(float* x, int c0, float sl2, float L2) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const float2 t = __ffma2_rn(make_float2(x[2 * i], x[2 * i + 1]), make_float2(sl2, sl2), make_float2(-L2, -L2));
    const float2 e = use_poly(c0 / 2 + i) ? ex2_pair<true>(t) : ex2_pair<false>(t);
    x[2 * i] = e.x;
    x[2 * i + 1] = e.y;
  }
}

// Exact pass-2 early-out. A 16-key block whose scores all satisfy
// S * sl2 - L2 <= -11.01 has P = exp2(S * sl2 - L2) <= 2^-11 for every key, for
// MUFU.EX2 and for the FMA-pipe polynomial alike (relative error <= 2.2e-7, so
// the 0.01 margin keeps P strictly below 2^-11). quantize_p16 then yields the
// bumped scale code 0x01 (amax / 6 < 2^-10 rounds to E4M3 zero, amax > 0 since
// every 16-key block holds one polynomial pair, which never returns 0) and
// P / 2^-9 <= 0.25 rounds to the even code 0 everywhere: the block's P^F is
// known without an exponential (codec.py:169-177, 196-202).
// p_skip_thr gives the per-row bound on the raw score, p_skip_mask bit b marks
// block b of this thread's columns as qualifying.
static_assert(AQ_POLY_PAIRS_OF_8 >= 1, "the early-out relies on one polynomial pair per 16-key block");
__device__ __forceinline__ float p_skip_thr(float L2, float sl2) {
  return (L2 - 11.02f - fabsf(L2) * 1e-6f) / sl2;
}
template <int NB>
__device__ __forceinline__ uint32_t p_skip_mask(const float* x, float thr) {
  uint32_t m = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const float* v = x + 16 * b;
    const float m0 = fmaxf(fmaxf(v[0], v[1]), v[2]), m1 = fmaxf(fmaxf(v[3], v[4]), v[5]);
    const float m2 = fmaxf(fmaxf(v[6], v[7]), v[8]), m3 = fmaxf(fmaxf(v[9], v[10]), v[11]);
    const float m4 = fmaxf(fmaxf(v[12], v[13]), v[14]);
    const float mx = fmaxf(fmaxf(fmaxf(m0, m1), m2), fmaxf(fmaxf(m3, m4), v[15]));
    m |= (mx <= thr ? 1u : 0u) << b;
  }
  return m;
}

// decoded value of code e (0..15) of a quantized block
__device__ __forceinline__ float pblock_value(const PBlock& b, int e) {
  return e2m1_to_f32((b.codes[e >> 3] >> (4 * (e & 7))) & 0xF) * b.sv;
}

}  // namespace aq
