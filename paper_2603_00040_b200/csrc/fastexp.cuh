// exp2 for the softmax warps, split across two pipes.
//
// The two-pass forward evaluates two exponentials per score; at one MUFU.EX2
// per element the SFU (16 lanes/clk/SM) alone would bound the kernel. A
// fraction of the elements instead goes through a degree-5 polynomial on the
// FMA pipe using packed fp32x2 math (sm_100 FFMA2 / FADD2):
//   2^x = 2^j * p(f),  j = rint(x) (magic-number add), f = x - j in [-0.5, 0.5]
//   p = minimax fit of 2^f, max relative error 2.2e-7 in fp32 Horner form
//   (ex2.approx.f32 is ~1.7e-7), exponent added with one integer shift-add.
// Inputs are clamped to >= -125 so the result stays a normal float (a masked
// -inf score gives 2^-125 instead of 0; callers that need exact zeros select).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace aq {

__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float2 magic = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 y = __fadd2_rn(x, magic);
  const float2 j = __fadd2_rn(y, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
  float2 p = make_float2(0.001326697412878275f, 0.001326697412878275f);
  p = __ffma2_rn(p, f, make_float2(0.009675459936261177f, 0.009675459936261177f));
  p = __ffma2_rn(p, f, make_float2(0.05550742521882057f, 0.05550742521882057f));
  p = __ffma2_rn(p, f, make_float2(0.24022121727466583f, 0.24022121727466583f));
  p = __ffma2_rn(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  // bits(y) = bits(magic) + j and bits(magic) << 23 == 0 (mod 2^32)
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(y.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(y.y) << 23)));
}

// exp2 of a pair: MUFU for both (kPoly == false) or the FMA-pipe polynomial.
template <bool kPoly>
__device__ __forceinline__ float2 ex2_pair(float2 t) {
  if (kPoly) return ex2_poly2(t);
  return make_float2(ex2(t.x), ex2(t.y));
}

// Which element pairs of a 16-pair group use the polynomial: pairs whose
// index mod 8 is < POLY_PAIRS_OF_8 (compile-time split of the exp work).
#ifndef AQ_POLY_PAIRS_OF_8
#define AQ_POLY_PAIRS_OF_8 2
#endif
__host__ __device__ constexpr bool use_poly(int pair) { return (pair & 7) < AQ_POLY_PAIRS_OF_8; }

// Pass-1 (exp-sum for L) split; independent of the pass-2 / backward split
// (P must match between forward and backward, L only between the two forward
// kernels, which share this code).
#ifndef AQ_POLY_P1_PAIRS_OF_8
#define AQ_POLY_P1_PAIRS_OF_8 1
#endif
__host__ __device__ constexpr bool use_poly_p1(int pair) { return (pair & 7) < AQ_POLY_P1_PAIRS_OF_8; }

}  // namespace aq
