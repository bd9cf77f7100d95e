// SageAttention3-style toggles (attnqat/sage3.py): the high-precision
// pre-processing around the FP4 attention kernel. All HBM-bound elementwise
// and reduction work on [heads][n][d] operands:
//   means   q_bar = per-b_q-tile token mean of Q, k_bar = token mean of K,
//           accumulated in fp64 like the reference (sage3.py:45-60);
//   center  gamma = x - mean, rounded once to fp32 (the quantizer input);
//   delta   q_bar_t gamma_k^T per (query tile, key): the score term that
//           never goes through FP4 (sage3.py:74-88);
//   bias    q_bar_t k_bar + gamma_q k_bar per row (sage3.py:84-87).
// delta and bias accumulate left to right in fp32 with separate multiply and
// add, the reference matmul's order (tensors.py:32-51), so they reproduce its
// bits from the same fp32 operands.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "attn.h"
#include "layouts.cuh"

namespace aq {
namespace sage {

__device__ __forceinline__ double load_d(const void* p, int64_t i, int dt) {
  if (dt == 1) return static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]));
  if (dt == 2) return static_cast<double>(__half2float(reinterpret_cast<const __half*>(p)[i]));
  return static_cast<double>(reinterpret_cast<const float*>(p)[i]);
}

// one CTA per (head, chunk of `chunk` rows): column sums of the chunk
__global__ void __launch_bounds__(256) sums_kernel(const void* x, int dt, int64_t n, int d, int64_t chunk,
                                                   double* sums) {
  __shared__ double part[256];
  const int64_t nch = n / chunk;
  const int64_t h = blockIdx.x / nch, s = blockIdx.x % nch;
  const int phases = 256 / d;
  const int c = threadIdx.x % d, ph = threadIdx.x / d;
  double acc = 0.0;
  const int64_t base = (h * n + s * chunk) * d + c;
#pragma unroll 8
  for (int64_t r = ph; r < chunk; r += phases) acc += load_d(x, base + r * d, dt);
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < d) {
    double t = 0.0;
    for (int q = 0; q < phases; ++q) t += part[q * d + threadIdx.x];
    sums[(h * nch + s) * d + threadIdx.x] = t;
  }
}

// means of segments of `per` consecutive chunks
__global__ void __launch_bounds__(256) finish_means_kernel(const double* sums, int64_t segs, int64_t per, int d,
                                                           double inv, double* mean) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= segs * d) return;
  const int64_t s = i / d, c = i % d;
  double t = 0.0;
  for (int64_t k = 0; k < per; ++k) t += sums[(s * per + k) * d + c];
  mean[i] = t * inv;
}

// gamma = x - mean (fp64), rounded once to fp32; 4 columns per thread
template <int D>
__global__ void __launch_bounds__(256) center_kernel(const void* x, int dt, int64_t heads, int64_t n, int64_t seg,
                                                     const double* mean, float* gamma) {
  const int64_t total4 = heads * n * (D / 4);
  const int64_t nseg = mean ? n / seg : 1;
  for (int64_t i4 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i4 < total4;
       i4 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rg = i4 / (D / 4);  // global row (head * n + row)
    const int c = static_cast<int>(i4 % (D / 4)) * 4;
    const double* mrow = nullptr;
    if (mean) {
      const int64_t h = rg / n;
      mrow = mean + (h * nseg + (rg - h * n) / seg) * D + c;
    }
    float4 o;
    float* of = reinterpret_cast<float*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double v = load_d(x, rg * D + c + e, dt);
      of[e] = static_cast<float>(mrow ? v - mrow[e] : v);
    }
    reinterpret_cast<float4*>(gamma)[i4] = o;
  }
}

// CTA = (head, 128 keys), thread = key j; q_bar rows staged 32 at a time in
// shared memory, four query tiles per step (independent accumulators)
template <int D>
__global__ void __launch_bounds__(128) delta_kernel(const double* q_bar, const float* gamma_k, int64_t t_q,
                                                    int64_t n_k, int64_t kpad, float* delta) {
  __shared__ __align__(16) float qs[32][D];
  const int64_t h = blockIdx.x;
  const int64_t j = static_cast<int64_t>(blockIdx.y) * TILE + threadIdx.x;
  float g[D];
#pragma unroll
  for (int c = 0; c < D; c += 4) {
    const float4 v = j < n_k ? *reinterpret_cast<const float4*>(gamma_k + (h * n_k + j) * D + c)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    g[c] = v.x;
    g[c + 1] = v.y;
    g[c + 2] = v.z;
    g[c + 3] = v.w;
  }
  for (int64_t t0 = 0; t0 < t_q; t0 += 32) {
    const int nt = static_cast<int>(t_q - t0 < 32 ? t_q - t0 : 32);
    __syncthreads();
    for (int i = threadIdx.x; i < nt * D; i += blockDim.x)
      qs[i / D][i % D] = static_cast<float>(q_bar[(h * t_q + t0) * D + i]);
    __syncthreads();
    for (int t = 0; t < nt; t += 4) {
      // scalar __fmul_rn / __fadd_rn: never contracted (ptxas fuses packed
      // fp32x2 multiply + add into FFMA2 even with .rn and -fmad=false)
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      const int t1 = t + 1 < nt ? t + 1 : t, t2 = t + 2 < nt ? t + 2 : t, t3 = t + 3 < nt ? t + 3 : t;
#pragma unroll
      for (int c = 0; c < D; c += 4) {
        const float4 q0 = *reinterpret_cast<const float4*>(&qs[t][c]);
        const float4 q1 = *reinterpret_cast<const float4*>(&qs[t1][c]);
        const float4 q2 = *reinterpret_cast<const float4*>(&qs[t2][c]);
        const float4 q3 = *reinterpret_cast<const float4*>(&qs[t3][c]);
        const float* f0 = reinterpret_cast<const float*>(&q0);
        const float* f1 = reinterpret_cast<const float*>(&q1);
        const float* f2 = reinterpret_cast<const float*>(&q2);
        const float* f3 = reinterpret_cast<const float*>(&q3);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          a0 = __fadd_rn(a0, __fmul_rn(f0[e], g[c + e]));
          a1 = __fadd_rn(a1, __fmul_rn(f1[e], g[c + e]));
          a2 = __fadd_rn(a2, __fmul_rn(f2[e], g[c + e]));
          a3 = __fadd_rn(a3, __fmul_rn(f3[e], g[c + e]));
        }
      }
      float* drow = delta + (h * t_q + t0 + t) * kpad + j;
      const bool ok = j < n_k;
      drow[0] = ok ? a0 : 0.f;
      if (t + 1 < nt) drow[kpad] = ok ? a1 : 0.f;
      if (t + 2 < nt) drow[2 * kpad] = ok ? a2 : 0.f;
      if (t + 3 < nt) drow[3 * kpad] = ok ? a3 : 0.f;
    }
  }
}

// CTA = 128 rows of one head, thread = row; gamma_q staged 32 columns at a
// time (coalesced) so each thread runs its row's dot product in column order
template <int D>
__global__ void __launch_bounds__(128) bias_kernel(const double* q_bar, const double* k_bar, const float* gamma_q,
                                                   int64_t n_q, int64_t b_q, float* bias) {
  __shared__ float gs[128][33];
  __shared__ float kb[D];
  const int64_t h = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 128;
  const int64_t row = r0 + threadIdx.x;
  for (int c = threadIdx.x; c < D; c += blockDim.x) kb[c] = static_cast<float>(k_bar[h * D + c]);
  float a1 = 0.f, a2 = 0.f;
  for (int c0 = 0; c0 < D; c0 += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
      const int rr = i / 32, cc = i % 32;
      gs[rr][cc] = r0 + rr < n_q ? gamma_q[(h * n_q + r0 + rr) * D + c0 + cc] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < 32; ++cc) a2 = __fadd_rn(a2, __fmul_rn(gs[threadIdx.x][cc], kb[c0 + cc]));
  }
  if (row >= n_q) return;
  if (q_bar) {
    const double* qb = q_bar + (h * (n_q / b_q) + row / b_q) * D;
#pragma unroll 8
    for (int c = 0; c < D; ++c) a1 = __fadd_rn(a1, __fmul_rn(static_cast<float>(qb[c]), kb[c]));
  }
  bias[h * n_q + row] = __fadd_rn(a1, a2);
}

int grid_for(int64_t n) {
  const int64_t b = ceil_div(n, 256);
  return static_cast<int>(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace sage

cudaError_t launch_sage_means(const void* x, int x_dt, int64_t heads, int64_t n, int d, int64_t seg,
                              double* scratch, double* mean, cudaStream_t st) {
  // column sums over chunks of rows (sage_chunk_rows(seg) divides seg) spread
  // a long segment (the whole of K) over many CTAs; the means then add the
  // chunk sums of each segment in order
  if (d <= 0 || 256 % d || seg <= 0 || n % seg) return cudaErrorInvalidValue;
  const int64_t chunk = sage_chunk_rows(seg);
  sage::sums_kernel<<<static_cast<unsigned>(heads * (n / chunk)), 256, 0, st>>>(x, x_dt, n, d, chunk, scratch);
  if (cudaGetLastError() != cudaSuccess) return cudaErrorLaunchFailure;
  const int64_t m = heads * (n / seg) * d;
  sage::finish_means_kernel<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, st>>>(
      scratch, heads * (n / seg), seg / chunk, d, 1.0 / static_cast<double>(seg), mean);
  return cudaGetLastError();
}

cudaError_t launch_sage_center(const void* x, int x_dt, int64_t heads, int64_t n, int d, int64_t seg,
                               const double* mean, float* gamma, cudaStream_t st) {
  const int g = sage::grid_for(heads * n * d / 4);
  if (d == 64) sage::center_kernel<64><<<g, 256, 0, st>>>(x, x_dt, heads, n, seg, mean, gamma);
  else if (d == 128) sage::center_kernel<128><<<g, 256, 0, st>>>(x, x_dt, heads, n, seg, mean, gamma);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_sage_delta(const double* q_bar, const float* gamma_k, int64_t heads, int64_t t_q, int64_t n_k,
                              int d, int64_t kpad, float* delta, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>(heads), static_cast<unsigned>(kpad / TILE));
  if (d == 64) sage::delta_kernel<64><<<grid, 128, 0, st>>>(q_bar, gamma_k, t_q, n_k, kpad, delta);
  else if (d == 128) sage::delta_kernel<128><<<grid, 128, 0, st>>>(q_bar, gamma_k, t_q, n_k, kpad, delta);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_sage_bias(const double* q_bar, const double* k_bar, const float* gamma_q, int64_t heads,
                             int64_t n_q, int d, int64_t b_q, float* bias, cudaStream_t st) {
  const dim3 g(static_cast<unsigned>(ceil_div(n_q, 128)), static_cast<unsigned>(heads));
  if (d == 64) sage::bias_kernel<64><<<g, 128, 0, st>>>(q_bar, k_bar, gamma_q, n_q, b_q, bias);
  else if (d == 128) sage::bias_kernel<128><<<g, 128, 0, st>>>(q_bar, k_bar, gamma_q, n_q, b_q, bias);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace aq
