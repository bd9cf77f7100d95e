// C-ABI entry points (include/attnqat_b200.h). Validates arguments the way the
// reference does (ShapeError / TileError / MissingOPrime), carves the
// caller-owned workspace, and launches the quantizers + attention kernels on
// the caller's stream. No host synchronisation, no device allocation.
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/attnqat_b200.h"
#include "attn.h"
#include "layouts.cuh"

using namespace aq;

namespace {

constexpr int kAbiVersion = 3;

int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

struct FwdWs {
  int64_t q_codes, q_sf, k_codes, k_sf, v_codes, v_sf, v_h16, q_hb, k_hb, v_hb, sched, total;
};

FwdWs fwd_ws(int64_t heads, int64_t n_q, int64_t n_k, int64_t d, int train, int keep) {
  const int64_t qt = ceil_div(n_q, TILE), kt = ceil_div(n_k, TILE);
  FwdWs w{};
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += align256(bytes);
    return o;
  };
  w.q_codes = take(heads * qt * fp4_tile_bytes(static_cast<int>(d)));
  w.q_sf = take(heads * qt * sf_tile_bytes_qk(static_cast<int>(d)));
  w.k_codes = take(heads * kt * fp4_tile_bytes(static_cast<int>(d)));
  w.k_sf = take(heads * kt * sf_tile_bytes_qk(static_cast<int>(d)));
  w.v_codes = take(heads * kt * fp4_tile_bytes(static_cast<int>(d)));
  w.v_sf = take(heads * kt * kSfTileBytesV);
  // fp16 V^F tiles feed the O' MMA; a kept workspace always carries them so the
  // layout does not depend on the forward mode
  w.v_h16 = (train || keep) ? take(heads * kt * h_tile_bytes(static_cast<int>(d))) : -1;
  w.q_hb = keep ? take(heads * qt * h_tile_bytes(static_cast<int>(d))) : -1;
  w.k_hb = keep ? take(heads * kt * h_tile_bytes(static_cast<int>(d))) : -1;
  w.v_hb = keep ? take(heads * kt * h_tile_bytes(static_cast<int>(d))) : -1;
  w.sched = take(256);  // the training kernel's item counter
  w.total = off;
  return w;
}

struct BwdWs {
  int64_t fwd, do_h, delta, total;
};

BwdWs bwd_ws(int64_t heads, int64_t n_q, int64_t n_k, int64_t d) {
  BwdWs w{};
  const FwdWs f = fwd_ws(heads, n_q, n_k, d, 0, 1);
  const int64_t qt = ceil_div(n_q, TILE);
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += align256(bytes);
    return o;
  };
  w.fwd = take(f.total);  // re-quantized operands when no forward workspace is given
  w.do_h = take(heads * qt * h_tile_bytes(static_cast<int>(d)));
  w.delta = take(heads * qt * TILE * 4);
  w.total = off;
  return w;
}

bool dtype_ok(int dt) { return dt == 0 || dt == 1 || dt == 2; }

int cuda_status(cudaError_t e) { return e == cudaSuccess ? AQ_OK : AQ_E_CUDA; }

// Per-tensor FP32 scales of the two-level NVFP4 format (0 = 1.0, the
// reference's semantics) and the softmax scale (0 = 1/sqrt(d), flash.py:207).
struct TScales {
  float q = 1.f, k = 1.f, v = 1.f, p = 1.f;
  double sm = 0.0;  // 0: default 1/sqrt(d)
};

bool take_scale(float x, float& out) {
  if (x == 0.f) return true;  // keep 1.0
  if (!(x > 0.f) || !std::isfinite(x)) return false;
  out = x;
  return true;
}

template <typename Args>
bool read_scales(const Args* a, TScales& t) {
  if (!take_scale(a->q_scale, t.q) || !take_scale(a->k_scale, t.k) || !take_scale(a->v_scale, t.v) ||
      !take_scale(a->p_scale, t.p))
    return false;
  if (a->softmax_scale != 0.f) {
    if (!(a->softmax_scale > 0.f) || !std::isfinite(a->softmax_scale)) return false;
    t.sm = a->softmax_scale;
  }
  return true;
}

// log2(e) * softmax scale * t_q * t_k; the default expression is the one the
// kernels were validated with (bit-identical L / P at unit scales)
float scale_log2_of(const TScales& t, int64_t d) {
  const double base = t.sm == 0.0 ? 1.4426950408889634 / std::sqrt(static_cast<double>(d)) : 1.4426950408889634 * t.sm;
  return static_cast<float>(base * static_cast<double>(t.q) * static_cast<double>(t.k));
}

void apply_fwd_scales(FwdParams& p, const TScales& t, int64_t d) {
  p.scale_log2 = scale_log2_of(t, d);
  p.o_mul = t.v * t.p;
  p.ohp_mul = t.v;
  p.p_r = 1.f / t.p;
  p.p_lshift = std::log2(t.p);
}

// Stage Q/K/V into the attention layouts (K1/K2 in tiled mode).
int stage_operands(const void* q, const void* k, const void* v, int in_dt, int64_t heads, int64_t n_q, int64_t n_k,
                   int64_t d, uint8_t* ws, const FwdWs& w, cudaStream_t st, const TScales& ts = TScales{},
                   int* nonfinite = nullptr) {
  RowsArgs a{};
  a.x_dt = in_dt;
  a.nonfinite = nonfinite;
  a.inv_ts = 1.f / ts.q;
  a.heads = heads;
  a.cols = d;
  a.ld = d;
  // Q
  a.x = q;
  a.n = n_q;
  a.hs = n_q * d;
  a.codes_t = ws + w.q_codes;
  a.sf_t = ws + w.q_sf;
  a.fqh_t = w.q_hb >= 0 ? ws + w.q_hb : nullptr;
  a.fqh_dt = 1;
  cudaError_t e = launch_quantize_rows(a, st);
  if (e != cudaSuccess) return AQ_E_CUDA;
  // K
  a.inv_ts = 1.f / ts.k;
  a.x = k;
  a.n = n_k;
  a.hs = n_k * d;
  a.codes_t = ws + w.k_codes;
  a.sf_t = ws + w.k_sf;
  a.fqh_t = w.k_hb >= 0 ? ws + w.k_hb : nullptr;
  e = launch_quantize_rows(a, st);
  if (e != cudaSuccess) return AQ_E_CUDA;
  // V (blocks along tokens): fp16 tiles for the O' MMA, bf16 tiles for the backward
  a.inv_ts = 1.f / ts.v;
  a.x = v;
  a.codes_t = ws + w.v_codes;
  a.sf_t = ws + w.v_sf;
  a.fqh_t = w.v_h16 >= 0 ? ws + w.v_h16 : nullptr;
  a.fqh_dt = 2;
  a.fqh2_t = w.v_hb >= 0 ? ws + w.v_hb : nullptr;
  a.fqh2_dt = 1;
  e = launch_quantize_cols(a, st);
  if (e != cudaSuccess) return AQ_E_CUDA;
  return AQ_OK;
}

}  // namespace

extern "C" {

int aq_abi_version(void) { return kAbiVersion; }

const char* aq_status_string(int s) {
  switch (s) {
    case AQ_OK: return "ok";
    case AQ_E_SHAPE: return "shape error";
    case AQ_E_TILE: return "tile error";
    case AQ_E_INVALID: return "invalid value";
    case AQ_E_MISSING_OPRIME: return "missing O_prime";
    case AQ_E_CUDA: return "CUDA error";
    case AQ_E_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

int aq_quantize_rows(const void* x, int x_dtype, int64_t heads, int64_t n, int64_t cols, int64_t ld, int64_t hs,
                     uint8_t* codes, uint8_t* scales, void* fq, int fq_dtype, float tensor_scale, int* nonfinite,
                     void* stream) {
  if (!x || !dtype_ok(x_dtype) || (fq && !dtype_ok(fq_dtype))) return AQ_E_INVALID;
  float ts = 1.f;
  if (!take_scale(tensor_scale, ts)) return AQ_E_INVALID;
  if (heads < 0 || n < 0 || cols <= 0 || cols % 16 || ld < cols) return AQ_E_SHAPE;
  if (heads == 0 || n == 0) return AQ_OK;
  RowsArgs a{};
  a.x = x;
  a.x_dt = x_dtype;
  a.heads = heads;
  a.n = n;
  a.cols = cols;
  a.ld = ld;
  a.hs = hs;
  a.codes_ref = codes;
  a.scales_ref = scales;
  a.fq = fq;
  a.fq_dt = fq_dtype;
  a.nonfinite = nonfinite;
  a.ts = ts;
  a.inv_ts = 1.f / ts;
  return cuda_status(launch_quantize_rows(a, static_cast<cudaStream_t>(stream)));
}

int aq_quantize_cols(const void* x, int x_dtype, int64_t heads, int64_t n, int64_t cols, int64_t ld, int64_t hs,
                     uint8_t* codes, uint8_t* scales, void* fq, int fq_dtype, float tensor_scale, int* nonfinite,
                     void* stream) {
  if (!x || !dtype_ok(x_dtype) || (fq && !dtype_ok(fq_dtype))) return AQ_E_INVALID;
  float ts = 1.f;
  if (!take_scale(tensor_scale, ts)) return AQ_E_INVALID;
  if (heads < 0 || n < 0 || cols <= 0 || ld < cols) return AQ_E_SHAPE;
  if (heads == 0 || n == 0) return AQ_OK;
  RowsArgs a{};
  a.x = x;
  a.x_dt = x_dtype;
  a.heads = heads;
  a.n = n;
  a.cols = cols;
  a.ld = ld;
  a.hs = hs;
  a.codes_ref = codes;
  a.scales_ref = scales;
  a.fq = fq;
  a.fq_dt = fq_dtype;
  a.nonfinite = nonfinite;
  a.ts = ts;
  a.inv_ts = 1.f / ts;
  return cuda_status(launch_quantize_cols(a, static_cast<cudaStream_t>(stream)));
}

int aq_round_codes(const void* x, int x_dtype, int64_t n, int format, uint8_t* codes, int* invalid, void* stream) {
  if (!x || !codes || (x_dtype != 0 && x_dtype != 3) || (format != 0 && format != 1)) return AQ_E_INVALID;
  if (n < 0) return AQ_E_SHAPE;
  if (n == 0) return AQ_OK;
  return cuda_status(launch_round_codes(x, x_dtype == 3, n, format, codes, invalid, static_cast<cudaStream_t>(stream)));
}

int aq_quantize_mx(const void* x, int x_dtype, int64_t rows, int64_t cols, uint8_t* codes, uint8_t* scales,
                   void* fq, int fq_dtype, int* nonfinite, void* stream) {
  if (!x || !dtype_ok(x_dtype) || (fq && !dtype_ok(fq_dtype))) return AQ_E_INVALID;
  if (rows < 0 || cols <= 0 || cols % 32) return AQ_E_SHAPE;
  if (rows == 0) return AQ_OK;
  return cuda_status(launch_quantize_mx(x, x_dtype, rows, cols, codes, scales, fq, fq_dtype, nonfinite,
                                        static_cast<cudaStream_t>(stream)));
}

int aq_dequantize_mx(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                     int out_dtype, void* stream) {
  if (!codes || !scales || !out || !dtype_ok(out_dtype)) return AQ_E_INVALID;
  if (rows < 0 || cols <= 0 || cols % 32) return AQ_E_SHAPE;
  if (rows == 0) return AQ_OK;
  return cuda_status(launch_dequantize_mx(codes, scales, rows, cols, out, out_dtype, static_cast<cudaStream_t>(stream)));
}

int aq_e8m0_codes(const void* x, int x_dtype, int64_t n, uint8_t* codes, int* invalid, void* stream) {
  if (!x || !codes || (x_dtype != 0 && x_dtype != 3)) return AQ_E_INVALID;
  if (n < 0) return AQ_E_SHAPE;
  if (n == 0) return AQ_OK;
  return cuda_status(launch_e8m0_codes(x, x_dtype == 3, n, codes, invalid, static_cast<cudaStream_t>(stream)));
}

int aq_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out, int out_dtype,
                  float tensor_scale, void* stream) {
  if (!codes || !scales || !out || !dtype_ok(out_dtype)) return AQ_E_INVALID;
  float ts = 1.f;
  if (!take_scale(tensor_scale, ts)) return AQ_E_INVALID;
  if (rows < 0 || cols <= 0 || cols % 16) return AQ_E_SHAPE;
  if (rows == 0) return AQ_OK;
  return cuda_status(
      launch_dequantize(codes, scales, rows, cols, out, out_dtype, static_cast<cudaStream_t>(stream), ts));
}

int64_t aq_fp4mm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0 || K <= 0 || K % 16) return 0;
  return fp4mm_workspace_bytes(M, N, K);
}

int aq_fp4mm(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
             const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, void* workspace, void* stream) {
  if (!a_codes || !a_scales || !b_codes || !b_scales || !c || !workspace) return AQ_E_INVALID;
  if (M < 0 || N < 0 || K <= 0 || K % 16 || ldc < N) return AQ_E_SHAPE;
  if (M == 0 || N == 0) return AQ_OK;
  return cuda_status(launch_fp4mm(a_codes, a_scales, M, b_codes, b_scales, N, K, c, ldc,
                                  static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream)));
}

int aq_fp4mm_mx(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
                const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, void* workspace, void* stream) {
  if (!a_codes || !a_scales || !b_codes || !b_scales || !c || !workspace) return AQ_E_INVALID;
  if (M < 0 || N < 0 || K <= 0 || K % 32 || ldc < N) return AQ_E_SHAPE;
  if (M == 0 || N == 0) return AQ_OK;
  return cuda_status(launch_fp4mm(a_codes, a_scales, M, b_codes, b_scales, N, K, c, ldc,
                                  static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream), true));
}

int64_t aq_attn_fwd_workspace_bytes(int64_t heads, int64_t n_q, int64_t n_k, int64_t d, int train, int keep) {
  if (heads <= 0 || n_q <= 0 || n_k <= 0 || (d != 64 && d != 128)) return 0;
  return fwd_ws(heads, n_q, n_k, d, train, keep).total;
}

int aq_attn_fwd(const AqFwdArgs* a, void* stream) {
  if (!a || !a->q || !a->k || !a->v || !a->o || !a->lse || !a->workspace) return AQ_E_INVALID;
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->o_dtype) || (a->o_hp && !dtype_ok(a->o_hp_dtype))) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d % 16) return AQ_E_SHAPE;  // flash.py:187-188
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;  // oracle.py:62-66
  TScales ts;
  if (!read_scales(a, ts)) return AQ_E_INVALID;
  if ((a->pf_codes == nullptr) != (a->pf_scales == nullptr)) return AQ_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const FwdWs w = fwd_ws(a->heads, a->n_q, a->n_k, a->d, a->train, a->keep_for_bwd);
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  if (!a->operands_staged) {
    int s = stage_operands(a->q, a->k, a->v, a->in_dtype, a->heads, a->n_q, a->n_k, a->d, ws, w, st, ts,
                           a->nonfinite);
    if (s != AQ_OK) return s;
  }
  FwdParams p{};
  p.q_codes = ws + w.q_codes;
  p.q_sf = ws + w.q_sf;
  p.k_codes = ws + w.k_codes;
  p.k_sf = ws + w.k_sf;
  p.v_codes = ws + w.v_codes;
  p.v_sf = ws + w.v_sf;
  p.v_h = a->train ? ws + w.v_h16 : nullptr;
  p.o = a->o;
  p.o_dt = a->o_dtype;
  p.o_hp = a->train ? a->o_hp : nullptr;
  p.o_hp_dt = a->o_hp_dtype;
  p.lse = a->lse;
  p.heads = a->heads;
  p.n_q = a->n_q;
  p.n_k = a->n_k;
  p.d = static_cast<int>(a->d);
  p.causal = a->causal;
  p.train = a->train;
  apply_fwd_scales(p, ts, a->d);
  p.pf_codes = a->pf_codes;
  p.pf_scales = a->pf_scales;
  p.item_ctr = reinterpret_cast<int*>(ws + w.sched);
  return cuda_status(launch_attn_fwd(p, st));
}

namespace {
struct SageWs {
  FwdWs f;
  int64_t fwd, gamma_q, gamma_k, q_bar, k_bar, delta, bias, sums, segmax, total, kpad;
};

bool sage_local_seg(int64_t n_k, int64_t b_k) {
  return b_k >= n_k || b_k == 16 || b_k == 32 || b_k == 64 || b_k == 128;
}

SageWs sage_ws(int64_t heads, int64_t n_q, int64_t n_k, int64_t d, int64_t b_q, int64_t b_k) {
  SageWs w{};
  w.f = fwd_ws(heads, n_q, n_k, d, 1, 0);
  w.kpad = ceil_div(n_k, TILE) * TILE;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += align256(bytes);
    return o;
  };
  w.fwd = take(w.f.total);
  w.gamma_q = take(heads * n_q * d * 4);
  w.gamma_k = take(heads * n_k * d * 4);
  w.q_bar = take(heads * (n_q / b_q) * d * 8);
  w.k_bar = take(heads * d * 8);
  w.delta = take(heads * (n_q / b_q) * w.kpad * 4);
  w.bias = take(heads * n_q * 4);
  const int64_t cq = n_q / sage_chunk_rows(b_q), ck = n_k / sage_chunk_rows(n_k);
  w.sums = take(heads * (cq > ck ? cq : ck) * d * 8);  // chunk sums of the means
  // two-level P segment maxima when segments do not sit inside one kernel tile
  w.segmax = (b_k > 0 && n_k % b_k == 0 && !sage_local_seg(n_k, b_k)) ? take(heads * n_q * (n_k / b_k) * 4) : -1;
  w.total = off;
  return w;
}
}  // namespace

int64_t aq_attn_fwd_sage3_workspace_bytes(int64_t heads, int64_t n_q, int64_t n_k, int64_t d, int64_t b_q,
                                          int64_t b_k) {
  if (heads <= 0 || n_q <= 0 || n_k <= 0 || (d != 64 && d != 128) || b_q <= 0 || n_q % b_q) return 0;
  return sage_ws(heads, n_q, n_k, d, b_q, b_k).total;
}

int aq_attn_fwd_sage3(const AqSage3Args* a, void* stream) {
  if (!a || !a->q || !a->k || !a->v || !a->o || !a->lse || !a->workspace) return AQ_E_INVALID;
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->o_dtype)) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d % 16) return AQ_E_SHAPE;
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;
  // TileConfig.validate (flash.py:60-71) and smooth's b_q check (sage3.py:50-53)
  if (a->b_q <= 0 || a->b_k <= 0 || a->n_q % a->b_q || a->n_k % a->b_k) return AQ_E_TILE;
  if (a->n_k > a->b_k && a->b_k % 16) return AQ_E_TILE;
  int seg = -2;  // no two-level P
  if (a->two_level_p) {
    if (a->b_k >= a->n_k) seg = 0;
    else if (sage_local_seg(a->n_k, a->b_k)) seg = static_cast<int>(a->b_k);
    else seg = -1;  // segment maxima from pass 1
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int d = static_cast<int>(a->d);
  const SageWs w = sage_ws(a->heads, a->n_q, a->n_k, a->d, a->b_q, a->b_k);
  uint8_t* base = static_cast<uint8_t*>(a->workspace);
  uint8_t* ws = base + w.fwd;
  float* gq = reinterpret_cast<float*>(base + w.gamma_q);
  float* gk = reinterpret_cast<float*>(base + w.gamma_k);
  double* q_bar = a->smooth_q ? reinterpret_cast<double*>(base + w.q_bar) : nullptr;
  double* k_bar = a->smooth_k ? reinterpret_cast<double*>(base + w.k_bar) : nullptr;
  float* delta = a->smooth_q ? reinterpret_cast<float*>(base + w.delta) : nullptr;
  float* bias = a->smooth_k ? reinterpret_cast<float*>(base + w.bias) : nullptr;
  double* sums = reinterpret_cast<double*>(base + w.sums);
  if (q_bar && launch_sage_means(a->q, a->in_dtype, a->heads, a->n_q, d, a->b_q, sums, q_bar, st) != cudaSuccess)
    return AQ_E_CUDA;
  if (k_bar && launch_sage_means(a->k, a->in_dtype, a->heads, a->n_k, d, a->n_k, sums, k_bar, st) != cudaSuccess)
    return AQ_E_CUDA;
  if (launch_sage_center(a->q, a->in_dtype, a->heads, a->n_q, d, a->b_q, q_bar, gq, st) != cudaSuccess ||
      launch_sage_center(a->k, a->in_dtype, a->heads, a->n_k, d, a->n_k, k_bar, gk, st) != cudaSuccess)
    return AQ_E_CUDA;
  if (delta && launch_sage_delta(q_bar, gk, a->heads, a->n_q / a->b_q, a->n_k, d, w.kpad, delta, st) != cudaSuccess)
    return AQ_E_CUDA;
  if (bias && launch_sage_bias(q_bar, k_bar, gq, a->heads, a->n_q, d, a->b_q, bias, st) != cudaSuccess)
    return AQ_E_CUDA;
  // gamma_q / gamma_k (fp32) and V into the attention tiles; V^F fp16 tiles feed
  // the two-level accumulation
  RowsArgs r{};
  r.x_dt = 0;
  r.heads = a->heads;
  r.cols = a->d;
  r.ld = a->d;
  r.x = gq;
  r.n = a->n_q;
  r.hs = a->n_q * a->d;
  r.codes_t = ws + w.f.q_codes;
  r.sf_t = ws + w.f.q_sf;
  if (launch_quantize_rows(r, st) != cudaSuccess) return AQ_E_CUDA;
  r.x = gk;
  r.n = a->n_k;
  r.hs = a->n_k * a->d;
  r.codes_t = ws + w.f.k_codes;
  r.sf_t = ws + w.f.k_sf;
  if (launch_quantize_rows(r, st) != cudaSuccess) return AQ_E_CUDA;
  r.x = a->v;
  r.x_dt = a->in_dtype;
  r.codes_t = ws + w.f.v_codes;
  r.sf_t = ws + w.f.v_sf;
  r.fqh_t = a->two_level_p ? ws + w.f.v_h16 : nullptr;
  r.fqh_dt = 2;
  if (launch_quantize_cols(r, st) != cudaSuccess) return AQ_E_CUDA;
  FwdParams p{};
  p.q_codes = ws + w.f.q_codes;
  p.q_sf = ws + w.f.q_sf;
  p.k_codes = ws + w.f.k_codes;
  p.k_sf = ws + w.f.k_sf;
  p.v_codes = ws + w.f.v_codes;
  p.v_sf = ws + w.f.v_sf;
  p.v_h = a->two_level_p ? ws + w.f.v_h16 : nullptr;
  p.o = a->two_level_p ? nullptr : a->o;  // two-level P: O comes out of the f16 accumulator
  p.o_dt = a->o_dtype;
  p.o_hp = a->two_level_p ? a->o : nullptr;
  p.o_hp_dt = a->o_dtype;
  p.lse = a->lse;
  p.heads = a->heads;
  p.n_q = a->n_q;
  p.n_k = a->n_k;
  p.d = d;
  p.causal = a->causal;
  p.train = a->two_level_p;
  p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(a->d)));
  p.sage_delta = delta;
  p.sage_bias = bias;
  p.sage_bq = a->b_q;
  p.sage_kpad = w.kpad;
  p.sage_seg = seg;
  p.sage_bk = a->b_k;
  {
    const char* e = std::getenv("AQ_SAGE_HEAD_GROUP");
    p.head_group = e ? std::atoi(e) : 0;
  }
  if (seg == -1) {
    p.sage_segmax = reinterpret_cast<unsigned*>(base + w.segmax);
    if (cudaMemsetAsync(p.sage_segmax, 0, a->heads * a->n_q * (a->n_k / a->b_k) * 4, st) != cudaSuccess)
      return AQ_E_CUDA;
  }
  return cuda_status(launch_attn_fwd_sage(p, st));
}

int aq_attn_fwd_mx(const AqFwdArgs* a, void* stream) {
  if (!a || !a->q || !a->k || !a->v || !a->o || !a->lse || !a->workspace) return AQ_E_INVALID;
  if (a->train && !a->o_hp) return AQ_E_INVALID;
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->o_dtype)) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d % 32) return AQ_E_SHAPE;  // flash.py:260 with block_size 32
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const FwdWs w = fwd_ws(a->heads, a->n_q, a->n_k, a->d, a->train, a->keep_for_bwd);
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  const int d = static_cast<int>(a->d);
  if (a->keep_for_bwd) {
    // the backward's operands too (aq_attn_bwd_mx with this workspace): the
    // codes plus bf16 Q^F / K^F / V^F tiles, then the fp16 V^F tiles of O'
    if (launch_mx_bwd_operands(a->q, a->k, a->v, a->in_dtype, a->heads, a->n_q, a->n_k, d, ws + w.q_codes,
                               ws + w.q_sf, ws + w.q_hb, ws + w.k_codes, ws + w.k_sf, ws + w.k_hb, ws + w.v_codes,
                               ws + w.v_sf, ws + w.v_hb, st, a->train ? ws + w.v_h16 : nullptr) != cudaSuccess)
      return AQ_E_CUDA;
  } else if (launch_mx_attn_operands(a->q, a->k, a->v, a->in_dtype, a->heads, a->n_q, a->n_k, d, ws + w.q_codes,
                                     ws + w.q_sf, ws + w.k_codes, ws + w.k_sf, ws + w.v_codes, ws + w.v_sf,
                                     a->train ? ws + w.v_h16 : nullptr, st) != cudaSuccess) {
    return AQ_E_CUDA;
  }
  FwdParams p{};
  p.q_codes = ws + w.q_codes;
  p.q_sf = ws + w.q_sf;
  p.k_codes = ws + w.k_codes;
  p.k_sf = ws + w.k_sf;
  p.v_codes = ws + w.v_codes;
  p.v_sf = ws + w.v_sf;
  p.v_h = a->train ? ws + w.v_h16 : nullptr;
  p.o = a->o;
  p.o_dt = a->o_dtype;
  p.o_hp = a->train ? a->o_hp : nullptr;
  p.o_hp_dt = a->o_hp_dtype;
  p.lse = a->lse;
  p.heads = a->heads;
  p.n_q = a->n_q;
  p.n_k = a->n_k;
  p.d = d;
  p.causal = a->causal;
  p.train = a->train;
  p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(a->d)));
  p.item_ctr = reinterpret_cast<int*>(ws + w.sched);
  return cuda_status(launch_attn_fwd_mx(p, st));
}

int aq_attn_fwd_plain(const AqFwdArgs* a, int fmt, void* stream) {
  if (!a || !a->q || !a->k || !a->v || !a->o || !a->lse || !a->workspace) return AQ_E_INVALID;
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->o_dtype) || (fmt != 0 && fmt != 1)) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const FwdWs w = fwd_ws(a->heads, a->n_q, a->n_k, a->d, 1, 1);
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  const int d = static_cast<int>(a->d);
  if (launch_tile16(a->q, a->in_dtype, a->heads, a->n_q, d, fmt, ws + w.q_hb, st) != cudaSuccess ||
      launch_tile16(a->k, a->in_dtype, a->heads, a->n_k, d, fmt, ws + w.k_hb, st) != cudaSuccess ||
      launch_tile16(a->v, a->in_dtype, a->heads, a->n_k, d, fmt, ws + w.v_hb, st) != cudaSuccess)
    return AQ_E_CUDA;
  FwdParams p{};
  p.q_codes = ws + w.q_hb;
  p.k_codes = ws + w.k_hb;
  p.v_h = ws + w.v_hb;
  p.o = nullptr;
  p.o_hp = a->o;  // the P^ V accumulator with 1/l is O here
  p.o_hp_dt = a->o_dtype;
  p.lse = a->lse;
  p.heads = a->heads;
  p.n_q = a->n_q;
  p.n_k = a->n_k;
  p.d = d;
  p.causal = a->causal;
  p.train = 1;
  p.plain_fmt = fmt;
  TScales ts;
  if (!read_scales(a, ts) || ts.q != 1.f || ts.k != 1.f || ts.v != 1.f || ts.p != 1.f) return AQ_E_INVALID;
  {
    // d = 128: the 16-bit K / V stream is HBM-bound in the global longest-first
    // order (22 GB read at C2); groups of 4 heads keep it in L2 (4.77 -> 4.15 ms)
    const char* e = std::getenv("AQ_PLAIN_HEAD_GROUP");
    p.head_group = e ? std::atoi(e) : (d == 128 ? 4 : 0);
  }
  p.scale_log2 = scale_log2_of(ts, a->d);
  return cuda_status(launch_attn_fwd_plain(p, st));
}

int aq_attn_fwd_kv4(const AqFwdArgs* a, const uint8_t* k_codes, const uint8_t* k_scales, const uint8_t* vt_codes,
                    const uint8_t* vt_scales, void* stream) {
  if (!a || !a->q || !a->o || !a->lse || !a->workspace) return AQ_E_INVALID;
  if (!k_codes || !k_scales || !vt_codes || !vt_scales) return AQ_E_INVALID;
  if (a->train) return AQ_E_INVALID;  // a KV cache serves inference (no O', no backward)
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->o_dtype)) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d % 16) return AQ_E_SHAPE;
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const FwdWs w = fwd_ws(a->heads, a->n_q, a->n_k, a->d, 0, 0);
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  RowsArgs r{};
  r.x = a->q;
  r.x_dt = a->in_dtype;
  r.heads = a->heads;
  r.n = a->n_q;
  r.cols = a->d;
  r.ld = a->d;
  r.hs = a->n_q * a->d;
  r.codes_t = ws + w.q_codes;
  r.sf_t = ws + w.q_sf;
  if (launch_quantize_rows(r, st) != cudaSuccess) return AQ_E_CUDA;
  if (launch_pack_kv4(k_codes, k_scales, vt_codes, vt_scales, a->heads, a->n_k, static_cast<int>(a->d),
                      ws + w.k_codes, ws + w.k_sf, ws + w.v_codes, ws + w.v_sf, st) != cudaSuccess)
    return AQ_E_CUDA;
  AqFwdArgs b = *a;
  b.operands_staged = 1;
  b.keep_for_bwd = 0;
  b.k = b.q;  // unused once staged
  b.v = b.q;
  return aq_attn_fwd(&b, stream);
}

int64_t aq_attn_bwd_workspace_bytes(int64_t heads, int64_t n_q, int64_t n_k, int64_t d) {
  if (heads <= 0 || n_q <= 0 || n_k <= 0 || (d != 64 && d != 128)) return 0;
  return bwd_ws(heads, n_q, n_k, d).total;
}

static int attn_bwd_impl(const AqBwdArgs* a, void* stream, bool mx);

int aq_attn_bwd(const AqBwdArgs* a, void* stream) { return attn_bwd_impl(a, stream, false); }

int aq_attn_bwd_mx(const AqBwdArgs* a, void* stream) { return attn_bwd_impl(a, stream, true); }

int aq_attn_bwd_plain(const AqBwdArgs* a, int fmt, void* stream) {
  if (!a || !a->q || !a->k || !a->v || !a->d_o || !a->lse || !a->dq || !a->dk || !a->dv || !a->workspace)
    return AQ_E_INVALID;
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->do_dtype) || !dtype_ok(a->o_dtype) || !dtype_ok(a->g_dtype))
    return AQ_E_INVALID;
  if (fmt != 0 && fmt != 1) return AQ_E_INVALID;
  const void* o_ref = a->o_hp ? a->o_hp : a->o;  // O' == O without quantization (flash.py:195-200)
  if (!o_ref) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;
  TScales ts;
  if (!read_scales(a, ts) || ts.q != 1.f || ts.k != 1.f || ts.v != 1.f || ts.p != 1.f) return AQ_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const BwdWs bw = bwd_ws(a->heads, a->n_q, a->n_k, a->d);
  const FwdWs fw = fwd_ws(a->heads, a->n_q, a->n_k, a->d, 0, 1);
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  uint8_t* b = ws + bw.fwd;
  const int d = static_cast<int>(a->d);
  // 16-bit T8x8 tiles of Q / K / V in the forward's format (one copy serves K- and MN-major reads)
  if (launch_tile16(a->q, a->in_dtype, a->heads, a->n_q, d, fmt, b + fw.q_hb, st) != cudaSuccess ||
      launch_tile16(a->k, a->in_dtype, a->heads, a->n_k, d, fmt, b + fw.k_hb, st) != cudaSuccess ||
      launch_tile16(a->v, a->in_dtype, a->heads, a->n_k, d, fmt, b + fw.v_hb, st) != cudaSuccess)
    return AQ_E_CUDA;
  float* delta = reinterpret_cast<float*>(ws + bw.delta);
  if (launch_bwd_pre(a->d_o, a->do_dtype, o_ref, a->o_dtype, a->heads, a->n_q, d, delta, ws + bw.do_h, st, 1.f,
                     fmt == 0 ? 1 : 0) != cudaSuccess)
    return AQ_E_CUDA;
  BwdParams p{};
  p.q_h = b + fw.q_hb;
  p.k_h = b + fw.k_hb;
  p.v_h = b + fw.v_hb;
  p.do_h = ws + bw.do_h;
  p.lse = a->lse;
  p.delta = delta;
  p.dq = a->dq;
  p.dk = a->dk;
  p.dv = a->dv;
  p.g_dt = a->g_dtype;
  p.heads = a->heads;
  p.n_q = a->n_q;
  p.n_k = a->n_k;
  p.d = d;
  p.causal = a->causal;
  p.fq_p = 0;
  p.plain = 1;
  p.plain_fmt = fmt;
  p.scale_log2 = scale_log2_of(ts, a->d);
  p.inv_sqrt_d = static_cast<float>(ts.sm == 0.0 ? 1.0 / std::sqrt(static_cast<double>(a->d)) : ts.sm);
  return cuda_status(launch_attn_bwd(p, st));
}

}  // extern "C"

static int attn_bwd_impl(const AqBwdArgs* a, void* stream, bool mx) {
  if (!a || !a->q || !a->k || !a->v || !a->d_o || !a->lse || !a->dq || !a->dk || !a->dv || !a->workspace)
    return AQ_E_INVALID;
  if (!dtype_ok(a->in_dtype) || !dtype_ok(a->do_dtype) || !dtype_ok(a->o_dtype) || !dtype_ok(a->g_dtype))
    return AQ_E_INVALID;
  if (a->variant < 0 || a->variant > 3) return AQ_E_INVALID;
  const bool uses_op = a->variant == AQ_BWD_CORRECT || a->variant == AQ_BWD_NO_FAKE_QUANT_P;  // flash.py:89-91
  const void* o_ref = uses_op ? a->o_hp : a->o;
  if (uses_op && !a->o_hp) return AQ_E_MISSING_OPRIME;  // flash.py:333-337
  if (!o_ref) return AQ_E_INVALID;
  if (a->heads <= 0 || a->n_q <= 0 || a->n_k <= 0) return AQ_E_SHAPE;
  if (a->d % 16) return AQ_E_SHAPE;
  if (a->d != 64 && a->d != 128) return AQ_E_UNSUPPORTED;
  if (a->causal && a->n_q > a->n_k) return AQ_E_SHAPE;
  TScales ts;
  if (!read_scales(a, ts)) return AQ_E_INVALID;
  if (mx && (ts.q != 1.f || ts.k != 1.f || ts.v != 1.f || ts.p != 1.f)) return AQ_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const BwdWs bw = bwd_ws(a->heads, a->n_q, a->n_k, a->d);
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  const FwdWs fw = fwd_ws(a->heads, a->n_q, a->n_k, a->d, 0, 1);
  const uint8_t* ops;
  FwdWs w;
  if (mx && a->fwd_workspace) {
    if (a->d % 32) return AQ_E_SHAPE;
    ops = static_cast<const uint8_t*>(a->fwd_workspace);  // aq_attn_fwd_mx with keep_for_bwd = 1
    w = fw;
  } else if (mx) {
    // MXFP4 (codec.py:123-203): Q / K codes + UE8M0 images for the S recompute,
    // bf16 Q^F / K^F / V^F tiles for the 16-bit MMAs
    if (a->d % 32) return AQ_E_SHAPE;
    uint8_t* b = ws + bw.fwd;
    if (launch_mx_bwd_operands(a->q, a->k, a->v, a->in_dtype, a->heads, a->n_q, a->n_k, static_cast<int>(a->d),
                               b + fw.q_codes, b + fw.q_sf, b + fw.q_hb, b + fw.k_codes, b + fw.k_sf, b + fw.k_hb,
                               b + fw.v_codes, b + fw.v_sf, b + fw.v_hb, st) != cudaSuccess)
      return AQ_E_CUDA;
    ops = b;
    w = fw;
  } else if (a->fwd_workspace) {
    ops = static_cast<const uint8_t*>(a->fwd_workspace);
    w = fw;
  } else {
    // re-fake-quantize Q, K, V from the originals (flash.py:344-349)
    int s = stage_operands(a->q, a->k, a->v, a->in_dtype, a->heads, a->n_q, a->n_k, a->d, ws + bw.fwd, fw, st, ts,
                           a->nonfinite);
    if (s != AQ_OK) return s;
    ops = ws + bw.fwd;
    w = fw;
  }
  float* delta = reinterpret_cast<float*>(ws + bw.delta);
  cudaError_t e = launch_bwd_pre(a->d_o, a->do_dtype, o_ref, a->o_dtype, a->heads, a->n_q, static_cast<int>(a->d),
                                 delta, ws + bw.do_h, st, 1.f / ts.v);
  if (e != cudaSuccess) return AQ_E_CUDA;
  BwdParams p{};
  p.q_codes = ops + w.q_codes;
  p.q_sf = ops + w.q_sf;
  p.k_codes = ops + w.k_codes;
  p.k_sf = ops + w.k_sf;
  p.q_h = ops + w.q_hb;
  p.k_h = ops + w.k_hb;
  p.v_h = ops + w.v_hb;
  p.do_h = ws + bw.do_h;
  p.lse = a->lse;
  p.delta = delta;
  p.dq = a->dq;
  p.dk = a->dk;
  p.dv = a->dv;
  p.g_dt = a->g_dtype;
  p.heads = a->heads;
  p.n_q = a->n_q;
  p.n_k = a->n_k;
  p.d = static_cast<int>(a->d);
  p.causal = a->causal;
  p.fq_p = (a->variant == AQ_BWD_CORRECT || a->variant == AQ_BWD_LOW_PREC_O) ? 1 : 0;  // flash.py:93-95
  p.mx = mx ? 1 : 0;
  p.scale_log2 = scale_log2_of(ts, a->d);
  // dS = P (t_v dP - D) * sm = P (dP - D / t_v) * (sm t_v); D arrives divided by t_v
  p.inv_sqrt_d = static_cast<float>((ts.sm == 0.0 ? 1.0 / std::sqrt(static_cast<double>(a->d)) : ts.sm) *
                                    static_cast<double>(ts.v));
  p.p_r = 1.f / ts.p;
  p.dq_mul = ts.k;
  p.dk_mul = ts.q;
  p.dv_mul = ts.p;
  if ((a->pf_codes == nullptr) != (a->pf_scales == nullptr)) return AQ_E_INVALID;
  if (!mx) {
    p.pf_codes = a->pf_codes;
    p.pf_scales = a->pf_scales;
  }
  return cuda_status(launch_attn_bwd(p, st));
}
