// Internal kernel parameter blocks and launchers (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace aq {

struct RowsArgs {
  const void* x;
  int x_dt;
  int64_t heads, n, cols, ld, hs;
  uint8_t* codes_ref;
  uint8_t* scales_ref;
  void* fq;
  int fq_dt;
  uint8_t* codes_t;
  uint8_t* sf_t;
  void* fqh_t;
  int fqh_dt;
  void* fqh2_t;   // optional second T8x8 copy in another 16-bit dtype (K2 only)
  int fqh2_dt;
  int* nonfinite;
  float inv_ts = 1.f;  // per-tensor FP32 scale t: blocks of x / t are quantized (1 = reference semantics)
  float ts = 1.f;      // t, applied to the dense fake-quant output (fq) only
};

struct FwdParams {
  const uint8_t* q_codes;
  const uint8_t* q_sf;
  const uint8_t* k_codes;
  const uint8_t* k_sf;
  const uint8_t* v_codes;  // V^T tiles
  const uint8_t* v_sf;
  const uint8_t* v_h;      // fp16 T8x8 tiles of V^F (train)
  void* o;
  int o_dt;
  void* o_hp;
  int o_hp_dt;
  float* lse;
  int64_t heads, n_q, n_k;
  int d;
  int causal;
  int train;
  float scale_log2;
  int debug;  // timing experiments only (0 in production): 1 skip P quant, 2 skip exp, 4 skip pass-1 math
  // SageAttention3 toggles (sage3.py; read by the K4 SAGE instances only)
  const float* sage_delta;  // [heads][n_q / sage_bq][sage_kpad]: q_bar gamma_k^T per query tile, or null
  const float* sage_bias;   // [heads][n_q]: q_bar k_bar + gamma_q k_bar per row, or null
  int64_t sage_bq, sage_kpad;
  int sage_seg;             // two-level P segment (keys): 16 / 32 / 64 / 128, 0 = the whole row,
                            // -1 = any other b_k: segment maxima of S from pass 1 in sage_segmax
  unsigned* sage_segmax;    // [heads][n_q][n_k / sage_bk], order-preserving float codes, zeroed
  int64_t sage_bk;
  int plain_fmt;            // PLAIN instances: 16-bit operand format, 0 = fp16, 1 = bf16
  int head_group;           // causal item order: 0 = longest-first over all heads, G > 0 = within groups of G heads
  // per-tensor FP32 scales (north_star two-level NVFP4; all 1 = reference semantics, bit for bit):
  // scale_log2 already holds t_q t_k; O is multiplied by o_mul = t_v t_p, O' by ohp_mul = t_v, and P
  // blocks are quantized as P * p_r (p_r = 1 / t_p; p_lshift = log2 t_p for the pass-2 early-out)
  float o_mul = 1.f, ohp_mul = 1.f, p_r = 1.f, p_lshift = 0.f;
  // instrument (flash.py:117-124, PTileRecord): when set, P^F of every visible row in the
  // reference's quantize_padded(P) layout per row: codes [heads][n_q][n16/2], scales [heads][n_q][n16/16]
  uint8_t* pf_codes = nullptr;
  uint8_t* pf_scales = nullptr;
  // K4 dynamic item queue: a workspace int the launch zeroes, or null (static order)
  int* item_ctr = nullptr;
  int item_band = 8;  // query tiles per band of the dynamic order
};

struct BwdParams {
  const uint8_t* q_codes;
  const uint8_t* q_sf;
  const uint8_t* k_codes;
  const uint8_t* k_sf;
  const uint8_t* q_h;    // bf16 T8x8 Q^F tiles
  const uint8_t* k_h;    // bf16 T8x8 K^F tiles
  const uint8_t* v_h;    // bf16 T8x8 V^F tiles
  const uint8_t* do_h;   // bf16 T8x8 dO tiles
  const float* lse;      // [heads][n_q]
  const float* delta;    // [heads][nq_pad] D = rowsum(dO . O_ref)
  void* dq;
  void* dk;
  void* dv;
  int g_dt;
  int64_t heads, n_q, n_k;
  int d;
  int causal;
  int fq_p;              // quantize the recomputed P for dV
  int mx;                // MXFP4: S on kind::mxf4 block32, P^F in 32-key UE8M0 blocks
  int plain = 0;         // quantized=False: S on kind::f16 from 16-bit Q / K tiles (q_h / k_h), P unquantized
  int plain_fmt = 1;     // PLAIN operand format: 1 = bf16, 0 = fp16 (every 16-bit tile and MMA)
  float scale_log2;      // log2(e)/sqrt(d) (times t_q t_k)
  float inv_sqrt_d;      // 1/sqrt(d) (times t_v: dS = P (t_v dP - D) / sqrt(d), D pre-divided by t_v)
  float p_r = 1.f;       // 1 / t_p: P^F quantized as P * p_r (1 = reference semantics)
  float dq_mul = 1.f, dk_mul = 1.f, dv_mul = 1.f;  // t_k, t_q, t_p (1 = reference semantics)
  uint8_t* pf_codes = nullptr;   // instrument: the recomputed P^F, layout as FwdParams::pf_codes
  uint8_t* pf_scales = nullptr;
};

cudaError_t launch_quantize_rows(const RowsArgs& a, cudaStream_t st);
cudaError_t launch_quantize_cols(const RowsArgs& a, cudaStream_t st);
cudaError_t launch_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                              int out_dt, cudaStream_t st, float ts = 1.f);
cudaError_t launch_attn_fwd(const FwdParams& p, cudaStream_t st);
cudaError_t launch_attn_fwd_infer(const FwdParams& p, cudaStream_t st);
cudaError_t launch_attn_fwd_infer_mx(const FwdParams& p, cudaStream_t st);
cudaError_t launch_attn_fwd_qat(const FwdParams& p, cudaStream_t st);
cudaError_t launch_attn_fwd_qat_mx(const FwdParams& p, cudaStream_t st);
// K4 with the sage3 score terms; p.train selects two-level P (O written from
// the f16 accumulator into p.o_hp) vs plain NVFP4 P (O into p.o)
cudaError_t launch_attn_fwd_sage(const FwdParams& p, cudaStream_t st);
// quantized=False on K4: 16-bit Q / K / V tiles (q_codes / k_codes / v_h hold T8x8
// images), O written to p.o_hp
cudaError_t launch_attn_fwd_plain(const FwdParams& p, cudaStream_t st);
// MXFP4 inference forward on K4 (kind::mxf4 block32; the attention tiles from
// launch_mx_attn_operands, P quantized in 32-key UE8M0 blocks)
cudaError_t launch_attn_fwd_mx(const FwdParams& p, cudaStream_t st);
// MXFP4 backward operands: Q / K codes + SF tiles with bf16 Q^F / K^F T8x8
// tiles, V^F bf16 T8x8 tiles
cudaError_t launch_mx_bwd_operands(const void* q, const void* k, const void* v, int x_dt, int64_t heads,
                                   int64_t n_q, int64_t n_k, int d, uint8_t* q_codes, uint8_t* q_sf, uint8_t* q_h,
                                   uint8_t* k_codes, uint8_t* k_sf, uint8_t* k_h, uint8_t* v_codes, uint8_t* v_sf,
                                   uint8_t* v_h, cudaStream_t st, uint8_t* v_h16 = nullptr);
cudaError_t launch_mx_attn_operands(const void* q, const void* k, const void* v, int x_dt, int64_t heads,
                                    int64_t n_q, int64_t n_k, int d, uint8_t* q_codes, uint8_t* q_sf,
                                    uint8_t* k_codes, uint8_t* k_sf, uint8_t* v_codes, uint8_t* v_sf,
                                    uint8_t* v_h16, cudaStream_t st);
// [heads][n][d] (x_dt) -> 16-bit T8x8 tiles (fmt 0 fp16 / 1 bf16), rows zero-padded to 128
cudaError_t launch_tile16(const void* x, int x_dt, int64_t heads, int64_t n, int d, int fmt, uint8_t* out,
                          cudaStream_t st);
// rows per partial-sum chunk of a mean over `seg` rows: the largest divisor of seg <= 128
inline int64_t sage_chunk_rows(int64_t seg) {
  int64_t c = seg < 128 ? seg : 128;
  while (c > 1 && seg % c) --c;
  return c;
}
cudaError_t launch_sage_means(const void* x, int x_dt, int64_t heads, int64_t n, int d, int64_t seg,
                              double* scratch, double* mean, cudaStream_t st);
cudaError_t launch_sage_center(const void* x, int x_dt, int64_t heads, int64_t n, int d, int64_t seg,
                               const double* mean, float* gamma, cudaStream_t st);
cudaError_t launch_sage_delta(const double* q_bar, const float* gamma_k, int64_t heads, int64_t t_q, int64_t n_k,
                              int d, int64_t kpad, float* delta, cudaStream_t st);
cudaError_t launch_sage_bias(const double* q_bar, const double* k_bar, const float* gamma_q, int64_t heads,
                             int64_t n_q, int d, int64_t b_q, float* bias, cudaStream_t st);
cudaError_t launch_attn_bwd(const BwdParams& p, cudaStream_t st);
int64_t fp4mm_workspace_bytes(int64_t M, int64_t N, int64_t K);
cudaError_t launch_fp4mm(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
                         const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, uint8_t* ws,
                         cudaStream_t st, bool mx = false);
cudaError_t launch_quantize_mx(const void* x, int x_dt, int64_t rows, int64_t cols, uint8_t* codes, uint8_t* scales,
                               void* fq, int fq_dt, int* nonfinite, cudaStream_t st);
cudaError_t launch_dequantize_mx(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                                 int out_dt, cudaStream_t st);
cudaError_t launch_e8m0_codes(const void* x, int x_is_f64, int64_t n, uint8_t* codes, int* invalid, cudaStream_t st);
cudaError_t launch_round_codes(const void* x, int x_is_f64, int64_t n, int format, uint8_t* codes, int* invalid,
                               cudaStream_t st);
cudaError_t launch_pack_kv4(const uint8_t* k_codes, const uint8_t* k_scales, const uint8_t* vt_codes,
                            const uint8_t* vt_scales, int64_t heads, int64_t n, int d, uint8_t* k_codes_t,
                            uint8_t* k_sf_t, uint8_t* v_codes_t, uint8_t* v_sf_t, cudaStream_t st);
cudaError_t launch_bwd_pre(const void* d_o, int do_dt, const void* o_ref, int o_dt, int64_t heads, int64_t n_q,
                           int d, float* delta, uint8_t* do_h, cudaStream_t st, float delta_mul = 1.f,
                           int tile_f16 = 0);

}  // namespace aq
