/*
 * attnqat_b200 -- C ABI of the B200 (sm_100a) NVFP4 Attn-QAT attention path.
 *
 * This is the drop-in boundary for the reference package's operator API
 * (/root/reference/pkg/src/attnqat). Plain pointers, sizes and a CUDA stream
 * (passed as void*); no torch types. Every function is stream-ordered, never
 * synchronises the host, never allocates device memory (callers pass
 * workspaces sized by the *_workspace_bytes queries) and returns an AqStatus.
 *
 * dtype codes: 0 = float32, 1 = bfloat16, 2 = float16.
 *
 * ABI version 3 (aq_abi_version): per-tensor FP32 scales (two-level NVFP4),
 * softmax scale, device non-finite flag and the P^F instrument dump. A scale
 * argument of 0 means 1.0, i.e. the reference's single-level semantics
 * (SPEC.md:129), which every kernel reproduces bit for bit.
 * Tensors are [heads][n][d] contiguous per head (head stride / row stride
 * given explicitly where noted). `heads` is the flattened batch*heads count.
 */
#ifndef ATTNQAT_B200_H_
#define ATTNQAT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference exception classes
 * (attnqat/errors.py:4-41). */
typedef enum {
  AQ_OK = 0,
  AQ_E_SHAPE = 1,          /* ShapeError     errors.py:12-13 */
  AQ_E_TILE = 2,           /* TileError      errors.py:16-17 */
  AQ_E_INVALID = 3,        /* InvalidValue   errors.py:8-9   */
  AQ_E_MISSING_OPRIME = 4, /* MissingOPrime  errors.py:30-31 */
  AQ_E_CUDA = 5,           /* CUDA launch / runtime failure   */
  AQ_E_UNSUPPORTED = 6     /* head dim other than 64 / 128    */
} AqStatus;

/* Backward variants (attnqat/flash.py:83-95, BwdVariant). */
typedef enum {
  AQ_BWD_CORRECT = 0,         /* D = rowsum(dO . O'), P^F in dV */
  AQ_BWD_LOW_PREC_O = 1,      /* D = rowsum(dO . O),  P^F in dV */
  AQ_BWD_NO_FAKE_QUANT_P = 2, /* D = rowsum(dO . O'), P   in dV */
  AQ_BWD_NAIVE_BF16 = 3       /* D = rowsum(dO . O),  P   in dV */
} AqBwdVariant;

int aq_abi_version(void);
const char* aq_status_string(int status);

/* ---- NVFP4 codec --------------------------------------------------------
 * Replaces attnqat.codec.quantize / fake_quantize (codec.py:302-340).
 * Blocks of 16 along the contiguous axis of x [heads][n][cols]
 * (row stride ld, head stride hs, in elements). Outputs in the reference
 * layout: codes [heads*n][cols/2] (low nibble = lower index), scales
 * [heads*n][cols/16] E4M3 codes; fq (optional) = dequantized values in
 * fq_dtype. nonfinite (optional, device int) is OR-ed with 1 when an input
 * is NaN/Inf (the reference raises InvalidValue, codec.py:313-314).
 * tensor_scale t (north_star's per-tensor FP32 scale; 0 or 1 = reference):
 * blocks of x / t are quantized, so x ~ t * scale * code; fq includes t. */
int aq_quantize_rows(const void* x, int x_dtype, int64_t heads, int64_t n, int64_t cols, int64_t ld,
                     int64_t hs, uint8_t* codes, uint8_t* scales, void* fq, int fq_dtype, float tensor_scale,
                     int* nonfinite, void* stream);

/* Replaces quantize_padded(V.T) / fake_quantize_cols (codec.py:359-381):
 * blocks of 16 along the token axis of x [heads][n][cols]; the token tail is
 * zero-padded to n16 = ceil(n/16)*16. codes [heads][cols][n16/2], scales
 * [heads][cols][n16/16]; fq (optional) [heads][n][cols]. */
int aq_quantize_cols(const void* x, int x_dtype, int64_t heads, int64_t n, int64_t cols, int64_t ld,
                     int64_t hs, uint8_t* codes, uint8_t* scales, void* fq, int fq_dtype, float tensor_scale,
                     int* nonfinite, void* stream);

/* Replaces attnqat.codec.round_to_fp4 (format 0, codec.py:76-88) and
 * round_to_e4m3 (format 1, codec.py:101-112): one code per element of x
 * (x_dtype 0 = fp32, 3 = fp64; exact in that precision, ties to even).
 * *invalid is set for non-finite input (and negative input for E4M3). */
int aq_round_codes(const void* x, int x_dtype, int64_t n, int format, uint8_t* codes, int* invalid, void* stream);

/* MXFP4 (BlockSpec(32, E8M0), codec.py:123-203): quantize(x, MXFP4) /
 * fake_quantize(x, MXFP4) / dequantize of an MXFP4 QuantTensor. x [rows][cols]
 * (cols % 32 == 0); codes [rows][cols/2], scales [rows][cols/32] (E8M0). */
int aq_quantize_mx(const void* x, int x_dtype, int64_t rows, int64_t cols, uint8_t* codes, uint8_t* scales,
                   void* fq, int fq_dtype, int* nonfinite, void* stream);
int aq_dequantize_mx(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                     int out_dtype, void* stream);
/* Replaces attnqat.codec.round_to_e8m0 (codec.py:123-136): nearest power of two,
 * ties up, code clamped to 0..254; x_dtype 0 = fp32, 3 = fp64; *invalid set for
 * non-finite or non-positive input. */
int aq_e8m0_codes(const void* x, int x_dtype, int64_t n, uint8_t* codes, int* invalid, void* stream);

/* Replaces attnqat.codec.dequantize (codec.py:327-333). rows x cols; values
 * code * scale * tensor_scale (0 or 1 = reference). */
int aq_dequantize(const uint8_t* codes, const uint8_t* scales, int64_t rows, int64_t cols, void* out,
                  int out_dtype, float tensor_scale, void* stream);

/* Replaces attnqat.tensors.fp4mm (tensors.py:54-86): C = A B^T from two NVFP4
 * QuantTensors blocked along the shared contraction axis K (K % 16 == 0):
 * A codes [M][K/2] + scales [M][K/16], B^T codes [N][K/2] + scales [N][K/16];
 * C [M][N] fp32 with row stride ldc. Block-scaled tcgen05 MMAs (exact block
 * products, fp32 accumulation). workspace: aq_fp4mm_workspace_bytes(M, N, K). */
int64_t aq_fp4mm_workspace_bytes(int64_t M, int64_t N, int64_t K);
/* The same for MXFP4 QuantTensors (codec.py:123-166): UE8M0 scales, one per
 * 32 codes (a_scales [M][K/32], b_scales [N][K/32]), K % 32 == 0, on
 * tcgen05.mma.kind::mxf4.block_scale.block32. Workspace as for aq_fp4mm. */
int aq_fp4mm_mx(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
                const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, void* workspace, void* stream);
int aq_fp4mm(const uint8_t* a_codes, const uint8_t* a_scales, int64_t M, const uint8_t* b_codes,
             const uint8_t* b_scales, int64_t N, int64_t K, float* c, int64_t ldc, void* workspace, void* stream);

/* ---- fused attention ----------------------------------------------------- */
typedef struct {
  const void* q; const void* k; const void* v; /* [heads][n_q|n_k][d], dtype in_dtype */
  int in_dtype;
  int64_t heads, n_q, n_k, d;
  int causal;        /* right-aligned causal mask (oracle.py:62-75) */
  int train;         /* 1: flash_forward_training (emit O_hp), 0: flash_forward_inference */
  void* o;           /* [heads][n_q][d], o_dtype */
  int o_dtype;
  void* o_hp;        /* [heads][n_q][d] O' (train only; may be NULL) */
  int o_hp_dtype;
  float* lse;        /* [heads][n_q] natural-log LSE L (flash.py:217) */
  void* workspace;   /* aq_attn_fwd_workspace_bytes(); keep it for the backward */
  int keep_for_bwd;  /* also stage the bf16 operands the backward reuses */
  int operands_staged; /* 1: workspace already holds this Q/K/V's quantized tiles
                          (e.g. an FP4 KV cache); skip the quantizers */
  /* --- ABI 3 --- */
  float softmax_scale; /* 0: 1/sqrt(d) (flash.py:207) */
  float q_scale, k_scale, v_scale; /* per-tensor FP32 scales t_q, t_k, t_v (0 or 1 = reference):
                          S = t_q t_k Q^F K^F^T, O = t_v (P^F V^F) */
  float p_scale;       /* t_p: P quantized as two-level NVFP4 P^F = t_p s code with the 16-key
                          block scales over P / t_p. 0 or 1 = the reference (single level,
                          2^-9 scale floor); e.g. 1/2688 keeps long-row P above the floor.
                          Not parity for t_p != 1 (the reference has no tensor scale). */
  int* nonfinite;      /* optional device int, OR-ed with 1 when Q / K / V hold NaN / Inf
                          (codec.py:313-314); the caller reads it and raises InvalidValue */
  uint8_t* pf_codes;   /* optional instrument dump (flash.py:117-124, PTileRecord): P^F of every
                          row as quantize_padded(P) would store it, codes [heads][n_q][n16/2] */
  uint8_t* pf_scales;  /* and scales [heads][n_q][n16/16], n16 = ceil(n_k/16)*16; both or neither */
} AqFwdArgs;

int64_t aq_attn_fwd_workspace_bytes(int64_t heads, int64_t n_q, int64_t n_k, int64_t d, int train,
                                    int keep_for_bwd);
/* Replaces flash_forward_training / flash_forward_inference (flash.py:176-314). */
int aq_attn_fwd(const AqFwdArgs* args, void* stream);

/* flash_forward_inference with cfg.spec = MXFP4 (flash.py:249-314,
 * codec.py:123-203): Q / K / V^T quantized in 32-element blocks with UE8M0
 * scales, P in 32-key blocks, S and PV on tcgen05.mma.kind::mxf4 block32.
 * args->train = 1 also writes O' (args->o_hp; flash.py:176-246); keep_for_bwd = 1
 * also stages the backward's operands so aq_attn_bwd_mx can take this workspace.
 * d % 32 == 0 (d in {64, 128}). Workspace: aq_attn_fwd_workspace_bytes(heads,
 * n_q, n_k, d, train, keep_for_bwd). */
int aq_attn_fwd_mx(const AqFwdArgs* args, void* stream);

/* quantized=False (flash.py:195-200): plain softmax attention on the same
 * kernel skeleton with 16-bit operands (fmt 0 = fp16, 1 = bf16; inputs are
 * converted), S and P^ V on kind::f16 MMAs with fp32 accumulation. Writes O
 * (args->o) and L; args->train / o_hp / keep_for_bwd / operands_staged are
 * ignored, and of the scale fields only softmax_scale (0 = 1/sqrt(d)).
 * Workspace: aq_attn_fwd_workspace_bytes(heads, n_q, n_k, d, 1, 1). */
int aq_attn_fwd_plain(const AqFwdArgs* args, int fmt, void* stream);

/* FP4 KV cache: inference forward (flash_forward_inference, flash.py:249-314)
 * over K and V already quantized in the reference QuantTensor layout -- the
 * payload of ATQ4 files (tensors.py:173-188):
 *   K   = quantize(K)            codes [heads][n_k][d/2],   scales [heads][n_k][d/16]
 *   V^T = quantize_padded(V.T)   codes [heads][d][n16/2],   scales [heads][d][n16/16]
 * (n16 = ceil(n_k/16)*16, codec.py:359-361). args->k / args->v are ignored,
 * args->train must be 0; Q is quantized on the fly. Bit-identical to aq_attn_fwd
 * on the K / V these caches were quantized from. */
int aq_attn_fwd_kv4(const AqFwdArgs* args, const uint8_t* k_codes, const uint8_t* k_scales,
                    const uint8_t* vt_codes, const uint8_t* vt_scales, void* stream);

/* SageAttention3-style forward (sage3_forward, sage3.py:113-194): Q / K
 * smoothing (per-b_q-tile Q means, global K mean, sage3.py:45-60), the score
 * decomposition S = fp4(gamma_q) fp4(gamma_k)^T + q_bar gamma_k^T + bias
 * (sage3.py:74-88) and two-level P (each row of each b_k key segment rescaled
 * onto [0, 448*6] before NVFP4, the product divided back, sage3.py:98-110,
 * 186-190). Every toggle is independent. b_q must divide n_q, b_k must
 * divide n_k (and be a multiple of 16 when n_k > b_k); AQ_E_TILE otherwise.
 * Outputs O [heads][n_q][d] (o_dtype) and L. */
typedef struct {
  const void* q; const void* k; const void* v; /* [heads][n][d], in_dtype */
  int in_dtype;
  int64_t heads, n_q, n_k, d;
  int causal;
  int64_t b_q, b_k;
  int smooth_q, smooth_k, two_level_p;
  void* o;           /* [heads][n_q][d], o_dtype */
  int o_dtype;
  float* lse;        /* [heads][n_q] */
  void* workspace;   /* aq_attn_fwd_sage3_workspace_bytes() */
} AqSage3Args;

int64_t aq_attn_fwd_sage3_workspace_bytes(int64_t heads, int64_t n_q, int64_t n_k, int64_t d, int64_t b_q,
                                          int64_t b_k);
/* Replaces sage3_forward (sage3.py:113-194) for quantized=True. */
int aq_attn_fwd_sage3(const AqSage3Args* args, void* stream);

typedef struct {
  const void* q; const void* k; const void* v; /* original operands, in_dtype */
  int in_dtype;
  const void* d_o;   /* [heads][n_q][d], do_dtype */
  int do_dtype;
  const void* o;     /* forward O  (LOW_PREC_O / NAIVE); dtype o_dtype */
  const void* o_hp;  /* forward O' (CORRECT / NO_FAKE_QUANT_P); dtype o_dtype */
  int o_dtype;
  const float* lse;  /* [heads][n_q] */
  int64_t heads, n_q, n_k, d;
  int causal;
  int variant;       /* AqBwdVariant */
  void* dq; void* dk; void* dv; /* [heads][n][d], g_dtype */
  int g_dtype;
  void* workspace;   /* aq_attn_bwd_workspace_bytes() */
  const void* fwd_workspace; /* forward workspace with keep_for_bwd=1, or NULL to re-quantize */
  /* --- ABI 3: as AqFwdArgs (the forward's values) --- */
  float softmax_scale;
  float q_scale, k_scale, v_scale, p_scale;
  int* nonfinite;
  uint8_t* pf_codes;   /* optional instrument dump of the recomputed P^F (flash.py:386-387; CORRECT /
                          LOW_PREC_O only), layout as AqFwdArgs::pf_codes */
  uint8_t* pf_scales;
} AqBwdArgs;

int64_t aq_attn_bwd_workspace_bytes(int64_t heads, int64_t n_q, int64_t n_k, int64_t d);
/* Replaces flash_backward (flash.py:317-390). */
int aq_attn_bwd(const AqBwdArgs* args, void* stream);
/* The same for MXFP4 operands (cfg.spec = MXFP4): S recomputed on
 * tcgen05.mma.kind::mxf4 block32, P^F in 32-key UE8M0 blocks, Q^F / K^F / V^F
 * re-quantized from args->q / k / v, or taken from args->fwd_workspace (an
 * aq_attn_fwd_mx workspace with keep_for_bwd = 1); d % 32 == 0. */
int aq_attn_bwd_mx(const AqBwdArgs* args, void* stream);
/* quantized=False backward (flash_backward with quantized=False,
 * flash.py:344-349 -- every variant reduces to it): the K7 skeleton with S
 * recomputed from 16-bit Q / K tiles on kind::f16, P = exp(S - L) unquantized,
 * D = rowsum(dO . O) with O = args->o_hp if set, else args->o (O' == O here).
 * fmt as for aq_attn_fwd_plain (0 = fp16, 1 = bf16: every 16-bit operand --
 * Q, K, V, dO, P, dS -- in that format; pass the forward's format so S and L
 * agree; for fp16 the caller keeps dO inside fp16's range, e.g. by an exact
 * power-of-two gain it divides out of the gradients), fp32 accumulation; only
 * softmax_scale of the scale fields is honoured (the others must be 0 / 1);
 * fwd_workspace and pf_* are ignored. Workspace: aq_attn_bwd_workspace_bytes(). */
int aq_attn_bwd_plain(const AqBwdArgs* args, int fmt, void* stream);

/* ---- measurement utilities (bench.py roofline denominators) ---------------
 * One CTA per SM issuing back-to-back tcgen05 MMAs from shared memory:
 * kind 0 = NVFP4 block-scaled (mxf4nvf4, M128 N256 K64), 1 = bf16 (f16 kind,
 * M128 N256 K16). Time the launch with events; FLOPs from aq_probe_mma_flops. */
int aq_probe_mma_peak(int kind, int ctas, int rounds, void* stream);
double aq_probe_mma_flops(int kind, int ctas, int rounds);
/* Cycle counters of the forward softmax warps (filled when the environment
 * sets AQ_FWD_DEBUG bit 32; tuning aid). out: 16 counters. */
int aq_debug_fwd_profile(unsigned long long* out, int reset);
/* Cycle counters of the backward compute warps (library built with
 * -DAQ_BWD_PROFILE; tuning aid). out: 16 counters. */
int aq_debug_bwd_profile(unsigned long long* out, int reset);
/* Per-CTA timeline of the last backward launch, 5 values per CTA (globaltimer ns
 * of entry / first S tile / tile loop done / exit, then smid | is_kv << 16);
 * only in -DAQ_BWD_PROFILE builds, otherwise returns AQ_E_CUDA. Measurement only. */
int aq_debug_bwd_timeline(unsigned long long* out, int ctas);

#ifdef __cplusplus
}
#endif
#endif /* ATTNQAT_B200_H_ */
