"""B200-native (sm_100a) NVFP4 Attn-QAT attention: drop-in for the reference
``attnqat`` operator API (quantize / dequantize / fake_quantize /
fake_quantize_cols, flash_forward_training / flash_forward_inference /
flash_backward) plus a torch.autograd.Function for batched CUDA tensors.
All compute runs in ``libattnqat_b200.so`` (hand-written sm_100a CUDA through
a C ABI); there is no CPU fallback.
"""

from .autograd import AttnQATFunction, attn_qat
from .codec import (MXFP4, NVFP4, BlockSpec, Fp4Block, QuantTensor, ScaleFormat, auto_tensor_scale, decode_e4m3,
                    decode_fp4, dequantize,
                    dequantize_block, encode_fp4, fake_quantize, fake_quantize_cols, fake_quantize_padded, quantize,
                    quantize_block, quantize_cols, quantize_padded, round_to_e4m3, round_to_e8m0, round_to_fp4,
                    decode_e8m0)
from .errors import (AttnQatError, FormatError, InvalidValue, MissingOPrime, ShapeError, StabilityError,
                     TileError)
from .flash import (AttnGrads, AttnOutputs, BwdVariant, PTileRecord, RowState, TileConfig, attn_backward,
                    attn_forward, attn_forward_host, attn_forward_mx, attn_qat_host, check_nonfinite,
                    flash_backward, flash_forward_inference, flash_forward_training, kernel_head_dim,
                    nonfinite_flag, pf_buffers)
from .kvcache import KV4Cache, attn_forward_kv4, attn_forward_kv4_host, kv4_quantize, load_kv4, save_kv4
from .materialized import OracleTrace, QuantPoints, oracle_backward, oracle_forward
from .sage3 import (P_RESCALE_MAX, ScoreDecomposition, SmoothedPair, TwoLevelP, attn_forward_sage3,
                    decompose_scores, quantize_p_two_level, sage3_forward, smooth)
from . import tracking
from .tensors import Rng, fp4mm, load_quant_tensor, load_tensor, matmul, randn, save_quant_tensor, save_tensor

__version__ = "0.1.0"
