"""Desk-scale QAT acceptance on the GPU (SPEC acceptance 7-8 analogues,
/root/reference/SPEC.md:564-565; harness.py:294-344).

    python scripts/qat_acceptance.py [steps] [lr] [seeds] [json_out]

The reference harness's toy config (harness.py:93-107: seq_len 16, d_model 32,
head_dim 32, one head, batch 8, 400 steps, lr 1e-3) trained through this
package's attention (attn_qat: NVFP4 two-pass forward + QAT backward; "bf16"
mode = quantized=False), projections in fp32. For every seed:

* 7 (QAT recovery): FP4-eval loss of the FP4-QAT model vs FP4-eval loss of the
  bf16-trained model (>= 50 % lower), and vs the bf16 model's bf16-eval loss
  (within 2x); eval batch 64 from the held-out seed (harness.py:347-351).
* 8 (stability): max grad norm of LOW_PREC_O vs CORRECT (>= 10x, or the run
  diverges with StabilityError); grad-norm variance of NO_FAKE_QUANT_P vs
  CORRECT (strictly larger).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00040_b200 import train as T  # noqa: E402
from paper_2603_00040_b200.errors import StabilityError  # noqa: E402

EVAL_SEED_OFFSET = 999_983   # harness.py:287


def run(mode, seed, steps, lr, **kw):
    cfg = T.TrainConfig(steps=steps, lr=lr, seed=seed, seq_len=kw.get("seq_len", 16), batch=kw.get("batch", 8),
                        d_model=kw.get("d_model", 32), n_heads=1, head_dim=kw.get("head_dim", 32),
                        attn_mode=mode, compute_dtype="fp32")
    try:
        layer, log = T.train(cfg)
    except StabilityError as e:
        return {"mode": mode, "seed": seed, "diverged": True, "step": e.step, "error": str(e)}
    X, Y = T.make_task(seed * 1_000_003 + EVAL_SEED_OFFSET, cfg.seq_len, cfg.d_model, 64)
    import torch
    out = {"mode": mode, "seed": seed, "diverged": False,
           "final_loss": float(np.mean(log.losses[-20:])),
           "max_gnorm": float(np.max(log.grad_norms)), "gnorm_var": float(np.var(log.grad_norms)),
           "eval_fp4": T.evaluate(layer, X, Y, "fp4", dtype=torch.float32),
           "eval_bf16": T.evaluate(layer, X, Y, "bf16", dtype=torch.float32),
           "eval_fp4_fake": T.evaluate(layer, X, Y, "fp4-fake", dtype=torch.float32),
           "baseline": T.random_prediction_baseline(Y)}
    return out


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    lr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
    seeds = [int(s) for s in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2]
    res = []
    for seed in seeds:
        for mode in ("bf16", "fp4-qat", "fp4-qat/lowpreco", "fp4-qat/nofqp"):
            r = run(mode, seed, steps, lr)
            res.append(r)
            print(json.dumps(r), flush=True)
    if len(sys.argv) > 4:
        with open(sys.argv[4], "w") as fh:
            json.dump({"steps": steps, "lr": lr, "seeds": seeds, "runs": res}, fh, indent=1)


if __name__ == "__main__":
    main()
