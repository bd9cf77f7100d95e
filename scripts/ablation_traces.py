"""QAT ablation traces on the GPU (harness.py:39-45 modes): the toy
associative-recall layer trained with each attention mode from the same seed.
Prints loss at checkpoints, the final eval-style mean of the last 20 steps, and
divergence (StabilityError) if it happens."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00040_b200 import train as T  # noqa: E402
from paper_2603_00040_b200.errors import StabilityError  # noqa: E402

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 300
LR = float(sys.argv[2]) if len(sys.argv) > 2 else 3e-3
print(f"# {STEPS} steps, lr {LR}, seq_len 256, batch 16, d_model 256, 2 heads x d 128, causal, seed 0")
print(f"# {'mode':26s} " + " ".join(f"{'step ' + str(s):>10s}" for s in (0, STEPS // 4, STEPS // 2, STEPS - 1))
      + f" {'last-20 mean':>13s} {'max gnorm':>10s}")
for mode in ("bf16", "fp4-qat", "fp4-qat/lowpreco", "fp4-qat/nofqp", "fp4-qat/naive-bf16-bwd"):
    cfg = T.TrainConfig(steps=STEPS, lr=LR, seq_len=256, batch=16, d_model=256, n_heads=2, head_dim=128,
                        causal=True, attn_mode=mode)
    try:
        _, log = T.train(cfg)
        L = np.array(log.losses)
        print(f"  {mode:26s} " + " ".join(f"{L[s]:10.4f}" for s in (0, STEPS // 4, STEPS // 2, STEPS - 1))
              + f" {L[-20:].mean():13.4f} {max(log.grad_norms):10.3f}", flush=True)
    except StabilityError as e:
        print(f"  {mode:26s} diverged: {e}", flush=True)
