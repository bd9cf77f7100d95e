"""Print forward parity numbers per golden case (debug aid; GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from oracle import nvfp4_attn_oracle as orc  # noqa: E402

att = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "attention.npz"))
for name in ["c1h0", "c1h1", "c1h0c", "d128", "d128c", "offc", "ragged"]:
    n_q, n_k, d, causal, bq, bk = (int(x) for x in att[f"{name}_meta"])
    Q, K, V = (att[f"{name}_{t}"] for t in "QKV")
    cfg = aq.TileConfig(b_q=bq, b_k=bk, causal=bool(causal))
    try:
        o = aq.flash_forward_training(Q, K, V, cfg)
        oi = aq.flash_forward_inference(Q, K, V, cfg)
        print(f"{name:7s} O {orc.rel_l2(o.O, att[name+'_O']):.2e} Op {orc.rel_l2(o.O_prime, att[name+'_Op']):.2e} "
              f"L {np.max(np.abs(o.L - att[name+'_L'])):.2e} Oinf {orc.rel_l2(oi.O, att[name+'_Oinf']):.2e} "
              f"|O| {np.linalg.norm(o.O):.3f} ref {np.linalg.norm(att[name+'_O']):.3f}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "ERROR", repr(e), flush=True)
