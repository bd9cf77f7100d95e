"""Print backward parity numbers per golden case and variant (debug aid; GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from oracle import nvfp4_attn_oracle as orc  # noqa: E402

att = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "attention.npz"))
for name in ["c1h0", "c1h1", "c1h0c", "d128", "d128c", "offc", "ragged"]:
    n_q, n_k, d, causal, bq, bk = (int(x) for x in att[f"{name}_meta"])
    Q, K, V, dO = (att[f"{name}_{t}"] for t in ("Q", "K", "V", "dO"))
    cfg = aq.TileConfig(b_q=bq, b_k=bk, causal=bool(causal))
    outs = aq.flash_forward_training(Q, K, V, cfg)
    for var in aq.BwdVariant:
        tag = var.value.replace("-", "_")
        try:
            g = aq.flash_backward(Q, K, V, dO, outs, cfg, variant=var)
            errs = [orc.rel_l2(x, att[f"{name}_{tag}_{n}"]) for x, n in ((g.dQ, "dQ"), (g.dK, "dK"), (g.dV, "dV"))]
            print(f"{name:7s} {tag:15s} dQ {errs[0]:.2e} dK {errs[1]:.2e} dV {errs[2]:.2e}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(name, tag, "ERROR", repr(e), flush=True)
