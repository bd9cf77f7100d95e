"""Print the GPU harness trajectories next to the reference's goldens (tests/golden/harness.npz)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2603_00040_b200 import harness as H
hg = np.load('tests/golden/harness.npz')
for i in range(4):
    mode = str(hg['modes'][i])
    cfg = H.TrainConfig(steps=30, lr=1e-2, seed=0, attn_mode=mode)
    m, log = H.train(H.ToyModel.init(32, 32, 0), cfg)
    L, wl = np.array(log.losses), hg[f'm{i}_losses']
    G, wg = np.array(log.grad_norms), hg[f'm{i}_gnorms']
    print(mode, 'loss rel diff per step:', np.round(np.abs(L - wl) / wl, 4).tolist())
    print('   gnorm rel diff:', np.round(np.abs(G - wg) / wg, 4).tolist())
    ev = H.eval_batch(cfg)
    print('   eval', [H.evaluate(m, ev, e) for e in ('bf16', 'fp4', 'fp4-fake')], hg[f'm{i}_eval'].tolist())
