import sys, numpy as np
sys.path.insert(0,'.')
from paper_2603_00040_b200 import harness as H
hg=np.load('tests/golden/harness.npz')
for i in range(4):
    mode=str(hg['modes'][i]); m=H.ToyModel.init(32,32,0)
    loss,grads=H.loss_and_grads(m,H.make_task(0,16,32,8),mode)
    print(mode, 'loss', loss, float(hg[f'm{i}_loss0']), {k: float(np.linalg.norm(g-hg[f'm{i}_g0_{k}'])/np.linalg.norm(hg[f'm{i}_g0_{k}'])) for k,g in grads.items()})
