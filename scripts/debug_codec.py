import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "codec.npz"))
x = z["randn_x"]
qt = aq.quantize(torch.from_numpy(x.astype(np.float32)).cuda())
c = qt.codes.cpu().numpy(); s = qt.scales.cpu().numpy()
print("codes eq", np.array_equal(c, z["randn_codes"]), "scales eq", np.array_equal(s, z["randn_scales"]))
bad = np.argwhere(c != z["randn_codes"])[:5]
for r, k in bad:
    print(r, k, hex(c[r, k]), hex(z["randn_codes"][r, k]), x[r, 2*k:2*k+2], s[r, k//8], z["randn_scales"][r, k//8])
fq = aq.fake_quantize(torch.from_numpy(x.astype(np.float32)).cuda()).cpu().numpy()
print("fq eq", np.array_equal(fq.astype(np.float64), z["randn_fq"]))
bad = np.argwhere(fq != z["randn_fq"])[:5]
for r, k in bad: print(r, k, fq[r, k], z["randn_fq"][r, k], x[r, k])
