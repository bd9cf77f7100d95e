"""Per-segment cycle breakdown of the forward softmax warps (AQ_FWD_DEBUG=32)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00040_b200 as aq  # noqa: E402
from paper_2603_00040_b200 import _lib  # noqa: E402
lib = _lib.load()
fn = lib.aq_debug_fwd_profile
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
B, H, N, d = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (4, 32, 8192, 128)
causal = True
train = os.environ.get("AQ_PROF_TRAIN", "0") == "1"
q, k, v = (torch.randn(B, H, N, d, device="cuda").bfloat16() for _ in range(3))
o, lse, _, ws = aq.attn_forward(q, k, v, causal=causal, train=train)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
fn(buf, 1)
aq.attn_forward(q, k, v, causal=causal, train=train, workspace=ws, operands_staged=True)
torch.cuda.synchronize()
fn(buf, 0)
v = list(buf)
tiles = v[10]
# S wait / TMEM ld: both passes (all items but the last one's pass 2), see the kernel
names = ["S wait", "TMEM ld", "p1 math", "epi: TMEM ld", "-", "p2 exp", "p2 P_EMPTY wait", "p2 quant+st",
         "p2 fence+arrive", "total"]
print("per warp-tile cycles (averaged over warps):")
for i, n in enumerate(names):
    if n != "-":
        print(f"  {n:18s} {v[i] / tiles:9.1f}")
for i, n in zip(range(12, 16), ["merge (m, l)", "O_FULL wait", "epilogue ld+st", "next item"]):
    print(f"  {n:18s} {v[i] / tiles:9.1f}")
acc = sum(v[i] for i in (0, 1, 2, 5, 6, 7, 8, 12, 13, 14, 15))  # [3] is inside [14]
print(f"  {'unaccounted':18s} {(v[9] - acc) / tiles:9.1f}")
print("warps", v[11], "tiles", tiles)
