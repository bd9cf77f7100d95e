"""K5 at the per-GPU shard sizes of C2 under N-GPU head sharding (128 / N heads of N=8192 causal)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from time_fwd import run  # noqa: E402
for heads in (128, 64, 32, 16):
    run(1, heads, 8192, 128, True, False)
