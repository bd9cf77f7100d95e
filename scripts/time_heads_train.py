"""K4 (training forward) at the per-GPU shard sizes of C4 under N-GPU head sharding (256 / N heads of N=4096 causal)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from time_fwd import run  # noqa: E402
for heads in (256, 128, 64, 32):
    run(1, heads, 4096, 128, True, True)
