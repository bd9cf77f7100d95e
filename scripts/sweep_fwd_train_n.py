"""Kernel time of the training forward (K4) and the inference forward (K5)
against sequence length at a fixed 64 K tokens x 32 heads, causal and not:
the per-item overhead shows up as the gap to the long-row rate. GPU."""
import sys
sys.path.insert(0, 'scripts')
sys.path.insert(0, '.')
from time_fwd import run  # noqa: E402

for N in (1024, 2048, 4096, 8192, 16384):
    for causal in (True, False):
        for train in (True, False):
            run(65536 // N, 32, N, 128, causal, train, reps=5)
