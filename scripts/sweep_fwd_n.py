import sys; sys.path.insert(0, 'scripts'); sys.path.insert(0, '.')
from time_fwd import run
for N in (8192, 16384, 32768):
    for causal in (True, False):
        run(max(1, 65536 // N), 32, N, 128, causal, False, reps=5)
