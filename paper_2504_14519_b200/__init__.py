"""SlimPipe sliced-1F1B step on B200 (see README.md / DESIGN.md)."""
import os

# One hardware work queue per CUDA stream: the executor runs up to ten streams
# per rank, and shared queues let a waiting stream stall an unrelated one.
# Takes effect only if no CUDA context exists yet (set it in the environment
# to be sure).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
