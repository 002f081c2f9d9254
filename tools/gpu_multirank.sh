# loopback multi-rank parity on one GPU, then the rest of the GPU suite (fast tests only)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -p no:cacheprovider 2>&1 | tail -30
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider 2>&1 | tail -5
