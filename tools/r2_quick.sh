./tools/gather_ceiling 2>&1 | head -8
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider 2>&1 | tail -3
