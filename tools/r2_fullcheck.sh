# the driver's round-end GPU tiers on the current tree: the whole -m gpu suite (slow included) and smoke()
set -x
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r02_gputest.log 2>&1; tail -22 gpurun_out/r02_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; tail -3 gpurun_out/r02_smoke.log
