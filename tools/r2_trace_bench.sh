# rational XNysTrace-exp bench line (Fig. 7 shape on C3) + the non-slow GPU suite
timeout 1200 python bench.py --trace --steps 1 --warmup 1 > gpurun_out/trace_rational_c3.json 2> gpurun_out/trace_rational_c3.err; tail -3 gpurun_out/trace_rational_c3.err
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -3
