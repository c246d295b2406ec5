#!/bin/bash
# full verification on the current tree: GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fb_gputests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/fb_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fb_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/fb_smoke.log
timeout 900 python bench.py > gpurun_out/fb_bench.json 2> gpurun_out/fb_bench.err; echo "bench_rc=$?" >> gpurun_out/fb_bench.err
tail -3 gpurun_out/fb_gputests.log; tail -2 gpurun_out/fb_smoke.log; head -c 300 gpurun_out/fb_bench.json
