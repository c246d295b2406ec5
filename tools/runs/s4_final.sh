#!/bin/bash
# session 4 final state: full GPU suite + smoke + bench lines (configs[3] default, configs[4], configs[2])
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/f_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_gputests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_bench_c3.json 2> gpurun_out/f_bench_c3.err; echo "bench_rc=$?" >> gpurun_out/f_bench_c3.err
timeout 1200 python bench.py --workload c4_sbm10m --steps 3 --warmup 3 --no-stability > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err; echo "c4_rc=$?" >> gpurun_out/f_bench_c4.err
timeout 600 python bench.py --workload c2_sbm100k > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.err; echo "c2_rc=$?" >> gpurun_out/f_bench_c2.err
tail -3 gpurun_out/f_gputests.log; tail -2 gpurun_out/f_smoke.log
for f in c3 c4 c2; do head -c 400 gpurun_out/f_bench_$f.json; echo; tail -1 gpurun_out/f_bench_$f.err; done
