#!/bin/bash
# bench variants on the current tree: reference arm, single-GPU partitioned path, configs[4] line
mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bm_ref.json 2> gpurun_out/bm_ref.err; echo "ref_rc=$?"
timeout 900 python bench.py --dist-path --no-cluster --no-stability --no-cpu-baseline > gpurun_out/bm_dist.json 2> gpurun_out/bm_dist.err; echo "dist_rc=$?"
timeout 1800 python bench.py --workload c4_sbm10m --no-stability > gpurun_out/bm_c4.json 2> gpurun_out/bm_c4.err; echo "c4_rc=$?"
head -c 300 gpurun_out/bm_ref.json; echo; head -c 300 gpurun_out/bm_dist.json; echo; head -c 600 gpurun_out/bm_c4.json; tail -3 gpurun_out/bm_dist.err gpurun_out/bm_c4.err
