#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --dist-path --no-cluster --no-stability --no-cpu-baseline > gpurun_out/bd_dist.json 2> gpurun_out/bd_dist.err; echo "dist_rc=$?"
timeout 900 python bench.py --dist-path --exchange nccl --no-cluster --no-stability --no-cpu-baseline > gpurun_out/bd_nccl.json 2> gpurun_out/bd_nccl.err; echo "nccl_rc=$?"
head -c 700 gpurun_out/bd_dist.json; echo; head -c 400 gpurun_out/bd_nccl.json; tail -n 3 gpurun_out/bd_dist.err
