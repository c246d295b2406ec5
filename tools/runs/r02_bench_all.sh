#!/bin/bash
# round-2 bench lines of the other configs and the R16 graphs
mkdir -p gpurun_out
for wl in c0_sbm2k c1_gmm20k c2_sbm100k x_chunglu1m x_gmm2d1m_rcm; do
  timeout 900 python bench.py --workload $wl --no-stability > gpurun_out/ba_$wl.json 2> gpurun_out/ba_$wl.err; echo "$wl rc=$?"
done
for wl in c0_sbm2k c1_gmm20k c2_sbm100k x_chunglu1m x_gmm2d1m_rcm; do head -c 250 gpurun_out/ba_$wl.json; echo; done
