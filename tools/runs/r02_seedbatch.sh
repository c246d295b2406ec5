#!/bin/bash
o=gpurun_out/r02_seedbatch.txt; : > $o
timeout 1500 python -m pytest tests -m gpu -x -q -k "kmeans or cluster or stability or pipeline" 2>&1 | tail -3 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
SC_CLUSTER_TRACE=1 timeout 600 python tools/time_cluster.py c3_sbm1m 3 >> $o 2>&1
SC_KMEANS_SEED_BATCH=0 SC_CLUSTER_TRACE=1 timeout 600 python tools/time_cluster.py c3_sbm1m 3 2>&1 | sed 's/^/nobatch /' >> $o
SC_CLUSTER_TRACE=1 timeout 600 python tools/time_cluster.py c3_sbm1m 3 2>&1 | sed 's/^/batch_again /' >> $o
timeout 600 python tools/time_stability.py 2>&1 | tail -3 >> $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> $o
cut -c1-250 $o
