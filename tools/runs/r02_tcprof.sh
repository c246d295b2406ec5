# round 2: per-phase cycle split of the tensor screen (thread 0 of every CTA), configs[3] pipeline
SC_TC_PROFILE=1 python tools/time_cluster.py c3_sbm1m 1 2>&1 | grep -E "cycles per CTA|sc_cluster" | tail -3
