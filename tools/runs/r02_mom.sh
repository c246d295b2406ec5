# round 2: moments pass (CSR MOMENTS kernel) vs SELL fp64 filter pass of the same width
python tools/time_moments.py c3_sbm1m 32
