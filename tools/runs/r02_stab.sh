# round 2: bisect the sc_stability failure
python tools/stab_probe.py
SC_KMEANS_TC=0 python tools/stab_probe.py
SC_KMEANS_AMB_WARP=0 python tools/stab_probe.py
SC_KMEANS_TC=0 SC_KMEANS_AMB_WARP=0 python tools/stab_probe.py
SC_STABILITY_WORKERS=1 python tools/stab_probe.py
