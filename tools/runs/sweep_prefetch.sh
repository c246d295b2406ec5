# A/B of the producer-warp L2 prefetch (SC_L2_PREFETCH) on c3_sbm1m, chunk widths 16..64
# (the build knob was removed from sc_filter.cu after the measurement; check out the commit named in profiles/r01_chunk_l2_sweep.md to rerun)
L=paper_1509_08863_b200
o=gpurun_out/sweep_pf.txt; : > $o
for rep in 1 2; do
for lib in libsc_b200 libsc_b200_nopf; do
  SC_B200_LIB=$PWD/$L/$lib.so python tools/sweep_filter.py --workload c3_sbm1m --chunks 32,16,24,64 --reps 3 --tag $lib >> $o 2>&1
done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> $o
