# bulk-copy landing slots beside the register window (SC_BULK_SLOTS / SC_EB_F32 builds):
# (the build knob was removed from sc_filter.cu after the measurement; check out the commit named in profiles/r01_chunk_l2_sweep.md to rerun)
# parity of one variant, then c3 pass times of every variant against the default build
L=$PWD/paper_1509_08863_b200
SC_B200_LIB=$L/libsc_b200_b6e5.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "filter_f32_parity or column_chunking or random_cases" > gpurun_out/t_bulk.log 2>&1
tail -n 2 gpurun_out/t_bulk.log
o=gpurun_out/sweep_bulk.txt; : > $o
for lib in libsc_b200 libsc_b200_b4e6 libsc_b200_b6e5 libsc_b200_b8e4 libsc_b200_b4e4 libsc_b200; do
  SC_B200_LIB=$L/$lib.so timeout 300 python tools/sweep_filter.py --workload c3_sbm1m --chunks 32 --reps 3 --tag $lib >> $o 2>&1
done
cat $o | cut -c1-140
