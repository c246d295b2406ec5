# stability scan on configs[2]: GPU utilisation sampled during the run, worker counts 1 / 8
python tools/time_stability.py c2_sbm100k > /dev/null 2>&1   # warm-up (graph cache, module load)
for wk in 8 1; do
  nvidia-smi --query-gpu=utilization.gpu,clocks.sm --format=csv,noheader -lms 50 > gpurun_out/util_$wk.csv &
  SMI=$!
  SC_STABILITY_WORKERS=$wk SC_STABILITY_TRACE=1 python tools/time_stability.py c2_sbm100k > gpurun_out/stab_$wk.log 2>&1
  kill $SMI
  echo "workers=$wk"; grep -v "^{" gpurun_out/stab_$wk.log | tail -n 4; grep "^{" gpurun_out/stab_$wk.log | cut -c1-120
  python -c "
import statistics
v=[int(l.split(',')[0].split()[0]) for l in open('gpurun_out/util_$wk.csv') if l.strip()]
print('util samples', len(v), 'mean', statistics.mean(v) if v else None, 'max', max(v) if v else None)"
done
