mkdir -p gpurun_out/s40
for i in 1 2; do
  for p in 1 10 100; do
    BENCH_CLOCK_PERIOD_MS=$p timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s40/p${p}_$i.json 2>>gpurun_out/s40/err.log
  done
done
