mkdir -p gpurun_out/s44
for i in 1 2 3; do
  BENCH_PACE=1 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s44/pace_$i.json 2>>gpurun_out/s44/err.log
  BENCH_PACE=0 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s44/nopace_$i.json 2>>gpurun_out/s44/err.log
done
