mkdir -p gpurun_out/s38
for i in 1 2 3; do
  timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s38/ev_$i.json 2>>gpurun_out/s38/err.log
  timeout 600 python bench.py --no-extras --no-cpu-baseline --no-gather-events > gpurun_out/s38/noev_$i.json 2>>gpurun_out/s38/err.log
done
