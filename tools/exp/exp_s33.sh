mkdir -p gpurun_out/s33
for i in 1 2; do
  timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s33/tuned_$i.json 2>>gpurun_out/s33/err.log
  timeout 600 python bench.py --no-extras --no-cpu-baseline --no-tuning > gpurun_out/s33/base_$i.json 2>>gpurun_out/s33/err.log
done
timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --tag "base" >> gpurun_out/s33/exp.jsonl 2>>gpurun_out/s33/err.log
MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5 timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --tag "tuned" >> gpurun_out/s33/exp.jsonl 2>>gpurun_out/s33/err.log
