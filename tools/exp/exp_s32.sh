mkdir -p gpurun_out/s32
for i in 1 2; do
for ge in "" "--gather-events"; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 20 $ge --tag "base $ge" >> gpurun_out/s32/exp.jsonl 2>>gpurun_out/s32/err.log
  MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5 timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 20 --prio-a $ge --tag "tuned $ge" >> gpurun_out/s32/exp.jsonl 2>>gpurun_out/s32/err.log
done; done
