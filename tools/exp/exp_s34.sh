mkdir -p gpurun_out/s34
export MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5
for i in 1 2; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --tag "tuned" >> gpurun_out/s34/exp.jsonl 2>>gpurun_out/s34/err.log
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --score-prio -2 --tag "tuned scoreD-2" >> gpurun_out/s34/exp.jsonl 2>>gpurun_out/s34/err.log
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --score-prio -3 --tag "tuned scoreD-3" >> gpurun_out/s34/exp.jsonl 2>>gpurun_out/s34/err.log
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --score-prio -1 --tag "tuned scoreD-1" >> gpurun_out/s34/exp.jsonl 2>>gpurun_out/s34/err.log
done
