mkdir -p gpurun_out/s43
export MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5
for i in 1 2; do
for g in -1 0 1; do
  MGNN_GATHER_GATE=$g timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --tag "gate$g" >> gpurun_out/s43/exp.jsonl 2>>gpurun_out/s43/err.log
done
for g in 0 1; do
  MGNN_GATHER_GATE=$g timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --tag "gate$g noprio" >> gpurun_out/s43/exp.jsonl 2>>gpurun_out/s43/err.log
done; done
