mkdir -p gpurun_out/s29
for i in 1 2; do
for v in "4:4" "4:8" "5:5" "5:8" "6:6" "6:8" "8:8"; do
  IFS=: read hb cb <<< "$v"
  MGNN_HOP_GRID_BPS=$hb MGNN_COMPACT_BPS=$cb timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --prio-a --tag "prioA hop$hb comp$cb" >> gpurun_out/s29/exp.jsonl 2>>gpurun_out/s29/err.log
done; done
