mkdir -p gpurun_out/s28
for fb in 4 16; do
for hb in 2 3 4; do
  MGNN_FLAT_BPS=$fb MGNN_HOP_GRID_BPS=$hb MGNN_COMPACT_BPS=$hb timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --prio-a --tag "prioA flat$fb hop$hb" >> gpurun_out/s28/exp.jsonl 2>>gpurun_out/s28/err.log
done; done
MGNN_FLAT_BPS=16 MGNN_HOP_GRID_BPS=3 MGNN_COMPACT_BPS=3 timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --prio-a --prio-b --tag "prioAB flat16 hop3" >> gpurun_out/s28/exp.jsonl 2>>gpurun_out/s28/err.log
