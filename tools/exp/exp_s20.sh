mkdir -p gpurun_out/s20
for n in 0 88 100 112 124; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --sm-split $n --tag "flat split$n" >> gpurun_out/s20/exp.jsonl 2>>gpurun_out/s20/err.log
done
for n in 100 112; do
  MGNN_FLAT_BPS=3 MGNN_FLAT_UNR=6 timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --sm-split $n --tag "flat36 split$n" >> gpurun_out/s20/exp.jsonl 2>>gpurun_out/s20/err.log
done
for v in "3:6" "3:8"; do
  IFS=: read b u <<< "$v"
  for h in 8 2; do
  MGNN_FLAT_BPS=$b MGNN_FLAT_UNR=$u MGNN_HOP_GRID_BPS=$h MGNN_COMPACT_BPS=$h timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --tag "flat$b$u hopgrid$h" >> gpurun_out/s20/exp.jsonl 2>>gpurun_out/s20/err.log
  done
done
