mkdir -p gpurun_out/s52
for i in 1 2; do
for gr in 4 3 2; do
  MGNN_FLAT_GRID=$gr timeout 300 python tools/exp_window.py --config products --relabel-stream --tuned --windows 30 --tag "grid$gr" >> gpurun_out/s52/exp.jsonl 2>>gpurun_out/s52/err.log
done; done
