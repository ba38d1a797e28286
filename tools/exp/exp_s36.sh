mkdir -p gpurun_out/s36
timeout 600 python -m pytest tests/test_gpu_variants.py -q -m gpu -k "FLAT" > gpurun_out/s36/tests.log 2>&1; echo tests $? >> gpurun_out/s36/status
export MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5
for i in 1 2; do
for u in 4 12 13; do
  MGNN_FLAT_UNR=$u timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --tag "tuned unr$u" >> gpurun_out/s36/exp.jsonl 2>>gpurun_out/s36/err.log
  [ $i = 1 ] && MGNN_FLAT_UNR=$u timeout 300 python tools/exp_window.py --config products --serial --windows 10 --tag "serial unr$u" >> gpurun_out/s36/exp.jsonl 2>>gpurun_out/s36/err.log
done; done
