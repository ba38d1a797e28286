mkdir -p gpurun_out/s16
timeout 600 python -m pytest tests/test_gpu_variants.py -q -m gpu -k "HOP_GRID" > gpurun_out/s16/tests.log 2>&1; echo tests $? >> gpurun_out/s16/status
for i in 1 2; do
for v in "8:8" "0:0" "6:6" "0:8" "8:0"; do
  IFS=: read h c <<< "$v"
  for p in "" "--prio-b"; do
  MGNN_HOP_GRID_BPS=$h MGNN_COMPACT_BPS=$c timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 $p --tag "hop$h comp$c $p" >> gpurun_out/s16/exp.jsonl 2>>gpurun_out/s16/err.log
  done
done; done
