mkdir -p gpurun_out/s25
for i in 1 2; do
for b in 4 16 64 256; do
  for p in "" "--prio-a"; do
  MGNN_FLAT_BPS=$b timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 $p --tag "bps$b $p" >> gpurun_out/s25/exp.jsonl 2>>gpurun_out/s25/err.log
  done
done; done
