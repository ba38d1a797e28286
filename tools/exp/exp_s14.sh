mkdir -p gpurun_out/s14
for i in 1 2; do
for c in products arxiv; do
for v in "" "--score-after-sample"; do
  timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 $v --tag "flat $v" >> gpurun_out/s14/exp.jsonl 2>>gpurun_out/s14/err.log
  MGNN_PDL=0 timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 $v --tag "flat nopdl $v" >> gpurun_out/s14/exp.jsonl 2>>gpurun_out/s14/err.log
done; done; done
