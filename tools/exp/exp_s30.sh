mkdir -p gpurun_out/s30
for i in 1 2; do
for c in arxiv reddit papers_s32 cfg1; do
  timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 --tag "base" >> gpurun_out/s30/exp.jsonl 2>>gpurun_out/s30/err.log
  MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5 timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 --prio-a --tag "prioA hop5 comp5" >> gpurun_out/s30/exp.jsonl 2>>gpurun_out/s30/err.log
  MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5 timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 --tag "hop5 comp5" >> gpurun_out/s30/exp.jsonl 2>>gpurun_out/s30/err.log
done; done
