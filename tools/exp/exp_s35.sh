mkdir -p gpurun_out/s35
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py -q -m gpu -k "eviction or products or arxiv" > gpurun_out/s35/tests.log 2>&1; echo tests $? >> gpurun_out/s35/status
export MGNN_HOP_GRID_BPS=5 MGNN_COMPACT_BPS=5
for i in 1 2; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --tag "tuned cta" >> gpurun_out/s35/exp.jsonl 2>>gpurun_out/s35/err.log
  MGNN_SORT_CTA=0 timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 40 --prio-a --tag "tuned multiblock" >> gpurun_out/s35/exp.jsonl 2>>gpurun_out/s35/err.log
done
timeout 300 python tools/exp_window.py --config products --serial --windows 12 --tag "serial cta" >> gpurun_out/s35/exp.jsonl 2>>gpurun_out/s35/err.log
MGNN_SORT_CTA=0 timeout 300 python tools/exp_window.py --config products --serial --windows 12 --tag "serial multiblock" >> gpurun_out/s35/exp.jsonl 2>>gpurun_out/s35/err.log
