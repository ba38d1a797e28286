mkdir -p gpurun_out/s56
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py -q -m gpu -k "eviction or cfg1 or products" > gpurun_out/s56/tests.log 2>&1; echo tests $? >> gpurun_out/s56/status
for i in 1 2; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --tuned --windows 30 --tag "cand16" >> gpurun_out/s56/exp.jsonl 2>>gpurun_out/s56/err.log
done
timeout 300 python tools/exp_window.py --config products --serial --windows 10 --tag "cand16 serial" >> gpurun_out/s56/exp.jsonl 2>>gpurun_out/s56/err.log
