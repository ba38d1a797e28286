mkdir -p gpurun_out/s55
MGNN_LIB=$PWD/paper_2410_22697_b200/libmgnn_sel16.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "eviction or cfg1_windows" > gpurun_out/s55/tests16.log 2>&1; echo tests16 $? >> gpurun_out/s55/status
for i in 1 2; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --tuned --windows 30 --tag "sel8" >> gpurun_out/s55/exp.jsonl 2>>gpurun_out/s55/err.log
  MGNN_LIB=$PWD/paper_2410_22697_b200/libmgnn_sel16.so timeout 300 python tools/exp_window.py --config products --relabel-stream --tuned --windows 30 --tag "sel16" >> gpurun_out/s55/exp.jsonl 2>>gpurun_out/s55/err.log
done
timeout 300 python tools/exp_window.py --config products --serial --windows 10 --tag "sel8 serial" >> gpurun_out/s55/exp.jsonl 2>>gpurun_out/s55/err.log
MGNN_LIB=$PWD/paper_2410_22697_b200/libmgnn_sel16.so timeout 300 python tools/exp_window.py --config products --serial --windows 10 --tag "sel16 serial" >> gpurun_out/s55/exp.jsonl 2>>gpurun_out/s55/err.log
