mkdir -p gpurun_out/s15
timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 10 --kprof --tag flat > gpurun_out/s15/exp.jsonl 2> gpurun_out/s15/kprof_flat.txt
MGNN_GATHER=tma timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 10 --kprof --tag tma >> gpurun_out/s15/exp.jsonl 2> gpurun_out/s15/kprof_tma.txt
timeout 300 python tools/exp_window.py --config products --serial --windows 10 --kprof --tag serial >> gpurun_out/s15/exp.jsonl 2> gpurun_out/s15/kprof_serial.txt
