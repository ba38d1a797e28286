mkdir -p gpurun_out/s27
export MGNN_FLAT_BPS=16
timeout 300 python tools/exp_window.py --config products --windows 12 --tag "bps16 norelabel" >> gpurun_out/s27/exp.jsonl 2>>gpurun_out/s27/err.log
timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --tag "bps16 relabel" >> gpurun_out/s27/exp.jsonl 2>>gpurun_out/s27/err.log
MGNN_KPROF_TIMELINE=1 timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 4 --kprof --tag bps16 > /dev/null 2> gpurun_out/s27/timeline_bps16.txt
