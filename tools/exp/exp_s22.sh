mkdir -p gpurun_out/s22
for i in 1 2; do
timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --tag "flat pf" >> gpurun_out/s22/exp.jsonl 2>>gpurun_out/s22/err.log
timeout 300 python tools/exp_window.py --config products --serial --windows 8 --tag "flat pf serial" >> gpurun_out/s22/exp.jsonl 2>>gpurun_out/s22/err.log
done
for c in reddit arxiv papers_s32; do timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 --tag "flat pf" >> gpurun_out/s22/exp.jsonl 2>>gpurun_out/s22/err.log; done
