mkdir -p gpurun_out/s17
python -c "import torch; print(torch.cuda.Stream.priority_range())" > gpurun_out/s17/prio.txt 2>&1
for i in 1 2; do
for c in products reddit arxiv papers_s32; do
  for p in "" "--prio-b"; do
  timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 $p --tag "flat $p" >> gpurun_out/s17/exp.jsonl 2>>gpurun_out/s17/err.log
  done
done; done
