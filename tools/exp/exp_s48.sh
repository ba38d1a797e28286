mkdir -p gpurun_out/s48
for c in reddit papers_s32 arxiv; do
for v in "4:4" "4:6" "3:8" "3:6" "4:2" "5:2"; do
  IFS=: read b u <<< "$v"
  MGNN_FLAT_BPS=$b MGNN_FLAT_UNR=$u timeout 300 python tools/exp_window.py --config $c --relabel-stream --tuned --windows 30 --tag "flat$b:$u" >> gpurun_out/s48/exp.jsonl 2>>gpurun_out/s48/err.log
done; done
