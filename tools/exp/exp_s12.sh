mkdir -p gpurun_out/s12
for i in 1 2; do
for c in reddit papers_s32 arxiv cfg1; do
for v in "tma" "flat:4:4" "flat:4:6"; do
  IFS=: read g b u <<< "$v"
  if [ $g = tma ]; then unset MGNN_GATHER; else export MGNN_GATHER=flat MGNN_FLAT_BPS=$b MGNN_FLAT_UNR=$u; fi
  timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 --tag "$v" >> gpurun_out/s12/exp.jsonl 2>>gpurun_out/s12/err.log
done; done; done
