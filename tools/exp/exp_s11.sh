mkdir -p gpurun_out/s11
for i in 1 2; do
for v in "tma" "flat:4:4" "flat:4:5" "flat:4:6"; do
  IFS=: read g b u <<< "$v"
  if [ $g = tma ]; then unset MGNN_GATHER; else export MGNN_GATHER=flat MGNN_FLAT_BPS=$b MGNN_FLAT_UNR=$u; fi
  for p in "" "--prio-b"; do
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 $p --tag "$v $p" >> gpurun_out/s11/exp.jsonl 2>>gpurun_out/s11/err.log
  done
  [ $i = 1 ] && [ $u = 5 ] && timeout 300 python tools/exp_window.py --config products --serial --windows 8 --tag "$v serial" >> gpurun_out/s11/exp.jsonl 2>>gpurun_out/s11/err.log
done; done
