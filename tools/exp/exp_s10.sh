mkdir -p gpurun_out/s10
timeout 600 python -m pytest tests/test_gpu_variants.py -q -m gpu -k "flat" > gpurun_out/s10/tests.log 2>&1; echo tests $? >> gpurun_out/s10/status
for i in 1 2; do
for v in "tma" "flat:4:4" "flat:4:6" "flat:3:6" "flat:5:2" "flat:4:2"; do
  IFS=: read g b u <<< "$v"
  if [ $g = tma ]; then unset MGNN_GATHER; else export MGNN_GATHER=flat MGNN_FLAT_BPS=$b MGNN_FLAT_UNR=$u; fi
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --tag "$v" >> gpurun_out/s10/exp.jsonl 2>>gpurun_out/s10/err.log
  [ $i = 1 ] && timeout 300 python tools/exp_window.py --config products --serial --windows 8 --tag "$v serial" >> gpurun_out/s10/exp.jsonl 2>>gpurun_out/s10/err.log
done; done
