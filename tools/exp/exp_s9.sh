mkdir -p gpurun_out/s9
timeout 600 python -m pytest tests/test_gpu_variants.py -q -m gpu -k "flat" > gpurun_out/s9/tests.log 2>&1; echo tests $? >> gpurun_out/s9/status
for i in 1 2; do
for v in "tma" "flat:3" "flat:4"; do
  g=${v%%:*}; b=${v##*:}
  if [ $g = tma ]; then unset MGNN_GATHER; else export MGNN_GATHER=flat MGNN_FLAT_BPS=$b; fi
  timeout 300 python tools/exp_window.py --config products --relabel-stream --windows 12 --tag "$v" >> gpurun_out/s9/exp.jsonl 2>>gpurun_out/s9/err.log
  [ $i = 1 ] && timeout 300 python tools/exp_window.py --config products --serial --windows 8 --tag "$v serial" >> gpurun_out/s9/exp.jsonl 2>>gpurun_out/s9/err.log
done; done
unset MGNN_GATHER
for v in "tma" "flat:3"; do
  g=${v%%:*}; b=${v##*:}
  if [ $g = tma ]; then unset MGNN_GATHER; else export MGNN_GATHER=flat MGNN_FLAT_BPS=$b; fi
  for c in reddit papers_s32 arxiv; do timeout 300 python tools/exp_window.py --config $c --relabel-stream --windows 12 --tag "$v" >> gpurun_out/s9/exp.jsonl 2>>gpurun_out/s9/err.log; done
done
