mkdir -p gpurun_out/s37
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "eviction or arxiv or cfg1" > gpurun_out/s37/tests.log 2>&1; echo tests $? >> gpurun_out/s37/status
for i in 1 2; do
for c in arxiv cfg1; do
  for g in flat tma; do
    MGNN_GATHER=$g timeout 600 python bench.py --config $c --no-extras --no-cpu-baseline > gpurun_out/s37/${c}_${g}_$i.json 2>>gpurun_out/s37/err.log
  done
done; done
for i in 1 2; do
  timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s37/products_fused_$i.json 2>>gpurun_out/s37/err.log
  MGNN_FUSED_DECAY=0 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/s37/products_nofused_$i.json 2>>gpurun_out/s37/err.log
done
