mkdir -p gpurun_out/s18
for o in gather,score,sample gather,sample,score sample,gather,score; do
  timeout 300 python tools/exp_order.py --config products --order $o >> gpurun_out/s18/exp.jsonl 2>>gpurun_out/s18/err.log
  MGNN_GATHER=tma timeout 300 python tools/exp_order.py --config products --order $o | sed 's/"config": "products"/"config": "products-tma"/' >> gpurun_out/s18/exp.jsonl 2>>gpurun_out/s18/err.log
done
