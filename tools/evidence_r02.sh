#!/bin/bash
# Round-2 evidence on the GPU box: per-config bench lines, ncu launch lists + DRAM traffic tables at
# HEAD, the bench command's launch list, and (part "multi") the 2- / 4-GPU tests and scaling lines.
#
#   tools/evidence_r02.sh single    # 1 GPU: bench lines, ncu tables
#   tools/evidence_r02.sh traffic   # 1 GPU: only the per-config ncu DRAM tables
#   tools/evidence_r02.sh final     # 1 GPU: GPU suite, smoke, bench lines of every config, launch list
#   tools/evidence_r02.sh multi N   # N GPUs: test_multi + bench at N for products (P=2N) and papers_s32 (P=8)
# Output under gpurun_out/evidence/ (copied into profiles/r02/ by hand after review).
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
part=${1:-single}

if [ "$part" = single ] || [ "$part" = traffic ]; then
    # 1. per-config DRAM traffic of every library kernel (cache-control none: in-situ bytes); the tables
    #    also go to profiles/r02/ on this box so the bench lines below read the HEAD numbers
    for c in cfg1 arxiv reddit products papers_s32; do
        timeout 900 ncu --cache-control none --clock-control none --kernel-name regex:"k_" \
            --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
            -s $([ $c = papers_s32 ] && echo 250 || echo 100) -c 100 --csv --log-file $OUT/launches_$c.csv \
            python tools/exp_window.py --config $c --relabel-stream --tuned --windows 12 > $OUT/ncu_$c.log 2>&1
        python tools/ncu_hbm_table.py $OUT/launches_$c.csv --json $OUT/traffic_$c.json --config $c \
            > $OUT/table_$c.txt 2>&1 && cp $OUT/traffic_$c.json profiles/r02/traffic_$c.json
    done
    [ "$part" = traffic ] && exit 0
    # 2. bench lines (the driver's default command first), each under its own timeout
    timeout 900 python bench.py > $OUT/bench_products.json 2> $OUT/bench_products.err
    for c in cfg1 arxiv reddit papers_s32; do
        timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
    done
    timeout 1500 python bench.py --config papers --no-cpu-baseline --steps 10 --warmup 3 --runs 1 \
        > $OUT/bench_papers.json 2> $OUT/bench_papers.err
    # 3. launch list of the bench's own default command (the gpu__time_duration pass of B200_PROFILING.md)
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 400 --csv \
        --log-file $OUT/bench_launches.csv python bench.py --steps 3 --warmup 3 --runs 1 --no-extras \
        --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
    python tools/launch_summary.py $OUT/bench_launches.csv > $OUT/bench_launches_summary.txt 2>&1
    exit 0
fi

if [ "$part" = final ]; then
    # end-of-round lines at HEAD: GPU suite, smoke, every config's bench line, full papers, the bench
    # command's launch list (traffic tables: part "traffic")
    timeout 1800 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $OUT/status
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status
    timeout 900 python bench.py > $OUT/bench_products.json 2> $OUT/bench_products.err
    for c in cfg1 arxiv reddit papers_s32; do
        timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
    done
    timeout 1500 python bench.py --config papers --no-cpu-baseline --steps 10 --warmup 3 --runs 1 \
        > $OUT/bench_papers.json 2> $OUT/bench_papers.err
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 400 --csv \
        --log-file $OUT/bench_launches.csv python bench.py --steps 3 --warmup 3 --runs 1 --no-extras \
        --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
    python tools/launch_summary.py $OUT/bench_launches.csv > $OUT/bench_launches_summary.txt 2>&1
    exit 0
fi

if [ "$part" = multi ]; then
    N=${2:-2}
    timeout 1500 python -m pytest tests/test_multi.py -q -m gpu -s > $OUT/test_multi_n$N.log 2>&1
    tail -3 $OUT/test_multi_n$N.log
    nvidia-smi topo -m > $OUT/topo_n$N.txt 2>&1
    for c in products papers_s32; do
        timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
            --master-port 29533 bench.py --gpus $N --config $c --no-cpu-baseline \
            > $OUT/bench_${c}_n$N.json 2> $OUT/bench_${c}_n$N.err
        tail -c 600 $OUT/bench_${c}_n$N.json
    done
    exit 0
fi
echo "unknown part $part"
exit 2
