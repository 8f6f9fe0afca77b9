#!/bin/bash
# final bench lines after the last K-c change (driver launch configuration)
O=gpurun_out/r4e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_config4.log 2>&1; tail -c 300 $O/bench_config4.log
timeout 900 python bench.py --config 3 --steps 8 --warmup 2 --no-e2e --no-cpu > $O/bench_config3.log 2>&1; tail -c 200 $O/bench_config3.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 1 --dist --steps 4 --warmup 2 --no-cpu > $O/bench_dist1.log 2>&1; tail -c 200 $O/bench_dist1.log
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_expand|k_nd_pass|k_materialize|k_patch" -s 8 -c 8 --log-file $O/dram_full.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/dram.log 2>&1
