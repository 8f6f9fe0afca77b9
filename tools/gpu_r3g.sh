#!/bin/bash
# config-3 launch list (per-kernel durations)
O=gpurun_out/r3g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_c3.csv python bench.py --config 3 --steps 3 --warmup 2 --no-e2e --no-cpu > $O/ncu.log 2>&1; tail -2 $O/ncu.log
