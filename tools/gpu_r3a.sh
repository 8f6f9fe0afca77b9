#!/bin/bash
# fresh source-level ncu of K-c at config 4 (F = 2^20) and of K-c + verification at config 3
O=gpurun_out/r3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > $O/bench_c4.log 2>&1; tail -c 400 $O/bench_c4.log
timeout 600 python bench.py --config 3 --steps 6 --warmup 2 --no-e2e --no-cpu > $O/bench_c3.log 2>&1; tail -c 400 $O/bench_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_materialize_bs" -s 4 -c 1 \
  -o $O/kc4 python bench.py --F 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu4.log 2>&1; tail -2 $O/ncu4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_materialize_bs|k_verify|k_expand" -s 6 -c 4 \
  -o $O/kc3 python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu3.log 2>&1; tail -2 $O/ncu3.log
ls -la $O
