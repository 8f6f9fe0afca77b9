#!/bin/bash
# ncu: verification + NARROW K-c at config 3
O=gpurun_out/r3n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_verify_m|k_materialize_bs" -s 4 -c 2 \
  -o $O/v3 python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1; tail -2 $O/ncu.log
