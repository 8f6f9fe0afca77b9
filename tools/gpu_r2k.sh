#!/bin/bash
O=gpurun_out/r2k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
AB_STEPS=20 AB_ARGS="--warmup 5" bash tools/gpu_ab.sh r2k_ab "" "|SNP_KC_BRANCHLESS=1" "|SNP_KC_GUNROLL=1"
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_config4.log 2>&1; echo bench_rc=$? >> $O/bench_config4.log
tail -c 700 $O/bench_config4.log
