#!/bin/bash
# NARROW tensor-core K-a for 16/32-bit counts
O=gpurun_out/r3j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tc_expand or wide_counts or random_system_parity or tiny_random or exact_dedup or pi" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
AB_ARGS="--config 3" AB_STEPS=6 bash tools/gpu_ab.sh r3j_c3 "SNP_KERNELS=no_tc" "SNP_KERNELS="
