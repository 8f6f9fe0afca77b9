#!/bin/bash
# NARROW K-c (16/32-bit counts as bytes): parity + config-3 A/B
O=gpurun_out/r3e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_counts or uint8_large or global_emit or random_system_parity or tiny_random" > $O/pytest.log 2>&1; tail -5 $O/pytest.log
AB_ARGS="--config 3" AB_STEPS=6 bash tools/gpu_ab.sh r3e_c3 "SNP_KERNELS=kc_wide_exact" "SNP_KERNELS="
