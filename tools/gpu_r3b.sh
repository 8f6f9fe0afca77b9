#!/bin/bash
# bank-conflict-free in-CSR rows: A/B on config 4 + config 3, parity subset
O=gpurun_out/r3b; mkdir -p $O
AB_STEPS=8 bash tools/gpu_ab.sh r3b "SNP_INPAD_BANKS=0" "SNP_INPAD_BANKS=1"
AB_ARGS="--config 3" AB_STEPS=6 bash tools/gpu_ab.sh r3b_c3 "SNP_INPAD_BANKS=0" "SNP_INPAD_BANKS=1"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
