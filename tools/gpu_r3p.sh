#!/bin/bash
# K-c with 8-warp CTAs for m <= 4096 (A/B at config 3), parity
O=gpurun_out/r3p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
AB_ARGS="--config 3" AB_STEPS=6 bash tools/gpu_ab.sh r3p_c3 "SNP_KC_CTA_WARPS=32" "SNP_KC_CTA_WARPS="
