#!/bin/bash
# K-c tail pass (A/B), parity
O=gpurun_out/r4a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "random_system_parity or global_emit or uint8_large or tc_expand or tiny or wide_counts" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
AB_STEPS=8 bash tools/gpu_ab.sh r4a_c4 "X=0|SNP_KC_TAILQ=0" "X=1"
AB_ARGS="--config 3" AB_STEPS=6 bash tools/gpu_ab.sh r4a_c3 "X=0|SNP_KC_TAILQ=0" "X=1"
