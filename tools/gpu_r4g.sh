#!/bin/bash
# K-c: store-program scratch dropped (cooperative stores), 72-byte staging rows (A/B); parity
O=gpurun_out/r4g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse_and_dense or random_system_parity or uint8_large or overflow or wide_counts or global_emit" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
AB_STEPS=8 bash tools/gpu_ab.sh r4g_c4 "X=0" "X=1|SNP_KC_XS72=1"
