#!/bin/bash
# r2c: K-c store / lane-order A/B, then the GPU tests except the full-size ones
O=gpurun_out/r2c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
AB_STEPS=6 bash tools/gpu_ab.sh r2c_ab "|SNP_KC_COOP=1 SNP_KC_PERM=0" "|SNP_KC_COOP=4 SNP_KC_PERM=0 SNP_KC_EDGEQ=0" \
  "|SNP_KC_COOP=4 SNP_KC_PERM=0 SNP_KC_EDGEQ=1" "" "|SNP_KC_COOP=3 SNP_KC_PERM=1"
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 --durations=15 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -30 $O/pytest.log
