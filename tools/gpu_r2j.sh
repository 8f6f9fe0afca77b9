#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
AB_STEPS=20 AB_ARGS="--warmup 5" bash tools/gpu_ab.sh r2j_ab "" "|SNP_TC_L2PF=2" "|SNP_KC_L2PF=2"
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 1200 -k "config4" > $O/pytest_c4.log 2>&1; tail -2 $O/pytest_c4.log
