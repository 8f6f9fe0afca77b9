#!/bin/bash
# parity (full file), K-a A/B: load-ahead 2 with 3 CTAs/SM
O=gpurun_out/r3q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
AB_STEPS=8 bash tools/gpu_ab.sh r3q_c4 "X=1" "X=2|SNP_TC_AHEAD=2 SNP_TC_MINB=3"
