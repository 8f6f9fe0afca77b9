#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
AB_STEPS=10 AB_ARGS="--warmup 3" bash tools/gpu_ab.sh r2i_ab "" "|SNP_KC_FLATQ=1" "|SNP_TC_MINB=4" "|SNP_KC_FLATQ=1 SNP_TC_MINB=4"
python tools/bench_pi.py > $O/pi.jsonl 2>&1; cat $O/pi.jsonl | cut -c1-300
timeout 900 python tools/drift_probe.py > $O/drift.jsonl 2> $O/drift.err; tail -2 $O/drift.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x --timeout 600 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
