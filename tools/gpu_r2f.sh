#!/bin/bash
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
timeout 900 python bench.py --config 3 --steps 6 --warmup 2 --no-cpu --no-e2e > $O/bench_c3.log 2>&1; tail -c 600 $O/bench_c3.log
AB_STEPS=20 AB_ARGS="--warmup 5" bash tools/gpu_ab.sh r2f_ab "" "|SNP_KC_EPF=148"
timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_workload.py > $O/sanitizer_initcheck.txt 2>&1
echo "initcheck rc=$?" >> $O/sanitizer_initcheck.txt; tail -3 $O/sanitizer_initcheck.txt
