#!/bin/bash
O=gpurun_out/r2m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 1200 -k config3 > $O/pytest_c3.log 2>&1; tail -2 $O/pytest_c3.log
timeout 900 python bench.py --config 3 --steps 8 --warmup 2 --no-e2e > $O/bench_c3.log 2>&1; tail -c 300 $O/bench_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_materialize_bs|k_verify" -s 4 -c 3 \
  -o $O/prof_c3 python bench.py --config 3 --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu_c3.log 2>&1; echo ncu_rc=$? >> $O/ncu_c3.log
