#!/bin/bash
O=gpurun_out/r2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo bench_rc=$? >> $O/bench.log
tail -c 1500 $O/bench.log
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 --durations=12 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -18 $O/pytest.log
