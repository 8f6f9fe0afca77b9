#!/bin/bash
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; tail -2 $O/pytest.log
python tools/bench_pi.py > $O/pi.jsonl 2>&1; cut -c1-260 $O/pi.jsonl
timeout 900 python bench.py --config 3 --steps 8 --warmup 2 --no-e2e --no-cpu > $O/bench_c3.log 2>&1; tail -c 300 $O/bench_c3.log
