#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
python tools/bench_pi.py > $O/pi.jsonl 2>&1; cat $O/pi.jsonl | cut -c1-400
timeout 600 nsys --version > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_verify_s" -s 2 -c 1 \
  -o $O/prof_verify python bench.py --config 3 --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu_v.log 2>&1; echo ncu_rc=$? >> $O/ncu_v.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_small_bfs" -s 3 -c 1 \
  -o $O/prof_small python tools/bench_pi.py > $O/ncu_s.log 2>&1; echo ncu_rc=$? >> $O/ncu_s.log
