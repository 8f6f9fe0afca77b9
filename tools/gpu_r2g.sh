#!/bin/bash
O=gpurun_out/r2g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --deselect tests/test_gpu_fullsize.py > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -25 $O/pytest.log
SNP_SMALL=0 timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --deselect tests/test_gpu_fullsize.py > $O/pytest_nosmall.log 2>&1; echo pytest_rc=$? >> $O/pytest_nosmall.log
tail -3 $O/pytest_nosmall.log
python tools/bench_pi.py > $O/pi.jsonl 2>&1; tail -5 $O/pi.jsonl
SNP_SMALL=0 python tools/bench_pi.py > $O/pi_nosmall.jsonl 2>&1; tail -3 $O/pi_nosmall.jsonl
timeout 900 python bench.py --config 3 --steps 6 --warmup 2 --no-cpu --no-e2e > $O/bench_c3.log 2>&1; tail -c 400 $O/bench_c3.log
