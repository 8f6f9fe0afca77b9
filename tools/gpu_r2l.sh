#!/bin/bash
O=gpurun_out/r2l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_generated.py -q -x --timeout 600 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 1200 -k config3 > $O/pytest_c3.log 2>&1; tail -2 $O/pytest_c3.log
timeout 900 python bench.py --config 3 --steps 8 --warmup 2 --no-e2e --no-cpu > $O/bench_c3.log 2>&1; tail -c 300 $O/bench_c3.log
SNP_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu > $O/bench_trace.log 2> $O/bench_trace.err; grep begin $O/bench_trace.err; tail -c 600 $O/bench_trace.log
