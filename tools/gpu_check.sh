#!/bin/bash
# One GPU session: parity tests, smoke, default bench, ncu source profile of the
# two hot kernels at F = 2^20 (config 4 system).  Output under gpurun_out/$TAG.
TAG=${1:-run}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py $BENCH_ARGS > $O/bench.log 2>&1; echo bench_rc=$? >> $O/bench.log
fi
if [ -n "$NCU" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 2 -c 2 \
  -o $O/prof python bench.py --F 1048576 --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu.log 2>&1
echo ncu_rc=$? >> $O/ncu.log
fi
tail -3 $O/pytest.log 2>/dev/null; tail -2 $O/smoke.log 2>/dev/null; tail -c 1500 $O/bench.log 2>/dev/null; tail -3 $O/ncu.log 2>/dev/null
