#!/bin/bash
# One GPU session: build, box facts, the GPU test suite (with durations), the
# default bench line.  TAG names gpurun_out/$TAG; PYTEST_ARGS / BENCH_ARGS /
# SKIP_TESTS / SKIP_BENCH adjust it.
TAG=${1:-sess}
O=gpurun_out/$TAG; mkdir -p $O
{ nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)|Socket"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > $O/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -30 $O/build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -x -q --durations=25 ${PYTEST_ARGS} > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
  tail -40 $O/pytest.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1200 python bench.py ${BENCH_ARGS} > $O/bench.log 2>&1; echo bench_rc=$? >> $O/bench.log
  tail -c 3000 $O/bench.log
fi
cat $O/box.txt
