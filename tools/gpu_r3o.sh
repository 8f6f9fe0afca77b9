#!/bin/bash
# verification with staged X|Y rows
O=gpurun_out/r3o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "exact_dedup or random_system_parity or wide_counts" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py --config 3 --steps 6 --warmup 2 --no-e2e --no-cpu > $O/bench_c3.log 2>&1
python - <<'PY'
import json
d=[json.loads(l) for l in open('gpurun_out/r3o/bench_c3.log') if l.startswith('{')][-1]
print('config3', d['value'], d['ms_per_step'], d['phase_ms_per_step'], d['digest'])
PY
