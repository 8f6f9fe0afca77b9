#!/bin/bash
# verification with a decoder warp (pipelined decode)
O=gpurun_out/r3u; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "exact_dedup or random_system_parity or wide_counts or tiny" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for st in 6 8; do
timeout 600 python bench.py --config 3 --steps $st --warmup 2 --no-e2e --no-cpu > $O/bench_c3_$st.log 2>&1
python - $O/bench_c3_$st.log <<'PY'
import json, sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')][-1]
print('config3', d['steps'], d['value'], d['ms_per_step'], d['phase_ms_per_step'], d['digest'], d['step_roofline']['frac'])
PY
done
