#!/bin/bash
# config 3 rerun (the r02h last level had a 16 ms host-side spike)
O=gpurun_out/r4c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for k in 1 2; do
timeout 900 python bench.py --config 3 --steps 8 --warmup 2 --no-e2e > $O/bench_config3_$k.log 2>&1
python - $O/bench_config3_$k.log <<'PY'
import json, sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')][-1]
print('config3', d['value'], d['ms_per_step'], d['step_roofline']['frac'], [l['ms'] for l in d['levels']])
PY
done
