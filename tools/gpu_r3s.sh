#!/bin/bash
# level-0 upload over 1 vs 2 copy streams (e2e through the ABI), upload parity tests
O=gpurun_out/r3s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "upload or chunk or e2e or pinned or begin" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for NS in 1 2 3; do
  SNP_UPLOAD_STREAMS=$NS timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu > $O/e2e_ns$NS.log 2>&1
  python - $O/e2e_ns$NS.log $NS <<'PY'
import json, sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')][-1]
print('streams', sys.argv[2], 'e2e', d['e2e']['value'], d['e2e']['breakdown_s'])
PY
done
