#!/bin/bash
# multi-GPU path: aggregated owner counters (pack / hist / keep); dist tests + 1-rank bench
O=gpurun_out/r3t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 1 --dist --steps 4 --warmup 2 --no-cpu --no-e2e > $O/bench_dist1.log 2>&1
python - <<'PY'
import json
d=[json.loads(l) for l in open('gpurun_out/r3t/bench_dist1.log') if l.startswith('{')][-1]
print('dist1', d['value'], d['ms_per_step'], d['phase_ms_per_step'], d['digest'])
PY
