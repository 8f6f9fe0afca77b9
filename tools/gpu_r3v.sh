#!/bin/bash
# verification: count-major first-rule table; dist tests with snp_set_device
O=gpurun_out/r3v; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "exact_dedup or random_system_parity or wide_counts or tiny or dist" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for st in 6 8; do
timeout 600 python bench.py --config 3 --steps $st --warmup 2 --no-e2e --no-cpu > $O/bench_c3_$st.log 2>&1
python - $O/bench_c3_$st.log <<'PY'
import json, sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')][-1]
print('config3', d['steps'], d['value'], d['ms_per_step'], d['phase_ms_per_step'], d['digest'], d['step_roofline']['frac'])
PY
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 1 --dist --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_dist1.log 2>&1; tail -c 200 $O/bench_dist1.log
