#!/bin/bash
# tiny-frontier BFS at 128 threads (A/B), Π tests; config-3 verify ncu
O=gpurun_out/r3i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
tail -1 $O/build.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pi or tiny_random or small" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
SNP_SMALL_NT=1024 python tools/bench_pi.py > $O/pi_1024.jsonl 2>&1; cut -c1-200 $O/pi_1024.jsonl
python tools/bench_pi.py > $O/pi_128.jsonl 2>&1; cut -c1-200 $O/pi_128.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_verify_m|k_verify_need|k_expand_t" -s 6 -c 3 \
  -o $O/v3 python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1; tail -2 $O/ncu.log
