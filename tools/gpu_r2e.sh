#!/bin/bash
# r2e: TMA clip probe, config-3 bench with the int32 bit-sliced K-c + ncu of its
# kernels, compute-sanitizer (memcheck, racecheck, synccheck, initcheck)
O=gpurun_out/r2e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
./tools/tma_clip_probe.bin > $O/tma_probe.txt 2>&1; cat $O/tma_probe.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random_system_parity or config1 or tiny_random" > $O/pytest_quick.log 2>&1; tail -2 $O/pytest_quick.log
timeout 900 python bench.py --config 3 --steps 6 --warmup 2 --no-cpu > $O/bench_c3.log 2>&1; tail -c 1200 $O/bench_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_verify|k_materialize|k_expand|k_patch" -s 6 -c 8 \
  -o $O/prof_c3 python bench.py --config 3 --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu_c3.log 2>&1; echo ncu_rc=$? >> $O/ncu_c3.log
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_workload.py > $O/sanitizer_$T.txt 2>&1
  echo "$T rc=$?" >> $O/sanitizer_$T.txt; tail -3 $O/sanitizer_$T.txt
done
