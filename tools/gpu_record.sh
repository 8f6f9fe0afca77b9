#!/bin/bash
# One recording session on the GPU box (results under gpurun_out/$TAG):
# parity tests, smoke, the default bench line (e2e + cpu_baseline), the
# per-launch device-time list, the dram-bytes capture for roofline.traffic,
# and a full ncu capture of the two hot kernels at F = 2^20.
TAG=${1:-rec}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench_rc=$? >> $O/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_expand|k_nd_pass|k_materialize|k_patch" -s 8 -c 8 --log-file $O/dram_full.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/dram.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_expand_tc|k_materialize_bs" -s 4 -c 2 \
  -o $O/prof python bench.py --F 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
tail -2 $O/pytest.log; tail -2 $O/smoke.log; tail -c 600 $O/bench.log; ls -la $O
