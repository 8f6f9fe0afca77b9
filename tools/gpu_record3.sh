#!/bin/bash
# Round-2 final recording session (one B200): everything judged goes to gpurun_out/$TAG
TAG=${1:-r02h}
O=gpurun_out/$TAG; mkdir -p $O
{ nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv; } > $O/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_config4.log 2>&1; echo bench_rc=$? >> $O/bench_config4.log
tail -c 300 $O/bench_config4.log
timeout 900 python bench.py --config 3 --steps 8 --warmup 2 --no-e2e > $O/bench_config3.log 2>&1; tail -c 200 $O/bench_config3.log
timeout 1500 python bench.py --config 5 --F 1000000 --steps 3 --warmup 1 --no-e2e --no-cpu > $O/bench_config5_slice.log 2>&1
tail -c 300 $O/bench_config5_slice.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 1 --dist --steps 4 --warmup 2 --no-cpu > $O/bench_dist1.log 2>&1; tail -c 300 $O/bench_dist1.log
timeout 600 python tools/bench_pi.py > $O/pi_warm.jsonl 2>&1
timeout 600 python tools/bench_pi.py > $O/pi_configs12.jsonl 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; tail -c 300 $O/bench_reference.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/launches.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_expand|k_nd_pass|k_materialize|k_patch" -s 8 -c 8 --log-file $O/dram_full.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/dram.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_expand_tc|k_materialize_bs" -s 4 -c 2 \
  -o $O/prof python bench.py --F 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
# compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset): the
# workload runs plain, with every result checked against the oracle
timeout 900 python tools/sanitize_workload.py > $O/sanitize_workload_plain.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 --durations=20 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
ls -la $O
