#!/bin/bash
# ncu of the tensor-core K-c store
O=gpurun_out/r3d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_materialize_bs" -s 4 -c 1 \
  -o $O/kctc python bench.py --F 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1; tail -2 $O/ncu.log
