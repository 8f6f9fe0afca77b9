#!/bin/bash
# shared-memory wavefronts of the store-phase pattern; verification with 128-thread CTAs
O=gpurun_out/r3r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lds_probe tools/lds_probe.cu && /tmp/lds_probe > $O/lds_probe.txt 2>&1
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum --csv /tmp/lds_probe > $O/lds_probe_ncu.csv 2>&1
cat $O/lds_probe.txt
AB_ARGS="--config 3" AB_STEPS=6 bash tools/gpu_ab.sh r3r_c3 "X=1" "X=2|SNP_VM_THREADS=128"
