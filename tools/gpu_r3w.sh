#!/bin/bash
# K-a: mbarrier addresses precomputed (A/B)
O=gpurun_out/r3w; mkdir -p $O
AB_STEPS=8 bash tools/gpu_ab.sh r3w_c4 "X=0|SNP_TC_UADDR=0" "X=1"
