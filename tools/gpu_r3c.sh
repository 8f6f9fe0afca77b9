#!/bin/bash
# tensor-core K-c store: parity, A/B vs byte permutes
O=gpurun_out/r3c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_generated.py -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
AB_STEPS=8 bash tools/gpu_ab.sh r3c "SNP_KERNELS=kc_prmt" "SNP_KERNELS="
