#!/bin/bash
# r2b: full GPU tests (incl. full-size parity), K-c store A/B, drift probe
O=gpurun_out/r2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 --durations=30 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
tail -45 $O/pytest.log
AB_STEPS=6 bash tools/gpu_ab.sh r2b_ab "|SNP_KC_COOP=1" "|SNP_KC_COOP=2"
timeout 900 python tools/drift_probe.py > $O/drift.jsonl 2> $O/drift.err; tail -3 $O/drift.err
cat $O/drift.jsonl | cut -c1-400
