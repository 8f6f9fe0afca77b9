#!/bin/bash
# A/B kernel variants on the bench workload:
#   tools/gpu_ab.sh TAG "ENV=.. ENV2=..|DEF1 DEF2" ...
# each argument: environment assignments, then optionally "|" and -D defines
# for a variant libsnp build (paper_1104_1824_b200/libsnp_v<i>.so).
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
i=0
for arg in "$@"; do
  envs=${arg%%|*}; defs=""
  [[ "$arg" == *"|"* ]] && defs=${arg#*|}
  lib=""
  if [ -n "$defs" ]; then
    lib=$PWD/paper_1104_1824_b200/libsnp_v$i.so
    python -c "from paper_1104_1824_b200 import build as b; b.build_variant('$lib', '$defs'.split())" >> $O/build.log 2>&1
  fi
  env $envs ${lib:+SNP_LIB=$lib} timeout 600 python bench.py --steps ${AB_STEPS:-8} --warmup 3 --no-e2e --no-cpu $AB_ARGS > $O/ab$i.log 2>&1
  python - $O/ab$i.log "$arg" <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[2], 'FAILED'); sys.exit()
d = json.loads(l[-1]); ph = d['phase_ms_per_step']
print(f"{sys.argv[2]:44s} {d['value']:.4g} t/s  {d['ms_per_step']:.1f} ms  expand {ph['expand']:.1f} mat {ph['materialize']:.1f} digest {d['digest']}")
PY
  i=$((i+1))
done
