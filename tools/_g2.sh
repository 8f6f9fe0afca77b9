# scratch GPU session: parity tests + default / no_tc bench A/B
O=gpurun_out/${TAG:-tc2}; mkdir -p $O
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -4 $O/pytest.log
fi
for K in ${VARIANTS:-"" no_tc}; do
SNP_KERNELS=$K timeout 600 python bench.py --steps ${STEPS:-6} --warmup 3 --no-e2e --no-cpu $BARGS > $O/bench_$K.log 2>&1
python -c "
import json;l=[x for x in open('$O/bench_$K.log') if x.startswith('{')];d=json.loads(l[-1]);print('$K',round(d['value']/1e6,2),'Mt/s',round(d['ms_per_step'],2),'ms',{k:round(v,2) for k,v in d['phase_ms_per_step'].items()},d['digest'])" || tail -20 $O/bench_$K.log
done
