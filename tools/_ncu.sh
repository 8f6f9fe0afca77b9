# scratch: ncu full capture (source-correlated) of the hot kernels at F = 2^20
O=gpurun_out/${TAG:-ncu}; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_expand_tc|k_materialize_bs}" -s ${SKIP:-4} -c ${COUNT:-2} \
  -o $O/prof python bench.py --F 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
echo ncu_rc=$? >> $O/ncu.log; tail -3 $O/ncu.log; ls -la $O
