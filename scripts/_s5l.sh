mkdir -p gpurun_out
rm -f gpurun_out/s5l_check.log
for v in 1.95 2.0 2.05; do
  NI_LIB=exp/libni_oc$v.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5l_bench_oc$v.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5l_bench_oc1.9.log 2>&1
for c in C4 C3 C1; do
  NI_LIB=exp/libni_oc2.0.so timeout 300 python scripts/fill_vs_golden.py $c >> gpurun_out/s5l_check.log 2>&1
done
for c in C1 C3 C4; do
  NI_LIB=exp/libni_oc2.0.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5l_cfg_${c}_oc2.0.log 2>&1
done
NI_LIB=exp/libni_oc2.0.so timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5l_pytest_oc2.0.log 2>&1
