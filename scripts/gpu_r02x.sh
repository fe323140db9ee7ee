mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02x_build.log 2>&1
if ! timeout 120 python scripts/stage_times.py C1 2 > gpurun_out/r02x_stages_C1.log 2>&1; then
  echo "C1 probe failed or hung" >> gpurun_out/r02x_stages_C1.log; exit 3
fi
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/r02x_pytest.log 2>&1
for c in C2 C3; do timeout 120 python scripts/stage_times.py $c 3 > gpurun_out/r02x_stages_$c.log 2>&1; done
timeout 400 python bench.py > gpurun_out/r02x_bench.log 2>&1
NI_LIB=exp/lib_a3.so timeout 400 python bench.py --no-cpu-baseline > gpurun_out/r02x_ab_a3.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02x_cfg_$c.log 2>&1
done
