mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scale_fused -c 1 -o gpurun_out/r02u_fused_full -f python scripts/stage_times.py C1 1 > gpurun_out/r02u_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02u_pytest.log 2>&1
for c in C1 C5; do timeout 300 python scripts/stage_times.py $c 3 > gpurun_out/r02u_stages_$c.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r02u_bench.log 2>&1
