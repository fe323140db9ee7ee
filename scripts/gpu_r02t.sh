mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_seams.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/r02t_pytest.log 2>&1
for c in C1 C2; do timeout 300 python scripts/stage_times.py $c 4 > gpurun_out/r02t_stages_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02t_launches_c1.csv python scripts/stage_times.py C1 1 > gpurun_out/r02t_ncu_c1.log 2>&1
