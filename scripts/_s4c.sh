mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4c_build.log 2>&1
timeout 200 python scripts/copy_probe.py > gpurun_out/s4c_copy.log 2>&1
timeout 600 python -m pytest tests/test_gpu_edge_cases.py tests/test_gpu_fullsize.py -x -q --timeout 300 > gpurun_out/s4c_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/s4c_bench.log 2>&1
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4c_cfg_C1.log 2>&1
