mkdir -p gpurun_out
timeout 900 python scripts/e2e_ab.py 2:-1:0 2:-1:2 2:-1:4 2:-1:8 2:-1:16 > gpurun_out/s5o_ab.log 2>&1
timeout 300 python -m pytest tests/test_gpu_edge_cases.py -x -q --timeout 300 > gpurun_out/s5o_pytest.log 2>&1
