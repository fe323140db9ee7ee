mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5m_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5m_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5m_bench.log 2>&1
for c in C1 C3; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5m_cfg_$c.log 2>&1
done
timeout 300 python scripts/gaps.py 64 > gpurun_out/s5m_gaps.log 2>&1
