mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02w_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02w_pytest.log 2>&1
for c in C1 C2 C3; do timeout 300 python scripts/stage_times.py $c 3 > gpurun_out/r02w_stages_$c.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r02w_bench.log 2>&1
bash scripts/gpu_configs.sh r02w
