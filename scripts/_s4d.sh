mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4d_build.log 2>&1
timeout 400 python scripts/gaps.py 64 stream > gpurun_out/s4d_gaps_stream.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4d_bench.log 2>&1
