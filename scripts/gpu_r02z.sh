mkdir -p gpurun_out
tag=${1:-r02z}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
if ! timeout 120 python scripts/stage_times.py C1 2 > gpurun_out/${tag}_stages_C1.log 2>&1; then
  echo "C1 probe failed or hung" >> gpurun_out/${tag}_stages_C1.log; exit 3
fi
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${tag}_pytest.log 2>&1
timeout 400 python bench.py > gpurun_out/${tag}_bench.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg_$c.log 2>&1
done
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg_maps8.log 2>&1
