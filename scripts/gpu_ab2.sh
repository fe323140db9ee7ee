mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/$1_ab_base.log 2>&1
for lib in "${@:2}"; do
  n=$(basename $lib .so)
  NI_LIB=$lib timeout 400 python bench.py --no-cpu-baseline > gpurun_out/$1_ab_$n.log 2>&1
  NI_LIB=$lib timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$1_ab_${n}_C3.log 2>&1
done
