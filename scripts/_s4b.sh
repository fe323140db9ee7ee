mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s4b_build.log 2>&1
timeout 200 python scripts/copy_probe.py > gpurun_out/s4b_copy.log 2>&1
timeout 400 python scripts/gaps.py 64 > gpurun_out/s4b_gaps.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coefficients -s 1 -c 1 \
  -o gpurun_out/s4b_coef_full -f python scripts/profile_mg.py 16 > gpurun_out/s4b_ncu_coef.log 2>&1
