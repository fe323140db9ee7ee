mkdir -p gpurun_out
for c in C4 C3 C5_00; do
  NI_MG_W_HI=1 timeout 300 python scripts/fill_vs_golden.py $c >> gpurun_out/s5g_check.log 2>&1
  timeout 300 python scripts/fill_vs_golden.py $c >> gpurun_out/s5g_check.log 2>&1
  NI_MG_W_HI=2 timeout 300 python scripts/fill_vs_golden.py $c >> gpurun_out/s5g_check.log 2>&1
done
