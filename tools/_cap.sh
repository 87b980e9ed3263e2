for R in 32768 16384 8192 4096; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_2sm_mc -s 1 -c 1 -o gpurun_out/r01_tc_bf16_2sm_$R python tools/prof_run.py tc_bf16_2sm $R 32768 32768 2 > gpurun_out/cap_$R.log 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_2sm_mc -s 1 -c 1 -o gpurun_out/r01_tc_bf16_2sm_8192cube python tools/prof_run.py tc_bf16_2sm 8192 8192 8192 2 > gpurun_out/cap_8192c.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wide -s 1 -c 1 -o gpurun_out/r01_tc_bf16_2sm_w_8192cube python tools/prof_run.py tc_bf16_2sm_w 8192 8192 8192 2 > gpurun_out/cap_8192w.log 2>&1
ls -la gpurun_out/*.ncu-rep
