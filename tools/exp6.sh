M="--metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_gemm -s 1 -c 1"
for cfg in "16384 16384 16384" ; do
 for G in 4 8 16 32; do echo "== group $G $cfg"; COMPAR_TC_GROUP=$G timeout 120 ncu $M python tools/prof_run.py tc_bf16_2sm $cfg 2 2>&1 | grep -E "dram__|gpu__time|hit_rate|per_second|TFLOP"; done
 echo "== pad 64"; timeout 120 ncu $M python tools/prof_run.py tc_bf16_2sm $cfg 2 --pad 64 2>&1 | grep -E "dram__|gpu__time|hit_rate|per_second|TFLOP"
 echo "== beta 0"; timeout 120 ncu $M python tools/prof_run.py tc_bf16_2sm $cfg 2 --beta 0 2>&1 | grep -E "dram__|gpu__time|hit_rate|per_second|TFLOP"
done
for G in 4 8 16; do echo "== 32768 group $G"; COMPAR_TC_GROUP=$G timeout 120 python tools/prof_run.py tc_bf16_2sm 32768 32768 32768 4 2>&1 | tail -2; done
echo "== 32768 1sm"; timeout 120 python tools/prof_run.py tc_bf16 32768 32768 32768 4 2>&1 | tail -2
