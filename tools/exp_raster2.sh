#!/bin/bash
M="--metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm -s 2 -c 1"
for G in 2 3 4 6 -2 -4 -8; do
  echo "== tc_bf16_2sm group $G"
  COMPAR_TC_GROUP=$G timeout 200 ncu $M python tools/prof_run.py tc_bf16_2sm 32768 32768 32768 3 2>&1 | grep -E "dram__|gpu__time"
  COMPAR_TC_GROUP=$G timeout 200 python tools/prof_run.py tc_bf16_2sm 32768 32768 32768 40 2>&1 | tail -2
done
for G in 4 2; do
  echo "== tc_bf16_2sm 8192 group $G"
  COMPAR_TC_GROUP=$G timeout 200 python tools/prof_run.py tc_bf16_2sm 8192 8192 8192 400 2>&1 | tail -2
  echo "== tc_bf16_2sm 16384 group $G"
  COMPAR_TC_GROUP=$G timeout 200 python tools/prof_run.py tc_bf16_2sm 16384 16384 16384 200 2>&1 | tail -2
done
