#!/bin/bash
# Raster / K-order experiments at 32768^3: DRAM bytes (ncu) and sustained TFLOP/s.
M="--metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm -s 2 -c 1"
for cfg in "tc_bf16 16 0" "tc_bf16 16 1" "tc_bf16 8 0" "tc_bf16 32 0" "tc_bf16 8 1" "tc_bf16_2sm 8 0" "tc_bf16_2sm 4 0" "tc_bf16_2sm 16 0"; do
  set -- $cfg
  echo "== $cfg"
  COMPAR_TC1_GROUP=$2 COMPAR_TC_GROUP=$2 COMPAR_TC_SERP=$3 timeout 200 ncu $M python tools/prof_run.py $1 32768 32768 32768 3 2>&1 | grep -E "dram__|gpu__time"
  COMPAR_TC1_GROUP=$2 COMPAR_TC_GROUP=$2 COMPAR_TC_SERP=$3 timeout 200 python tools/prof_run.py $1 32768 32768 32768 40 2>&1 | tail -3
done
