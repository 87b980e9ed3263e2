#!/bin/bash
# Wide pair kernel at 32768^3 BF16: raster band (pair rows) vs DRAM bytes and sustained rate.
# usage (GPU box): bash tools/raster_sweep.sh OUTDIR
OUT=${1:-gpurun_out}
for G in 4 8 12 16; do
  echo "== G=$G"
  COMPAR_TCW_GROUP=$G ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm_2sm_wide -c 1 python tools/prof_run.py tc_bf16_2sm_w 32768 32768 32768 1 2>&1 | grep -E "dram__|gpu__time|per_second|hit_rate"
  COMPAR_TCW_GROUP=$G python tools/prof_run.py tc_bf16_2sm_w 32768 32768 32768 12 2>&1 | tail -4
done > $OUT/raster_sweep.log 2>&1
