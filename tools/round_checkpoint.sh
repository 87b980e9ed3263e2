#!/bin/bash
# One GPU checkpoint of the round's evidence (run on the gpurun box from the repo root):
# full -m gpu suite, bench line, native host-overhead probe, ncu of the headline kernel
# and the bench launch list, single-wave kernel times.  Outputs under gpurun_out/ck_<tag>/.
TAG=${1:-r02}
O=gpurun_out/ck_$TAG
mkdir -p $O
# (compute-sanitizer runs were dropped: the GPU pool closed compute-sanitizer late in round 2; the
# committed sanitizer logs under profiles/sanitizer/ are from the earlier checkpoints)
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 --timeout 900 > $O/pytest.log 2>&1; echo "pytest_rc=$?" >> $O/pytest.log
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench_rc=$?"
g++ -O2 -I include -I /usr/local/cuda/include tools/host_overhead_c.cpp -L paper_2311_03543_b200 -lcompar \
    -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2311_03543_b200 -o /tmp/host_overhead_c && \
    { /tmp/host_overhead_c virtual; /tmp/host_overhead_c gpu; } > $O/host_overhead.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_2sm_wide -c 1 -o $O/tc_bf16_2sm_w_32768 \
    python tools/prof_run.py tc_bf16_2sm_w 32768 32768 32768 1 > $O/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-targets --no-yardstick > $O/launches_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sw_ncu.csv python tools/single_wave_ncu.py run > /dev/null 2>&1
python tools/single_wave_ncu.py parse $O/sw_ncu.csv $O/sw_ncu.json > $O/sw_ncu.txt 2>&1
echo checkpoint_done
