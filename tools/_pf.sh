timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "2sm" > gpurun_out/pf_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pf_parity.log
P="tc_bf16_2sm_w:8192:8192:8192,tc_bf16_2sm:8192:8192:8192,tc_bf16_2sm:65536:256:4096,tc_tf32_2sm_w:8192:8192:8192,tc_tf32_2sm:256:256:256,tc_bf16_2sm_w:32768:32768:32768"
for PF in 0 1 0 1; do echo "PREFETCH=$PF"; COMPAR_CIN_PREFETCH=$PF timeout 300 python tools/probe.py $P; done > gpurun_out/pf_probe.log 2>&1
tail -2 gpurun_out/pf_parity.log; cat gpurun_out/pf_probe.log
