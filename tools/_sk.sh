timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "simt or tma" > gpurun_out/ffma2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ffma2_parity.log
P="simt_f32:4096:4096:4096,tma_f32:4096:4096:4096,simt_f32:8192:8192:8192,tma_f32:8192:8192:8192,simt_f32:1024:1024:1024,tma_f32:1024:1024:1024,simt_f32:4096:4096:4096:1,tma_f32:4096:4096:4096:1"
timeout 300 python tools/probe.py $P > gpurun_out/ffma2_probe.log 2>&1
tail -3 gpurun_out/ffma2_parity.log; cat gpurun_out/ffma2_probe.log
