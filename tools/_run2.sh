timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
COMPAR_TC2_PAIRS=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "2sm and not 2sm_w" > gpurun_out/mc2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/mc2_parity.log
timeout 600 python tools/config3.py gpurun_out/config3.json 2.0 > gpurun_out/config3.log 2>&1
timeout 900 python tools/selector_sweep.py gpurun_out/selector.json > gpurun_out/selector.log 2>&1; echo "rc=$?" >> gpurun_out/selector.log
tail -3 gpurun_out/pytest_gpu.log gpurun_out/mc2_parity.log; cat gpurun_out/config3.log | grep -v "^ "; tail -5 gpurun_out/selector.log
