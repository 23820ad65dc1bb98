timeout 300 python tools/tcw_mode_check.py > gpurun_out/w8_mode.log 2>&1; cat gpurun_out/w8_mode.log | tail -3
timeout 600 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -k "pack or weights" > gpurun_out/w8_pytest_pack.log 2>&1; tail -2 gpurun_out/w8_pytest_pack.log
timeout 300 python tools/tcw_probe.py --layers --reps 10 > gpurun_out/w8_probe.json 2>&1
echo done
