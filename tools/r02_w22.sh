BITSERIAL_LIB=build/sw128/libbitserial.so timeout 600 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 -x -k "conv_tcw_parity and 2-1 or sentinel or group" > gpurun_out/w22_pytest.log 2>&1; tail -3 gpurun_out/w22_pytest.log
BITSERIAL_LIB=build/sw128/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w22_sw128.json 2>&1
echo done
