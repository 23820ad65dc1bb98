timeout 600 python -m pytest tests/test_parity_gpu.py -v -x --timeout 60 -k "three_call_conv_tc_weight_slots" > gpurun_out/r02m_pytest.log 2>&1; tail -40 gpurun_out/r02m_pytest.log | grep -v "^$" | tail -25
python tools/small_probe.py > gpurun_out/r02m_small_probe.json 2>&1
echo done
