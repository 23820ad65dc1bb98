timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -rs --timeout 120 -k "small or conv_parity or config1 or config3 or dense_i8 or multicast" > gpurun_out/r02o_pytest.log 2>&1; tail -4 gpurun_out/r02o_pytest.log
python tools/small_probe.py > gpurun_out/r02o_small_probe.json 2>&1
timeout 300 python -m pytest tests/test_parity_gpu.py -q -s --timeout 200 -k "three_call_headline" > gpurun_out/r02o_headline.log 2>&1; grep "three-call" gpurun_out/r02o_headline.log
echo done
