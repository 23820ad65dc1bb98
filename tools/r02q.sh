timeout 900 python -m pytest tests/test_parity_gpu.py -x -q --timeout 120 -k "tc or three_call or fp4" > gpurun_out/r02q_pytest.log 2>&1; tail -2 gpurun_out/r02q_pytest.log
python tools/layer_sweep.py --tc --raw > gpurun_out/r02q_sweep_raw.json 2>&1
python tools/layer_sweep.py --tc --group > gpurun_out/r02q_sweep_prep.json 2>&1
timeout 300 python -m pytest tests/test_parity_gpu.py -q -s --timeout 200 -k "three_call_headline" > gpurun_out/r02q_headline.log 2>&1; grep "three-call" gpurun_out/r02q_headline.log
python bench.py --no-e2e > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
echo done
