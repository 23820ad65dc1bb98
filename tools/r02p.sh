timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -rs --timeout 120 -k "small or multicast" > gpurun_out/r02p_pytest.log 2>&1; tail -4 gpurun_out/r02p_pytest.log
python tools/small_probe.py > gpurun_out/r02p_small_probe.json 2>&1
python tools/layer_sweep.py --tc --raw > gpurun_out/r02p_sweep_raw.json 2>&1
python tools/layer_sweep.py --tc > gpurun_out/r02p_sweep_prep.json 2>&1
echo done
