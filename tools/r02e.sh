timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "tc or fp4" > gpurun_out/r02e_pytest.log 2>&1; tail -3 gpurun_out/r02e_pytest.log
python tools/layer_sweep.py --tc --group > gpurun_out/r02e_sweep.json 2>&1
python bench.py --no-e2e > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
echo done
