timeout 900 python -m pytest tests/test_parity_gpu.py -x -q --timeout 120 -k "tc or three_call or fp4" > gpurun_out/r02w_pytest.log 2>&1; tail -2 gpurun_out/r02w_pytest.log
python tools/layer_sweep.py --tc --group > gpurun_out/r02w_sweep_prep.json 2>&1
python bench.py --no-e2e --no-cpu > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
echo done
