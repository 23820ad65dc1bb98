timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "tc" > gpurun_out/r02c_pytest.log 2>&1; tail -3 gpurun_out/r02c_pytest.log
python tools/layer_sweep.py --tc --group > gpurun_out/r02c_sweep.json 2>&1
for d in 1 48 176; do
 BITSERIAL_LIB=build/libbitserial_knobs.so BS_TC_DEBUG=$d python tools/layer_sweep.py --tc --layers 2,5,6,9,12 > gpurun_out/r02c_knob$d.json 2>&1
done
python bench.py --no-e2e > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
echo done
