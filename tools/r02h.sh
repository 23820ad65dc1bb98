python tools/layer_sweep.py --tc --group > gpurun_out/r02h_sweep.json 2>&1
BITSERIAL_LIB=build/libbitserial_w256.so python tools/layer_sweep.py --tc --group > gpurun_out/r02h_sweep256.json 2>&1
echo done
