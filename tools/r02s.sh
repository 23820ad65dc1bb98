python tools/layer_sweep.py --tc --group > gpurun_out/r02s_sweep_prep.json 2>&1
BITSERIAL_LIB=build/libbitserial_nomc.so python tools/layer_sweep.py --tc --group > gpurun_out/r02s_sweep_nomc.json 2>&1
python tools/layer_sweep.py --tc --group > gpurun_out/r02s_sweep_prep2.json 2>&1
echo done
