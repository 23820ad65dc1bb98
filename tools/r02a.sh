set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/store_bench > gpurun_out/r02a_store.jsonl 2>&1
python tools/layer_sweep.py --tc > gpurun_out/r02a_sweep.json 2>&1
for d in 0 1 48 176 128; do
 BITSERIAL_LIB=build/libbitserial_knobs.so BS_TC_DEBUG=$d python tools/layer_sweep.py --tc --layers 2,5,6,9,12 > gpurun_out/r02a_knob$d.json 2>&1
done
python tools/layer_sweep.py --tc --group > gpurun_out/r02a_group.json 2>&1
echo done
