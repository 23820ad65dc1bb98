./tools/mma_swz_bench > gpurun_out/w10_mma_swz.jsonl 2>&1
timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w10_base.json 2>&1
BITSERIAL_LIB=build/mmaonly/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w10_mmaonly.json 2>&1
echo done
