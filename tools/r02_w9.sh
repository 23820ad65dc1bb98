BITSERIAL_LIB=build/prof/libbitserial.so timeout 120 python tools/tcw_one.py --layers 2 --iters 1 > gpurun_out/w9_prof_l2.log 2>&1
BITSERIAL_LIB=build/prof/libbitserial.so timeout 120 python tools/tcw_one.py --layers 12 --iters 1 > gpurun_out/w9_prof_l12.log 2>&1
BITSERIAL_LIB=build/mmaonly/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w9_mmaonly.json 2>&1
echo done
