timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w4_probe.json 2>&1
BITSERIAL_LIB=build/nostore/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w4_probe_nostore.json 2>&1
echo done
