for v in mmaonly loadonly; do
  BITSERIAL_LIB=build/$v/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w6_$v.json 2>&1
done
echo done
