for v in base nostore noepi nomma; do
  if [ $v = base ]; then L=""; else L="BITSERIAL_LIB=build/$v/libbitserial.so"; fi
  env $L timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w5_$v.json 2>&1
done
echo done
