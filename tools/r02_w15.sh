for L in 2 5; do
BITSERIAL_LIB=build/profstg/libbitserial.so timeout 120 python tools/tcw_one.py --layers $L --iters 1 > gpurun_out/w15_profstg_l$L.log 2>&1
done
for v in stg nostore; do
BITSERIAL_LIB=build/$v/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 > gpurun_out/w15_$v.json 2>&1
done
echo done
