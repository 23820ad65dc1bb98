for L in 2 5; do
BITSERIAL_LIB=build/prof/libbitserial.so timeout 120 python tools/tcw_one.py --layers $L --iters 1 > gpurun_out/w34_prof_l$L.log 2>&1
done
echo done
