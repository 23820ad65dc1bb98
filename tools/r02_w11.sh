for v in prof mmaprof; do for L in 2 5; do
BITSERIAL_LIB=build/$v/libbitserial.so timeout 120 python tools/tcw_one.py --layers $L --iters 1 > gpurun_out/w11_${v}_l$L.log 2>&1
done; done
echo done
