for L in 2 5 12; do
BITSERIAL_LIB=build/prof/libbitserial.so timeout 120 python tools/tcw_one.py --layers $L --iters 1 > gpurun_out/w13_prof_l$L.log 2>&1
done
timeout 300 python tools/tcw_probe.py --layers --reps 10 > gpurun_out/w13_base.json 2>&1
timeout 300 python tools/tcw_mode_check.py > gpurun_out/w13_mode.log 2>&1
echo done
