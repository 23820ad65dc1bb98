BITSERIAL_LIB=build/libbitserial_prof.so python tools/prof_probe.py 2 5 9 12 > gpurun_out/r02f_prof.txt 2>&1
echo done
