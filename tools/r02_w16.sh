timeout 600 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -k "conv_tcw_parity and (2-1 or 2-2) or group or sentinel" > gpurun_out/w16_pytest.log 2>&1; tail -2 gpurun_out/w16_pytest.log
for L in 2 5; do
BITSERIAL_LIB=build/prof/libbitserial.so timeout 120 python tools/tcw_one.py --layers $L --iters 1 > gpurun_out/w16_prof_l$L.log 2>&1
done
timeout 300 python tools/tcw_probe.py --layers --reps 10 > gpurun_out/w16_base.json 2>&1
BITSERIAL_LIB=build/nostore/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w16_nostore.json 2>&1
echo done
