BITSERIAL_LIB=build/e16/libbitserial.so timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 -x -k "group or resnet or sentinel or 2-1" > gpurun_out/w50_pytest.log 2>&1; tail -1 gpurun_out/w50_pytest.log
BITSERIAL_LIB=build/e16/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups "all;2,5,6,8" > gpurun_out/w50_e16.json 2>&1
timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups "all;2,5,6,8" > gpurun_out/w50_base.json 2>&1
BITSERIAL_LIB=build/e16/libbitserial.so timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" > gpurun_out/w50_hybrid_e16.jsonl 2>&1
timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" > gpurun_out/w50_hybrid_base.jsonl 2>&1
echo done
