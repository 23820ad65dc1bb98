timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 > gpurun_out/w44_pytest.log 2>&1; tail -1 gpurun_out/w44_pytest.log
timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups "all;2,5,6,8|9,10,12" > gpurun_out/w44_base.json 2>&1
BITSERIAL_LIB=build/nopair/libbitserial.so timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w44_nopair.json 2>&1
timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" --spec "tcw=2,5,6,8,12;tc=4,7,9,10,11" --spec "tcw=2,5,6,8,9,12;tc=4,7,10,11" --spec "tcw=2,5,6,8,9,10,12;tc=4,7,11" > gpurun_out/w44_hybrid.jsonl 2>&1
echo done
