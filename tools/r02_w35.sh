timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 -x > gpurun_out/w35_pytest.log 2>&1; tail -2 gpurun_out/w35_pytest.log
timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w35_base.json 2>&1
for L in 2; do
BITSERIAL_LIB=build/prof/libbitserial.so timeout 120 python tools/tcw_one.py --layers $L --iters 1 > gpurun_out/w35_prof_l$L.log 2>&1
done
timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,8;tc=4,6,7,9,10,11,12" --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" --spec "tcw=2,4,5,6,8;tc=7,9,10,11,12" > gpurun_out/w35_hybrid.jsonl 2>&1
echo done
