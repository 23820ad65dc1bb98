timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 -x -k "pack or group or resnet" > gpurun_out/w52_pytest.log 2>&1; tail -1 gpurun_out/w52_pytest.log
timeout 300 python tools/winpack_probe.py > gpurun_out/w52_winpack.json 2>&1
timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" --spec "tcw=2,5,8;tc=4,6,7,9,10,11,12" > gpurun_out/w52_hybrid.jsonl 2>&1
echo done
