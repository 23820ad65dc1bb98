timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 -x -k "group or resnet or sentinel or 2-1" > gpurun_out/w43_pytest.log 2>&1; tail -1 gpurun_out/w43_pytest.log
timeout 300 python tools/tcw_probe.py --layers --reps 10 --groups all > gpurun_out/w43_base.json 2>&1
timeout 600 python tools/hybrid_probe.py --spec "tcw=2,5,6,8;tc=4,7,9,10,11,12" --spec "tcw=2,5,8;tc=4,6,7,9,10,11,12" > gpurun_out/w43_hybrid.jsonl 2>&1
echo done
