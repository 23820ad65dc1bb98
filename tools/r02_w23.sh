timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 120 > gpurun_out/w23_pytest.log 2>&1; tail -2 gpurun_out/w23_pytest.log
timeout 300 python tools/tcw_probe.py --layers --reps 10 > gpurun_out/w23_base.json 2>&1
echo done
