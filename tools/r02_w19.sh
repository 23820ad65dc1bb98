timeout 1200 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -rs > gpurun_out/w19_pytest.log 2>&1; tail -3 gpurun_out/w19_pytest.log
echo done
