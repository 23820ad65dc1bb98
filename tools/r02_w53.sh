timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -rs > gpurun_out/w53_pytest.log 2>&1; tail -4 gpurun_out/w53_pytest.log
echo done
