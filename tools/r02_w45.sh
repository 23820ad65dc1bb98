timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -k "fp4_bound" -rs > gpurun_out/w45_pytest.log 2>&1; tail -3 gpurun_out/w45_pytest.log
echo done
