# first GPU run of the window path: parity subset (stop at first failure), then timing probe
timeout 600 python -m pytest tests/test_parity_tcw_gpu.py -x -q --timeout 300 -k "pack or weights" > gpurun_out/w1_pytest_pack.log 2>&1; tail -3 gpurun_out/w1_pytest_pack.log
timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -k "not pack and not weights" --maxfail 5 > gpurun_out/w1_pytest_conv.log 2>&1; tail -3 gpurun_out/w1_pytest_conv.log
timeout 300 python tools/tcw_probe.py --layers > gpurun_out/w1_probe.json 2> gpurun_out/w1_probe.err; tail -3 gpurun_out/w1_probe.err
echo done
