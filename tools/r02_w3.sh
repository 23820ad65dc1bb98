timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q --timeout 300 -k "not pack and not weights" --maxfail 8 > gpurun_out/w3_pytest_conv.log 2>&1; tail -3 gpurun_out/w3_pytest_conv.log
for b in 16 256; do timeout 300 python tools/tcw_probe.py --layers --batch $b --reps 10 > gpurun_out/w3_probe_b$b.json 2>&1; done
echo done
