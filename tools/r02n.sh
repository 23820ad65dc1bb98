timeout 900 python -m pytest tests/test_parity_gpu.py -v -x --timeout 120 -k "three_call or multicast" > gpurun_out/r02n_pytest.log 2>&1; grep -E "passed|failed|PASSED.*multicast|SKIPPED|three-call step|Error" gpurun_out/r02n_pytest.log | tail -8
python tools/small_one.py 6 > gpurun_out/r02n_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:small_conv -s 2 -c 1 -o /tmp/r02n_s6 python tools/small_one.py 6 > gpurun_out/r02n_ncu.log 2>&1
ncu -i /tmp/r02n_s6.ncu-rep --page details --csv > gpurun_out/r02n_s6_details.csv 2>&1
ncu -i /tmp/r02n_s6.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02n_s6_src.csv 2>&1
echo done
