timeout 900 python -m pytest tests/test_parity_gpu.py -x -q --timeout 120 -k "gemv or dense or config2" > gpurun_out/r02y_pytest.log 2>&1; tail -2 gpurun_out/r02y_pytest.log
python bench.py --workload gemv > gpurun_out/r02y_bench_gemv.json 2> gpurun_out/r02y_bench_gemv.err
python bench.py --workload conv1 > gpurun_out/r02y_bench_conv1.json 2> gpurun_out/r02y_bench_conv1.err
echo done
