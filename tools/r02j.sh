timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "small or conv_parity or config1 or config2 or config3 or dense or gemv" > gpurun_out/r02j_pytest.log 2>&1; tail -3 gpurun_out/r02j_pytest.log
for w in conv1 resnet1 gemv; do python bench.py --workload $w --no-e2e > gpurun_out/r02j_bench_$w.json 2> gpurun_out/r02j_bench_$w.err; done
echo done
