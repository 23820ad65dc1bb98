timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "three_call or small or tc_b_modes" -s > gpurun_out/r02l_pytest.log 2>&1; tail -3 gpurun_out/r02l_pytest.log; grep "three-call step" gpurun_out/r02l_pytest.log
for w in conv1 resnet1; do python bench.py --workload $w --no-e2e > gpurun_out/r02l_bench_$w.json 2> gpurun_out/r02l_bench_$w.err; done
echo done
