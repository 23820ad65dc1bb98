timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "small or conv_parity or config1 or config3 or dense_i8 or gemv" > gpurun_out/r02i_pytest.log 2>&1; tail -3 gpurun_out/r02i_pytest.log
for w in conv1 resnet1 gemv; do python bench.py --workload $w --no-e2e > gpurun_out/r02i_bench_$w.json 2> gpurun_out/r02i_bench_$w.err; done
python bench.py --workload resnet1 --path tc --no-e2e > gpurun_out/r02i_bench_resnet1_tc.json 2>&1
python bench.py --no-e2e --group-layers "2|4,5,6,7,8,9,10,11,12" > gpurun_out/r02i_bench_g2.json 2>&1
echo done
