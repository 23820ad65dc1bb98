# bench lines with the algorithmic-bytes roofline for the window-path layers (bit-packed input, not the layout)
python bench.py > gpurun_out/r02v6_bench.json 2> gpurun_out/r02v6_bench.err
python bench.py --workload resnet1 > gpurun_out/r02v6_bench_resnet1.json 2> gpurun_out/r02v6_bench_resnet1.err
echo done
