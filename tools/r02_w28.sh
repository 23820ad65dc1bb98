python bench.py --path hybrid > gpurun_out/w28_bench_hybrid.json 2> gpurun_out/w28_bench_hybrid.err
echo done
