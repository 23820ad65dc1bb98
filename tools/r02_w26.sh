python bench.py --path hybrid > gpurun_out/w26_bench_hybrid.json 2> gpurun_out/w26_bench_hybrid.err
python bench.py > gpurun_out/w26_bench_tc.json 2> gpurun_out/w26_bench_tc.err
python bench.py --path hybrid --tcw-layers 2,5,6,8 --no-e2e --no-cpu > gpurun_out/w26_bench_hybrid2568.json 2> gpurun_out/w26_bench_hybrid2568.err
echo done
