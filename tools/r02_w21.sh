python bench.py > gpurun_out/w21_bench.json 2> gpurun_out/w21_bench.err
python bench.py --path tcw > gpurun_out/w21_bench_tcw.json 2> gpurun_out/w21_bench_tcw.err
python bench.py --workload resnet1 --path tcw > gpurun_out/w21_bench_resnet1_tcw.json 2> gpurun_out/w21_bench_resnet1_tcw.err
python bench.py --workload resnet1 > gpurun_out/w21_bench_resnet1.json 2> gpurun_out/w21_bench_resnet1.err
python bench.py --workload conv1 --path tcw > gpurun_out/w21_bench_conv1_tcw.json 2> gpurun_out/w21_bench_conv1_tcw.err
python bench.py --workload conv1 > gpurun_out/w21_bench_conv1.json 2> gpurun_out/w21_bench_conv1.err
python bench.py --workload gemv > gpurun_out/w21_bench_gemv.json 2> gpurun_out/w21_bench_gemv.err
echo done
