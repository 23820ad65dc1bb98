# baseline re-check of the restored HEAD: default bench + tcd parity subset
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02z_smi.txt 2>&1
python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
python bench.py --workload resnet1 > gpurun_out/r02z_bench_resnet1.json 2> gpurun_out/r02z_bench_resnet1.err
echo done
