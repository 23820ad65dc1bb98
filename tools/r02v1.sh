set -o pipefail
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -rs > gpurun_out/r02v1_pytest_gpu.log 2>&1; tail -4 gpurun_out/r02v1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v1_smoke.log 2>&1; tail -2 gpurun_out/r02v1_smoke.log
python bench.py > gpurun_out/r02v1_bench.json 2> gpurun_out/r02v1_bench.err; tail -c 300 gpurun_out/r02v1_bench.json
python bench.py --impl reference > gpurun_out/r02v1_bench_reference.json 2> gpurun_out/r02v1_bench_reference.err
for w in conv1 resnet1 gemv; do python bench.py --workload $w > gpurun_out/r02v1_bench_$w.json 2> gpurun_out/r02v1_bench_$w.err; done
python bench.py --workload gemm --size 8192 --no-e2e > gpurun_out/r02v1_bench_gemm8192.json 2> gpurun_out/r02v1_bench_gemm.err
echo done
