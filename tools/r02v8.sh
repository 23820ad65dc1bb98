# final headline lines of the final tree (default hybrid step, unified e2e pipeline)
python bench.py > gpurun_out/r02v8_bench.json 2> gpurun_out/r02v8_bench.err
python bench.py --impl reference > gpurun_out/r02v8_bench_reference.json 2> gpurun_out/r02v8_bench_reference.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v8_smoke.log 2>&1
echo done
