# round-2 final tree: full GPU parity, smoke, both bench arms, batch-1 and GEMM lines, shards, ncu launch list
o=gpurun_out/r02zq
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -rs > ${o}_pytest_gpu.log 2>&1; tail -1 ${o}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; tail -1 ${o}_smoke.log
python bench.py > ${o}_bench.json 2> ${o}_bench.err
python bench.py --impl reference > ${o}_bench_reference.json 2> ${o}_bench_reference.err
bash tools/bench_all.sh r02zq
timeout 600 python tools/shard_check.py > ${o}_shard_parity.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > ${o}_plain2.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > ${o}_ncu_launch.log 2>&1
python tools/ncu_summary.py launch ${o}_launches.csv ${o}_launches.json
echo done
