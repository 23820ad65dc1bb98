# --path popc forced onto the integer-pipe kernel (BS_ALGO_POPC; AUTO now reaches the tensor cores);
# limit study (f1) refreshed on the round-2 tree
o=gpurun_out/r02zi
: > ${o}_bench_popc.jsonl
run() { timeout 300 python bench.py --no-cpu --no-e2e "$@" >> ${o}_bench_popc.jsonl 2>> ${o}.err || echo "{\"failed\": \"$*\"}" >> ${o}_bench_popc.jsonl; }
run --workload resnet256 --path popc
run --workload conv1 --steps 50 --path popc
run --workload resnet1 --steps 50 --path popc
run --workload gemm --size 4096 --steps 5 --path popc
run --workload gemm --size 8192 --steps 5 --a-bits 4 --w-bits 2 --path popc
timeout 900 python tools/limit_study.py --path tc > ${o}_limit_study_tc.json 2>> ${o}.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_popc_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --path popc > ${o}_ncu_launch.log 2>&1
python tools/ncu_summary.py launch ${o}_popc_launches.csv ${o}_popc_launches.json
echo done
