# digit formation in the packers with a pairwise PRMT compress (window pack was ALU-bound): parity, step, pack rates
o=gpurun_out/r02zo
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -x > ${o}_pytest_gpu.log 2>&1; tail -1 ${o}_pytest_gpu.log
python bench.py --no-e2e --no-cpu > ${o}_bench_b.json 2> ${o}_bench.err
python bench.py --no-e2e --no-cpu --workload gemm --size 8192 --steps 5 > ${o}_bench_gemm8192.json 2>> ${o}_bench.err
python bench.py --no-e2e --no-cpu --workload resnet1 --steps 50 > ${o}_bench_resnet1.json 2>> ${o}_bench.err
timeout 300 python tools/winpack_probe.py > ${o}_winpack_layers.json 2>> ${o}_bench.err
python - <<'P'
import json
for f in ('bench_b', 'bench_gemm8192', 'bench_resnet1'):
    d = json.loads(open(f'gpurun_out/r02zo_{f}.json').read().strip().splitlines()[-1])
    print(f, round(d['ms_per_step'], 4), d['parity']['result'], d.get('breakdown'))
P
tail -c 1500 ${o}_winpack_layers.json
