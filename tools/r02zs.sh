# window pack: two tasks per iteration (both loads in flight), 6 resident CTAs per SM
o=gpurun_out/r02zs
timeout 900 python -m pytest tests/test_parity_tcw_gpu.py -q -m gpu --timeout 300 -x > ${o}_pytest_tcw.log 2>&1; tail -1 ${o}_pytest_tcw.log
python bench.py --no-e2e --no-cpu > ${o}_bench_b.json 2> ${o}_bench.err
python bench.py --no-e2e --no-cpu --workload resnet1 --steps 50 > ${o}_bench_resnet1.json 2>> ${o}_bench.err
timeout 300 python tools/winpack_probe.py > ${o}_winpack_layers.json 2>> ${o}_bench.err
python - <<'P'
import json
for f in ('bench_b', 'bench_resnet1'):
    d = json.loads(open(f'gpurun_out/r02zs_{f}.json').read().strip().splitlines()[-1])
    print(f, round(d['ms_per_step'], 4), d['parity']['result'], d.get('breakdown'))
for b in json.load(open('gpurun_out/r02zs_winpack_layers.json')): print(b['layer'], round(b['win_us'],1), round(b['win_gbs']))
P
