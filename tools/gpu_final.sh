#!/bin/bash
# Round-end GPU session: parity suite, smoke, bench (both arms), ncu launch list and one
# full capture of a step's kernels (summarised on the box: .ncu-rep files stay in /tmp),
# layer sweep, limit study, every BASELINE config.  Outputs gpurun_out/${1}_*.
tag=${1:-final}
o=gpurun_out/${tag}
timeout 1500 python -m pytest tests -q -m gpu > ${o}_pytest_gpu.log 2>&1; echo rc=$? >> ${o}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1
timeout 600 python bench.py > ${o}_bench.json 2> ${o}_bench.err
timeout 600 python bench.py --impl reference > ${o}_bench_reference.json 2>> ${o}_bench.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > ${o}_plain2.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > ${o}_ncu_launch.log 2>&1
python tools/ncu_summary.py launch ${o}_launches.csv ${o}_launches.json
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tc_conv_kernel|bitpack_group" -c 4 \
  -o /tmp/${tag}_full python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-graph > ${o}_ncu_full.log 2>&1
python tools/ncu_summary.py full /tmp/${tag}_full.ncu-rep ${o}_ncu_full.json
ncu -i /tmp/${tag}_full.ncu-rep --page details --csv > ${o}_ncu_details.csv 2>/dev/null
timeout 600 python tools/layer_sweep.py --tc > ${o}_layer_sweep.json 2>> ${o}_bench.err
timeout 900 python tools/limit_study.py --path tc > ${o}_limit_study_tc.json 2>> ${o}_bench.err
bash tools/bench_all.sh ${tag}
echo done
