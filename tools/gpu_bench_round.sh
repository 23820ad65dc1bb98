#!/bin/bash
# One GPU session: plain bench (JSON line), launch list under ncu, and a full ncu capture
# of the ten conv launches of one step (traffic per launch).  Outputs in gpurun_out/$1_*.
tag=${1:-run}
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || exit 1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_plain2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -c 10 \
    -o gpurun_out/${tag}_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-graph \
    > gpurun_out/${tag}_ncu_full.log 2>&1
echo done
