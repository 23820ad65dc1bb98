#!/bin/bash
# Step-configuration sweep of the headline workload (configs[3]); one JSON line per variant.
out=${1:-gpurun_out/step_sweep}
mkdir -p $(dirname $out)
run() { tag=$1; shift; python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity "$@" > ${out}_$tag.json 2> ${out}_$tag.err; }
run base_nosplit --no-pack-split
run split_c1 --group-layers '2|4,5,6,7,8,9,10,11,12' --split-pack-ctas-per-sm 1
run split_c2 --group-layers '2|4,5,6,7,8,9,10,11,12' --split-pack-ctas-per-sm 2
run split_c4 --group-layers '2|4,5,6,7,8,9,10,11,12' --split-pack-ctas-per-sm 4
run split_def_c1 --split-pack-ctas-per-sm 1
run split_3_c1 --group-layers '2|4,5,6,7|8,9,10,11,12' --split-pack-ctas-per-sm 1
