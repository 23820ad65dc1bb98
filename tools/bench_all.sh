#!/bin/bash
# Every BASELINE config through bench.py (one JSON line each, both conv/GEMM paths) into
# gpurun_out/${1:-all}_bench_all.jsonl.  configs[0] conv1, [1] gemv, [2] resnet1 (3
# precisions x 2 encodings), [3] resnet256 (default), [4] gemm sweep.
tag=${1:-all}
out=gpurun_out/${tag}_bench_all.jsonl
err=gpurun_out/${tag}_bench_all.err
run() { timeout 300 python bench.py --no-cpu --no-e2e "$@" >> $out 2>>$err || echo "{\"failed\": \"$*\"}" >> $out; }
for path in tc popc; do
  run --workload resnet256 --path $path
  run --workload conv1 --steps 50 --path $path
  for p in "1 1" "2 1" "2 2"; do set -- $p
    run --workload resnet1 --steps 50 --a-bits $1 --w-bits $2 --path $path
    run --workload resnet1 --steps 50 --a-bits $1 --w-bits $2 --unipolar --path $path
  done
  for s in 4096 8192 16384; do for p in "1 1" "2 1" "4 2"; do set -- $p
    run --workload gemm --size $s --steps 5 --a-bits $1 --w-bits $2 --path $path
  done; done
done
run --workload gemv --steps 50
run --workload resnet256 --tc-format i8
