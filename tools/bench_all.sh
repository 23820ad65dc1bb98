# Run bench.py over every BASELINE config (one JSON line each) into gpurun_out/bench_all.jsonl
out=gpurun_out/bench_all.jsonl
python bench.py --workload conv1 --steps 50 >> $out 2>>gpurun_out/bench_all.err
python bench.py --workload gemv --steps 50 >> $out 2>>gpurun_out/bench_all.err
for p in "1 1" "2 1" "2 2"; do set -- $p
  python bench.py --workload resnet1 --steps 50 --a-bits $1 --w-bits $2 --no-cpu >> $out 2>>gpurun_out/bench_all.err
  python bench.py --workload resnet1 --steps 50 --a-bits $1 --w-bits $2 --unipolar --no-cpu --no-e2e >> $out 2>>gpurun_out/bench_all.err
done
for s in 4096 8192 16384; do for p in "1 1" "2 1" "4 2"; do set -- $p
  python bench.py --workload gemm --size $s --steps 5 --a-bits $1 --w-bits $2 --no-cpu --no-e2e >> $out 2>>gpurun_out/bench_all.err
done; done
