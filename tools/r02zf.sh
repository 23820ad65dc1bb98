# round-2 final tree: full GPU parity, smoke, bench lines (default = hybrid step), ncu launch list,
# traffic of the step's conv launches, one full capture of the window-path launch
o=gpurun_out/r02zf
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -rs > ${o}_pytest_gpu.log 2>&1; tail -3 ${o}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; tail -1 ${o}_smoke.log
python bench.py > ${o}_bench.json 2> ${o}_bench.err
python bench.py --impl reference > ${o}_bench_reference.json 2> ${o}_bench_reference.err
python bench.py --path tc > ${o}_bench_tc.json 2> ${o}_bench_tc.err
for w in conv1 resnet1 gemv; do python bench.py --workload $w > ${o}_bench_$w.json 2> ${o}_bench_$w.err; done
python bench.py --workload gemm --size 8192 --no-e2e > ${o}_bench_gemm8192.json 2> ${o}_bench_gemm.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > ${o}_plain2.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > ${o}_ncu_launch.log 2>&1
python tools/ncu_summary.py launch ${o}_launches.csv ${o}_launches.json
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > ${o}_plain1.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum \
    --clock-control none -k "regex:tcw_conv_kernel|tc_conv_kernel" --csv --log-file ${o}_traffic.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > ${o}_ncu_traffic.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcw_conv_kernel -c 1 -o /tmp/r02zf_tcw \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > ${o}_ncu_full.log 2>&1
python tools/ncu_summary.py full /tmp/r02zf_tcw.ncu-rep ${o}_ncu_full_tcw.json
ncu -i /tmp/r02zf_tcw.ncu-rep --page details --csv > ${o}_ncu_details_tcw.csv 2>/dev/null
echo done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -c 1 -o /tmp/r02zf_tc \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > gpurun_out/r02zf_ncu_full_tc.log 2>&1
python tools/ncu_summary.py full /tmp/r02zf_tc.ncu-rep gpurun_out/r02zf_ncu_full_tc.json
echo done2
