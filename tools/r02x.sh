python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > gpurun_out/r02x_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -k regex:tc_conv_kernel --csv --log-file gpurun_out/r02x_traffic.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > gpurun_out/r02x_ncu_traffic.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02x_plain2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02x_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02x_ncu_launch.log 2>&1
python bench.py --workload gemv --no-e2e --no-cpu --no-parity --steps 2 --warmup 3 > gpurun_out/r02x_gemv_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemv -s 5 -c 1 -o /tmp/r02x_gemv python bench.py --workload gemv --no-e2e --no-cpu --no-parity --steps 2 --warmup 3 > gpurun_out/r02x_ncu_gemv.log 2>&1
ncu -i /tmp/r02x_gemv.ncu-rep --page details --csv > gpurun_out/r02x_gemv_details.csv 2>&1
ncu -i /tmp/r02x_gemv.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02x_gemv_src.csv 2>&1
echo done
