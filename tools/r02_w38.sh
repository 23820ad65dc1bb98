python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > gpurun_out/w38_plain.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:digitpack_win -c 1 -s 2 -o gpurun_out/w38_pack python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph > gpurun_out/w38_ncu.log 2>&1
echo done
