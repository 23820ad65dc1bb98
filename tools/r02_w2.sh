python tools/tcw_one.py --layers 11 > /dev/null 2>&1 || echo FAIL
ncu --set full --clock-control none -k regex:tcw_conv -c 1 -s 1 -o gpurun_out/w2_l11 python tools/tcw_one.py --layers 11 > gpurun_out/w2_ncu_l11.log 2>&1
ncu --set full --clock-control none -k regex:tcw_conv -c 1 -s 1 -o gpurun_out/w2_l2 python tools/tcw_one.py --layers 2 > gpurun_out/w2_ncu_l2.log 2>&1
for b in 16 64 256; do python tools/tcw_probe.py --layers --batch $b --groups all --reps 10 > gpurun_out/w2_probe_b$b.json 2>&1; done
echo done
