timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcw_conv -c 1 -s 1 -o gpurun_out/w41_l2 python tools/tcw_one.py --layers 2 > gpurun_out/w41_ncu.log 2>&1
echo done
