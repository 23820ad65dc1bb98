python tools/one_layer.py 2 > gpurun_out/r02d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 2 -c 1 -o gpurun_out/r02d_l2 python tools/one_layer.py 2 > gpurun_out/r02d_ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 2 -c 1 -o gpurun_out/r02d_l9 python tools/one_layer.py 9 > gpurun_out/r02d_ncu_l9.log 2>&1
echo done
