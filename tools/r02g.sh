python tools/one_layer.py 2 > gpurun_out/r02g_plain.log 2>&1 || exit 1
for L in 2 9; do
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:tc_conv_kernel -s 2 -c 1 -o /tmp/r02g_l$L python tools/one_layer.py $L > gpurun_out/r02g_ncu_l$L.log 2>&1
ncu -i /tmp/r02g_l$L.ncu-rep --page details --csv > gpurun_out/r02g_l${L}_details.csv 2>&1
ncu -i /tmp/r02g_l$L.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02g_l${L}_src.csv 2>&1
ncu -i /tmp/r02g_l$L.ncu-rep --page raw --csv > gpurun_out/r02g_l${L}_raw.csv 2>&1
done
ls -la gpurun_out/r02g*
echo done
