timeout 300 python tools/winpack_probe.py > gpurun_out/w47_winpack.json 2>&1
echo done
